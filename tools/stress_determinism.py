"""Race evidence in place of compute-sanitizer racecheck (closed on this pool,
profiles/r02/sanitizer_closed_memcheck.log): every kernel family with an
in-kernel hand-off (the stream-K fix-up flags of the Ozaki passes, the Jacobi
rotation log replayed by other CTAs, the predicated TSQR fallback, the
cluster reductions of the X slicer, a rank group) is run N times back to back
with no host synchronisation between calls and each result is compared BITWISE
with the first.  A race in a hand-off shows up as a differing bit sooner or
later; usage: python tools/stress_determinism.py [N]   (not product code)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1608_02148_b200 as rb  # noqa: E402
import synthetic  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1000


def stress(name, fn, n):
    ref = [t.clone() for t in fn()]
    bad = torch.zeros((), dtype=torch.int64, device="cuda")
    t0 = time.time()
    for _ in range(n):
        out = fn()
        for a, b in zip(out, ref):
            bad += (a != b).sum()
    torch.cuda.synchronize()
    nbad = int(bad.item())
    print("%-44s %6d calls  %7.2f s  differing elements: %d" % (name, n, time.time() - t0, nbad), flush=True)
    return nbad


def main():
    total = 0
    A1, m1 = synthetic.make_config(1)
    A1 = A1.cuda()
    total += stress("cfg1 rsvd (TSQR fallback, register HQR)",
                    lambda: tuple(rb.rsvd(A1, 10, p=10, q=2, seed=m1["seed_omega"], sync=False)[:3]), N)
    A2, m2 = synthetic.make_config(2)
    A2 = A2.cuda()
    total += stress("cfg2 rsvd (Np=64 stream-K, Jacobi replay)",
                    lambda: tuple(rb.rsvd(A2, 50, p=10, q=2, sdist="rademacher", seed=m2["seed_omega"], sync=False)[:3]), N)
    total += stress("cfg2 rsvd l=120 (paired 2-CTA passes)",
                    lambda: tuple(rb.rsvd(A2, 100, p=20, q=1, seed=2, sync=False)[:3]), N // 2)
    A4 = A2.float()
    total += stress("cfg2 FP32 rsvd l=120 (row pairs, cluster slicer)",
                    lambda: tuple(rb.rsvd(A4, 100, p=20, q=1, seed=3, sync=False)[:3]), N // 2)

    def pca():
        o = rb.rpca(A2, 30, p=10, q=1, seed=4, sync=False)
        return o["eigvals"], o["rotation"], o["x"]
    total += stress("cfg2 rpca centre+scale (f(A) slices)", pca, N // 2)
    As, _, _ = synthetic.sparse_plus_lowrank(20000, 500, rank=10, frac=0.05, seed=7)
    As = As.cuda()

    def rr():
        o = rb.rrpca(As, k=10, p=10, q=2, tol=1e-7, maxiter=50, seed=8)
        return o["L"], o["S"]
    total += stress("rrpca 20000x500 (IALM fused update)", rr, max(N // 50, 5))
    Aw = A2[:, :1500].contiguous()
    total += stress("wide plan l=160 (cooperative kernels)",
                    lambda: tuple(rb.rsvd(Aw, 150, p=10, q=1, seed=9, sync=False)[:3]), max(N // 50, 5))
    parts = rb.row_partition(A2.shape[0], 4)

    def grp():
        out = rb.run_ranks(lambda ctx, rk: rb.rsvd(A2[parts[rk][0]:parts[rk][0] + parts[rk][1]], 50, ctx=ctx, p=10, q=2,
                                                   m_global=A2.shape[0], row_offset=parts[rk][0], seed=11), 4)
        return (out[0].d, out[0].v, torch.cat([o.u for o in out], 0))
    total += stress("cfg2 rsvd over a 4-rank group", grp, max(N // 50, 5))
    print("TOTAL differing elements:", total)
    sys.exit(1 if total else 0)


if __name__ == "__main__":
    main()

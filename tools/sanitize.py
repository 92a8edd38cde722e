"""compute-sanitizer driver: one small call of every kernel family on config-1
and a reduced config-2 input (Ozaki passes incl. the 2-CTA paired kernel, the
TSQR fallback, Jacobi with its replay CTAs, rpca, rrpca, rid / rcur, FP32
tcgen05 passes, a rank group).  Not product code."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1608_02148_b200 as rb  # noqa: E402
import synthetic  # noqa: E402

A1, m1 = synthetic.make_config(1)
A1 = A1.cuda()
r = rb.rsvd(A1, 10, p=10, q=2, seed=m1["seed_omega"])                     # rank-deficient: TSQR fallback
A2, _ = synthetic.make_config(2, scale_rows=3000)
A2 = A2[:, :1500].contiguous().cuda()
rb.rsvd(A2, 50, p=10, q=2, sdist="rademacher", seed=1)                     # Np = 64 passes
rb.rsvd(A2, 100, p=20, q=1, seed=2)                                        # Np = 128: paired passes
rb.rpca(A2, 20, p=10, q=1, seed=3, loadings=True, whiten=True, explained=True)
rb.rid(A2, 20, p=10, q=1, seed=4)
rb.rcur(A2, 16, p=10, q=1, seed=5)
rb.rsvd(A2.float(), 30, p=10, q=1, seed=6)                                 # FP32 tcgen05 passes
rb.rsvd(A2, 150, p=10, q=1, seed=9)                                        # wide plan (l = 160): cooperative kernels
As, _, _ = synthetic.sparse_plus_lowrank(2000, 200, rank=5, frac=0.05, seed=7)
rb.rrpca(As.cuda(), k=10, p=10, q=1, tol=1e-6, maxiter=20, seed=8)
parts = rb.row_partition(3000, 2)
rb.run_ranks(lambda ctx, rk: rb.rsvd(A2[parts[rk][0]:parts[rk][0] + parts[rk][1]], 20, ctx=ctx, m_global=3000,
                                     row_offset=parts[rk][0]), 2)
torch.cuda.synchronize()
print("sanitize driver done", float(r.d[0]))

"""Wall time of wide-plan calls (l = k + p > 120) on a config-2-sized matrix; not product code."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1608_02148_b200 as rb
import synthetic

A, meta = synthetic.make_config(2)
A = A.cuda()
ctx = rb.default_context(A.device)
for k in (110, 150, 290, 500):
    rb.rsvd(A, k, p=10, q=2, seed=1)
    torch.cuda.synchronize()
    ctx.profile_reset(); ctx.set_profiling(1)
    t0 = time.perf_counter()
    for _ in range(3):
        rb.rsvd(A, k, p=10, q=2, seed=1)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3 * 1e3
    ctx.set_profiling(False)
    kinds = {i: round(ctx.profile(i)[0] / 3, 3) for i in range(7)}
    print("k=%d l=%d  %.2f ms per rsvd (10000 x 5000, q=2)  per-kind ms %s  sweeps %d" % (k, k + 10, dt, kinds, ctx.stats()["jacobi_sweeps"]), flush=True)

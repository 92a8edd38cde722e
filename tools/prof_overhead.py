"""Step time of the cfg-2 rsvd with profiling off / pass kernels only / every kind."""
import sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
import paper_1608_02148_b200 as rb
import synthetic
A, meta = synthetic.make_config(2)
A = A.cuda()
ctx = rb.default_context(A.device)
out = (torch.empty(50, dtype=torch.float64, device='cuda'), torch.empty(10000, 50, dtype=torch.float64, device='cuda'),
       torch.empty(5000, 50, dtype=torch.float64, device='cuda'))
for _ in range(5):
    rb.rsvd(A, 50, p=10, q=2, sdist="rademacher", seed=meta["seed_omega"], ctx=ctx, out=out)
for level in [0, 2, 1, 0]:
    ctx.set_profiling(level)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        rb.rsvd(A, 50, p=10, q=2, sdist="rademacher", seed=meta["seed_omega"], ctx=ctx, out=out)
    e1.record(); torch.cuda.synchronize()
    ctx.set_profiling(0)
    print("profiling level", level, "%.4f ms/step" % (e0.elapsed_time(e1) / 50))

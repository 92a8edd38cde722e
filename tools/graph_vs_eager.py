"""Probe (not product code): one rsvd per step, eager back-to-back calls vs a
captured CUDA graph replayed, configs 1 and 2; CUDA-event timing.
python tools/graph_vs_eager.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1608_02148_b200 as rb
import synthetic

for cfg, k in ((1, 10), (2, 50)):
    A, meta = synthetic.make_config(cfg)
    A = A.cuda()
    st = torch.cuda.Stream()
    ctx = rb.Context(0, st)
    kw = dict(p=meta["p"], q=meta["q"], sdist=meta["sdist"], seed=meta["seed_omega"], ctx=ctx)
    with torch.cuda.stream(st):
        ref = rb.rsvd(A, k, **kw)
        d, u, v = torch.empty_like(ref.d), torch.empty_like(ref.u), torch.empty_like(ref.v)
        for _ in range(5):
            rb.rsvd(A, k, out=(d, u, v), sync=False, **kw)
        ctx.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 200
        e0.record(st)
        for _ in range(n):
            rb.rsvd(A, k, out=(d, u, v), sync=False, **kw)
        e1.record(st)
        ctx.sync()
        torch.cuda.synchronize()
        eager = e0.elapsed_time(e1) / n
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            rb.rsvd(A, k, out=(d, u, v), sync=False, **kw)
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(n):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        graph = e0.elapsed_time(e1) / n
    print("cfg %d: eager %.4f ms  graph %.4f ms per rsvd" % (cfg, eager, graph), flush=True)

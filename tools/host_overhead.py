"""Host enqueue time per call (ctypes + library host code) vs GPU time per call,
and a CUDA-graph replay of the same call.  Not product code."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1608_02148_b200 as rb
import synthetic

for cfg in (1, 2, 3):
    A, meta = synthetic.make_config(cfg, device="cuda")
    k, p, q = meta["k"], meta["p"], meta["q"]
    st = torch.cuda.Stream()
    ctx = rb.Context(0, st)
    kw = dict(p=p, q=q, sdist=meta["sdist"], seed=meta["seed_omega"], ctx=ctx)
    with torch.cuda.stream(st):
        if meta["center"]:
            call = lambda: rb.rpca(A, k, center=True, scale=False, sync=False, **kw)  # noqa: E731
        else:
            d = torch.empty(k, dtype=A.dtype, device="cuda"); u = torch.empty(A.shape[0], k, dtype=A.dtype, device="cuda")
            v = torch.empty(A.shape[1], k, dtype=A.dtype, device="cuda")
            call = lambda: rb.rsvd(A, k, out=(d, u, v), sync=False, **kw)  # noqa: E731
        for _ in range(3):
            call()
        ctx.sync()
        n = 20
        t0 = time.perf_counter()
        for _ in range(n):
            call()
        t_host = (time.perf_counter() - t0) / n
        ctx.sync()
        t_all = (time.perf_counter() - t0) / n
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            call()
        g.replay(); ctx.sync()
        t0 = time.perf_counter()
        for _ in range(n):
            g.replay()
        t_gh = (time.perf_counter() - t0) / n
        ctx.sync()
        t_g = (time.perf_counter() - t0) / n
    print("cfg%d host enqueue %.3f ms  stream total %.3f ms | graph replay host %.3f ms total %.3f ms" %
          (cfg, t_host * 1e3, t_all * 1e3, t_gh * 1e3, t_g * 1e3), flush=True)
    del A

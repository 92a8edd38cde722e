"""Host-side logic of the row-sharded (multi-GPU) path, on CPU with the gloo
backend, world size 2.  No GPU: the NCCL kernels themselves are
not exercised, but everything around them is:

* the sharding algebra the library relies on: per-rank partials of A^T Q,
  of the Gram Y^T Y and of the column sums, summed across ranks, equal the
  unsharded quantities (computed here with the oracle's own routines);
* a row-sharded subspace iteration (Alg. 2) with allreduced Grams reproduces
  the single-process oracle's singular values;
* the NCCL unique id made by the library on rank 0 reaches every rank intact
  through torch.distributed (the plumbing of Context.init_comm);
* bench.py's max-over-ranks timing reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synthetic
        res = {}
        A, _ = synthetic.lowrank(600, 120, torch.as_tensor(np.exp(-np.arange(120) / 10.0)), noise=1e-9, seed=4)
        A = A.numpy()
        m, n = A.shape
        rows = [(m * r) // world for r in range(world + 1)]
        Ar = A[rows[rank]:rows[rank + 1]]
        l = 20
        # (1) sharding algebra: A^T Q, Y^T Y, column sums
        Om = oracle.omega(n, l, "normal", seed=9)
        Yr = Ar @ Om
        Z = torch.from_numpy(np.ascontiguousarray(Ar.T @ Yr))
        G = torch.from_numpy(np.ascontiguousarray(Yr.T @ Yr))
        c = torch.from_numpy(np.ascontiguousarray(Ar.sum(axis=0)))
        for t in (Z, G, c):
            dist.all_reduce(t)
        Y = A @ Om
        res["atq"] = float(np.abs(Z.numpy() - A.T @ Y).max() / np.abs(A.T @ Y).max())
        res["gram"] = float(np.abs(G.numpy() - Y.T @ Y).max() / np.abs(Y.T @ Y).max())
        res["colsum"] = float(np.abs(c.numpy() - A.sum(axis=0)).max())
        # (2) row-sharded subspace iteration with CholeskyQR (allreduced Gram), as the library does
        def orth_dist(Yloc):
            Gl = torch.from_numpy(np.ascontiguousarray(Yloc.T @ Yloc))
            dist.all_reduce(Gl)
            R = np.linalg.cholesky(Gl.numpy()).T
            return np.linalg.solve(R.T, Yloc.T).T
        Yl = Yr
        for _ in range(2):
            Ql = orth_dist(Yl)
            Zt = torch.from_numpy(np.ascontiguousarray(Ar.T @ Ql))
            dist.all_reduce(Zt)
            Qz, _ = oracle.hqr(Zt.numpy())
            Yl = Ar @ Qz
        Ql = orth_dist(orth_dist(Yl))
        Bt = torch.from_numpy(np.ascontiguousarray(Ar.T @ Ql))
        dist.all_reduce(Bt)
        d = np.linalg.svd(Bt.numpy(), compute_uv=False)
        o = oracle.oracle_rsvd(A, 10, p=10, q=2, sdist="normal", seed=9)
        res["d"] = float(np.max(np.abs(d[:10] - o["d"]) / o["d"]))
        # (3) NCCL unique id plumbing (library call on rank 0, broadcast to all)
        import ctypes
        import paper_1608_02148_b200 as rb
        buf = ctypes.create_string_buffer(128)
        if rank == 0:
            assert rb.lib().rsvd_nccl_unique_id(buf) == 0
        obj = [bytes(buf.raw)]
        dist.broadcast_object_list(obj, src=0)
        digest = torch.tensor(list(obj[0][:16]), dtype=torch.int64)
        ref = digest.clone()
        dist.broadcast(ref, src=0)
        res["uid_same"] = bool(torch.equal(digest, ref)) and len(obj[0]) == 128 and any(obj[0])
        # (4) max-over-ranks timing
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res["tmax"] = float(t.item())
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_row_sharded_algebra_gloo():
    try:
        from paper_1608_02148_b200 import build
        build.build()
    except Exception as e:   # pragma: no cover
        pytest.skip("library not buildable here: %s" % e)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        res = out[r]
        assert res["atq"] < 1e-13 and res["gram"] < 1e-13 and res["colsum"] < 1e-11
        assert res["d"] < 1e-10
        assert res["uid_same"]
        assert res["tmax"] == 2.0

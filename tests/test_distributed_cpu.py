"""Host-side code of the row-sharded (multi-GPU) path, on CPU with the gloo
backend, world size 2.  The library's nranks > 1 path itself
(collectives inside rsvd / rpca / rrpca) needs a GPU and runs in
tests/test_gpu_distributed.py as an in-process rank group; here, without a
GPU, the product code around it is exercised with real processes:

* rb.row_partition -- the row blocks every rank (bench.py, the tests, users)
  takes; checked as an exact partition and against the per-rank partial sums
  the library's allreduces combine (A^T Q, the Gram Y^T Y, the column sums:
  Alg. 4 steps (3), (10)), each rank computing only on
  its own block and the sums reduced over gloo;
* the NCCL unique id made by the library's rsvd_nccl_unique_id on rank 0
  reaching every rank intact through torch.distributed (the plumbing of
  Context.init_comm);
* bench.py's per-rank bookkeeping: its row block, the algorithmic bytes of a
  step and the max-over-ranks timing reduction.
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
        import ctypes

        import bench
        import paper_1608_02148_b200 as rb
        import synthetic
        res = {}
        A, _ = synthetic.lowrank(601, 120, torch.as_tensor(np.exp(-np.arange(120) / 10.0)), noise=1e-9, seed=4)
        A = A.numpy()
        m, n = A.shape
        parts = rb.row_partition(m, world)
        off, rows = parts[rank]
        # (1) the partition is exact and contiguous
        res["partition_ok"] = (sum(r for _, r in parts) == m and parts[0][0] == 0 and
                               all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(world - 1)))
        Ar = A[off:off + rows]
        rng = np.random.default_rng(9)
        Om = rng.standard_normal((n, 20))
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
        # (2) NCCL unique id plumbing (library call on rank 0, broadcast to all)
        buf = ctypes.create_string_buffer(128)
        if rank == 0:
            assert rb.lib().rsvd_nccl_unique_id(buf) == 0
        obj = [bytes(buf.raw)]
        dist.broadcast_object_list(obj, src=0)
        digest = torch.tensor(list(obj[0][:16]), dtype=torch.int64)
        ref = digest.clone()
        dist.broadcast(ref, src=0)
        res["uid_same"] = bool(torch.equal(digest, ref)) and len(obj[0]) == 128 and any(obj[0])
        # (3) bench.py bookkeeping: step bytes depend only on the global shape;
        # the step time is the max over ranks
        meta = dict(q=2, center=False)
        res["step_bytes"] = bench.step_bytes_for(meta, m, n, 8)
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res["tmax"] = float(t.item())
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_row_sharded_host_code_gloo():
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
        assert res["partition_ok"]
        assert res["atq"] < 1e-13 and res["gram"] < 1e-13 and res["colsum"] < 1e-11
        assert res["uid_same"]
        assert res["tmax"] == 2.0
        assert res["step_bytes"] == 6 * 601 * 120 * 8

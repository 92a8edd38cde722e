"""The library's row-sharded (nranks > 1) path, executed on ONE GPU through an
in-process rank group (rsvd_group): R contexts, one host thread
and one stream each, rank r holding rows [offset_r, offset_r + m_r) of A; the
collectives (the n x l allreduce of A^T Q, the l x l Gram allreduce of
CholeskyQR, the column sums of rpca, the allgather of the TSQR fallback, the
IALM scalars) are fixed-rank-order device reductions.  Alg. 4 steps (3) and
(10) computed per row block and summed.

Checks: d equal to the 1-rank run within 1e-12 relative and to the oracle
within 1e-10 (BASELINE.json north_star FP64 tolerance); U (gathered rows) and V
orthonormal to 1e-12; the rank-deficient config 1 exercises the distributed
TSQR fallback."""
import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1608_02148_b200 as rb
    return rb


def _np(t):
    return t.detach().cpu().numpy().astype(np.float64)


def _sharded_rsvd(rb, A, k, world, **kw):
    """rsvd of the device matrix A split into `world` row blocks; returns
    (d, U gathered in row order, V, fallback flags per rank)."""
    m = A.shape[0]
    parts = rb.row_partition(m, world)

    def fn(ctx, r):
        off, rows = parts[r]
        res = rb.rsvd(A[off:off + rows], k, ctx=ctx, m_global=m, row_offset=off, sync=False, **kw)
        ctx.sync()
        return res, ctx.stats()["tsqr_fallback"]

    out = rb.run_ranks(fn, world)
    d0 = out[0][0].d
    for res, _ in out[1:]:
        assert torch.equal(res.d, d0), "ranks disagree on d"
        assert torch.equal(res.v, out[0][0].v), "ranks disagree on V"
    U = torch.cat([res.u for res, _ in out], dim=0)
    return _np(d0), _np(U), _np(out[0][0].v), [f for _, f in out]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_config1_sharded_exact_rank(rb, world):
    """Config 1 (exact rank 10, l = 20) row-sharded: every rank's CholeskyQR of
    the rank-deficient sketch breaks down, the distributed TSQR fallback
    (local TSQR, allgather of the R factors, QR of the stack) runs, and the
    planted singular values come back to 1e-12 (J:7)."""
    A, meta = synthetic.make_config(1)
    Ad = A.cuda()
    d, U, V, fb = _sharded_rsvd(rb, Ad, 10, world, p=10, q=2, sdist="normal", seed=meta["seed_omega"])
    s = meta["s"].numpy()
    assert np.max(np.abs(d - s) / s) <= 1e-12
    assert all(fb), "the TSQR fallback should have run on every rank"
    assert np.abs(U.T @ U - np.eye(10)).max() <= 1e-12
    assert np.abs(V.T @ V - np.eye(10)).max() <= 1e-12
    o = oracle.oracle_rsvd(A.numpy(), 10, p=10, q=2, sdist="normal", seed=meta["seed_omega"])
    assert np.max(np.abs(d - o["d"]) / o["d"]) <= 1e-10
    r1 = rb.rsvd(Ad, 10, p=10, q=2, sdist="normal", seed=meta["seed_omega"])
    assert np.max(np.abs(d - _np(r1.d)) / _np(r1.d)) <= 1e-12


@pytest.mark.parametrize("world", [2, 4, 8])
def test_config2_sharded(rb, world):
    """Config 2 (J:8, 10000 x 5000, Rademacher Omega) row-sharded over 2/4/8
    ranks: d within 1e-12 of the 1-rank run and 1e-10 of the oracle, the
    reconstruction error within 1.0001 x the oracle's (+1e-13, R24)."""
    A, meta = synthetic.make_config(2)
    Ad = A.cuda()
    kw = dict(p=10, q=2, sdist="rademacher", seed=meta["seed_omega"])
    d, U, V, _ = _sharded_rsvd(rb, Ad, 50, world, **kw)
    r1 = rb.rsvd(Ad, 50, **kw)
    d1 = _np(r1.d)
    assert np.max(np.abs(d - d1) / d1) <= 1e-12
    o = oracle.oracle_rsvd(A.numpy(), 50, **kw)
    assert np.max(np.abs(d - o["d"]) / o["d"]) <= 1e-10
    assert np.abs(U.T @ U - np.eye(50)).max() <= 1e-12
    An = A.numpy()
    e = np.linalg.norm(An - (U * d) @ V.T) / np.linalg.norm(An)
    eo = np.linalg.norm(An - (o["u"] * o["d"]) @ o["v"].T) / np.linalg.norm(An)
    assert e <= 1.0001 * eo + 1e-13


@pytest.mark.parametrize("world", [2, 3])
def test_rpca_sharded_matches_single_rank(rb, world):
    """rpca with centring and scaling row-sharded: the column means and s.d. are
    allreduced, everything else matches the 1-rank run and the oracle."""
    g = torch.Generator().manual_seed(4)
    A = (torch.randn(6000, 300, generator=g, dtype=torch.float64) *
         torch.exp(-torch.arange(300, dtype=torch.float64) / 40) + torch.linspace(0, 5, 300, dtype=torch.float64))
    Ad = A.cuda()
    parts = rb.row_partition(A.shape[0], world)

    def fn(ctx, r):
        off, rows = parts[r]
        return rb.rpca(Ad[off:off + rows], 20, center=True, scale=True, p=10, q=2, seed=3, ctx=ctx,
                       m_global=A.shape[0], row_offset=off, explained=True)

    out = rb.run_ranks(fn, world)
    one = rb.rpca(Ad, 20, center=True, scale=True, p=10, q=2, seed=3, explained=True)
    o = oracle.oracle_rpca(A.numpy(), 20, center=True, scale=True, p=10, q=2, seed=3)
    for key in ("eigvals", "center", "scale", "var_ratio"):
        got = _np(out[0][key])
        assert np.max(np.abs(got - _np(one[key])) / np.abs(_np(one[key]))) <= 1e-12, key
        assert np.max(np.abs(got - o[key]) / np.abs(o[key])) <= 1e-10, key
    x = np.concatenate([_np(res["x"]) for res in out], axis=0)
    assert np.linalg.norm(x - o["x"]) / np.linalg.norm(o["x"]) < 1e-9


def test_rrpca_sharded(rb):
    """rrpca (Alg. 7) over 2 ranks: the IALM scalars (||A||_F^2 partials, max|A|,
    the residual) are allreduced; same iterations and L, S as the 1-rank run."""
    A, L0, S0 = synthetic.sparse_plus_lowrank(4000, 300, rank=5, frac=0.05, seed=12)
    Ad = A.cuda()
    parts = rb.row_partition(A.shape[0], 2)

    def fn(ctx, r):
        off, rows = parts[r]
        return rb.rrpca(Ad[off:off + rows].contiguous(), k=10, p=10, q=2, tol=1e-7, maxiter=100, seed=3, ctx=ctx,
                        m_global=A.shape[0], row_offset=off)

    out = rb.run_ranks(fn, 2)
    one = rb.rrpca(Ad, k=10, p=10, q=2, tol=1e-7, maxiter=100, seed=3)
    assert out[0]["iters"] == out[1]["iters"] == one["iters"]
    L = np.concatenate([_np(o["L"]) for o in out], axis=0)
    S = np.concatenate([_np(o["S"]) for o in out], axis=0)
    assert np.linalg.norm(L - _np(one["L"])) / np.linalg.norm(_np(one["L"])) < 1e-10
    assert np.linalg.norm(S - _np(one["S"])) / np.linalg.norm(_np(one["S"])) < 1e-10
    assert np.linalg.norm(L - L0.numpy()) / np.linalg.norm(L0.numpy()) < 1e-6


def test_group_abort_releases_peers(rb):
    """A member failing inside a call (bad argument after the group formed) must
    not hang the others: they see RSVD_ENCCL / an exception, not a deadlock."""
    A = torch.randn(2000, 100, dtype=torch.float64, device="cuda")
    parts = rb.row_partition(2000, 2)

    def fn(ctx, r):
        off, rows = parts[r]
        if r == 1:
            # rank 1 asks for an impossible k: it fails validation before any
            # collective, which aborts the group, so rank 0 is released
            rb.rsvd(A[off:off + rows], 500, ctx=ctx, m_global=2000, row_offset=off)
        return rb.rsvd(A[off:off + rows], 10, ctx=ctx, m_global=2000, row_offset=off)

    with pytest.raises(Exception):
        rb.run_ranks(fn, 2)


@pytest.mark.parametrize("world", [2, 3])
def test_fp32_sharded_row_pairs(rb, world):
    """FP32 A (config 4's path: 3-digit Ozaki slices, l = 120 -> the row-pair
    cta_group::2 pass, 4096-row X exponent blocks) row-sharded over 2 / 3 ranks
    of unequal row counts: ranks agree bitwise on d and V, d within 1e-5 of
    the 1-rank run (the slices of each rank's rows carry the same per-row
    exponents; only the reduction split of A^T Q differs) and within 1e-4 of
    the FP64 oracle on the same FP32 data (J:5)."""
    g = torch.Generator().manual_seed(31)
    m, n = 9001, 1300
    U = torch.linalg.qr(torch.randn(m, 200, generator=g, dtype=torch.float64))[0]
    V = torch.linalg.qr(torch.randn(n, 200, generator=g, dtype=torch.float64))[0]
    s = torch.exp(-torch.arange(200, dtype=torch.float64) / 50.0)
    A = ((U * s) @ V.T + 1e-4 * torch.randn(m, n, generator=g, dtype=torch.float64)).to(torch.float32)
    Ad = A.cuda()
    d, Ug, Vg, _ = _sharded_rsvd(rb, Ad, 100, world, p=20, q=2, sdist="normal", seed=7)
    assert np.abs(Ug.T @ Ug - np.eye(100)).max() <= 1e-5
    r1 = rb.rsvd(Ad, 100, p=20, q=2, sdist="normal", seed=7)
    d1 = _np(r1.d)
    assert np.max(np.abs(d - d1) / d1) <= 1e-5
    o = oracle.oracle_rsvd(A.numpy().astype(np.float64), 100, p=20, q=2, sdist="normal", seed=7)
    assert np.max(np.abs(d - o["d"]) / o["d"]) <= 1e-4


@pytest.mark.parametrize("world", [2, 3])
def test_wide_plan_sharded(rb, world):
    """A wide plan (l = 170 > 120, reading R34) row-sharded: the Gram of every
    shifted-CholeskyQR3 panel is allreduced, the cooperative Cholesky and the
    grid-wide Jacobi run redundantly on every rank (identical bits); d within
    1e-12 of the 1-rank run and 1e-10 of the oracle, U and V orthonormal."""
    s = np.exp(-np.arange(600) / 100.0)
    A, _ = synthetic.lowrank(2500, 600, torch.as_tensor(s), noise=1e-8, seed=44)
    Ad = A.cuda()
    d, U, V, _ = _sharded_rsvd(rb, Ad, 150, world, p=20, q=2, seed=8)
    r1 = rb.rsvd(Ad, 150, p=20, q=2, seed=8)
    assert np.max(np.abs(d - _np(r1.d)) / _np(r1.d)) <= 1e-12
    o = oracle.oracle_rsvd(A.numpy(), 150, p=20, q=2, seed=8)
    assert np.max(np.abs(d - o["d"]) / o["d"]) <= 1e-10
    assert np.abs(U.T @ U - np.eye(150)).max() <= 1e-12
    assert np.abs(V.T @ V - np.eye(150)).max() <= 1e-12


def test_one_rank_nccl_communicator(rb, monkeypatch):
    """The NCCL communicator itself on ONE GPU (RSVD_NCCL_SINGLE=1: a one-rank
    ncclCommInitRank; every Gram / A^T X / column-sum / IALM-scalar allreduce of
    the call is then a real in-stream ncclAllReduce, an identity at one rank,
    followed by the library's stream fence).  rsvd, rpca and rrpca must equal the
    communicator-free run bitwise (Alg. 4 steps (3)/(10))."""
    monkeypatch.setenv("RSVD_NCCL_SINGLE", "1")
    ctx = rb.Context()
    ctx.init_comm(0, 1)
    monkeypatch.delenv("RSVD_NCCL_SINGLE")
    A, meta = synthetic.make_config(1)
    Ad = A.cuda()
    kw = dict(p=10, q=2, sdist="normal", seed=meta["seed_omega"])
    r0 = rb.rsvd(Ad, 10, **kw)
    r1 = rb.rsvd(Ad, 10, ctx=ctx, **kw)
    assert torch.equal(r0.d, r1.d) and torch.equal(r0.u, r1.u) and torch.equal(r0.v, r1.v)
    g = torch.Generator().manual_seed(5)
    B = (torch.randn(3000, 40, generator=g, dtype=torch.float64) @ torch.randn(40, 300, generator=g, dtype=torch.float64)
         + 3.0 + 0.01 * torch.randn(3000, 300, generator=g, dtype=torch.float64)).cuda()
    p0 = rb.rpca(B, 20, seed=3)
    p1 = rb.rpca(B, 20, seed=3, ctx=ctx)
    for key in ("eigvals", "rotation", "x", "center", "scale"):
        assert torch.equal(p0[key], p1[key]), key
    L0 = torch.randn(400, 5, generator=g, dtype=torch.float64) @ torch.randn(5, 200, generator=g, dtype=torch.float64)
    S0 = torch.zeros(400, 200, dtype=torch.float64)
    idx = torch.rand(400, 200, generator=g) < 0.05
    S0[idx] = 10.0 * torch.randn(int(idx.sum()), generator=g, dtype=torch.float64)
    M = (L0 + S0).cuda()
    q0 = rb.rrpca(M, k=10, maxiter=20, seed=1)
    q1 = rb.rrpca(M, k=10, maxiter=20, seed=1, ctx=ctx)
    assert q0["iters"] == q1["iters"]
    assert torch.equal(q0["L"], q1["L"]) and torch.equal(q0["S"], q1["S"])


def test_host_buffer_calls_sharded(rb):
    """The host-buffer C-ABI calls on a row-sharded matrix (2 ranks): each rank
    passes its own rows from host memory (m_global / row_offset place them), the
    library copies them in, runs the sharded path and copies its rows of U / the
    scores back.  Results equal the device-buffer sharded run bitwise and the
    1-rank run to 1e-12 (Alg. 4 steps (3)/(10); Alg. 6)."""
    A, meta = synthetic.make_config(2, scale_rows=3000)
    A = A[:, :1200].contiguous()
    Ad = A.cuda()
    m = A.shape[0]
    world = 2
    parts = rb.row_partition(m, world)
    kw = dict(p=10, q=2, sdist="rademacher", seed=meta["seed_omega"])

    def fn_host(ctx, r):
        off, rows = parts[r]
        blk = A[off:off + rows].contiguous().pin_memory()
        res = rb.rsvd_host(blk, 30, ctx=ctx, m_global=m, row_offset=off, **kw)
        pca = rb.rpca(blk, 20, ctx=ctx, m_global=m, row_offset=off, seed=3)
        return res, pca

    def fn_dev(ctx, r):
        off, rows = parts[r]
        res = rb.rsvd(Ad[off:off + rows], 30, ctx=ctx, m_global=m, row_offset=off, **kw)
        pca = rb.rpca(Ad[off:off + rows], 20, ctx=ctx, m_global=m, row_offset=off, seed=3)
        return res, pca

    oh = rb.run_ranks(fn_host, world)
    od = rb.run_ranks(fn_dev, world)
    for (rh, ph), (rd, pd) in zip(oh, od):
        assert not rh.d.is_cuda and not ph["x"].is_cuda
        assert torch.equal(rh.d, rd.d.cpu()) and torch.equal(rh.u, rd.u.cpu()) and torch.equal(rh.v, rd.v.cpu())
        for key in ("eigvals", "rotation", "x", "center", "scale", "sdev"):
            assert torch.equal(ph[key], pd[key].cpu()), key
    r1 = rb.rsvd(Ad, 30, **kw)
    d1 = _np(r1.d)
    assert np.max(np.abs(_np(oh[0][0].d) - d1) / d1) <= 1e-12
    p1 = rb.rpca(Ad, 20, seed=3)
    e1 = _np(p1["eigvals"])
    assert np.max(np.abs(_np(oh[0][1]["eigvals"]) - e1) / e1) <= 1e-12
    x = torch.cat([o[1]["x"] for o in oh], 0)
    assert x.shape == (m, 20)
    # rrpca through rsvd_rrpca_host on the same two ranks
    As, _, _ = synthetic.sparse_plus_lowrank(2000, 200, rank=5, frac=0.05, seed=7)
    Asd = As.cuda()
    parts2 = rb.row_partition(2000, world)

    def rr(host):
        def fn(ctx, r):
            off, rows = parts2[r]
            blk = As[off:off + rows].contiguous() if host else Asd[off:off + rows]
            return rb.rrpca(blk, k=10, p=10, q=2, tol=1e-7, maxiter=60, seed=8, ctx=ctx, m_global=2000, row_offset=off)
        return rb.run_ranks(fn, world)

    qh, qd = rr(True), rr(False)
    for a, b in zip(qh, qd):
        assert a["iters"] == b["iters"]
        assert torch.equal(a["L"], b["L"].cpu()) and torch.equal(a["S"], b["S"].cpu())

"""The C-ABI boundary on the GPU (include/rsvd_b200.h): non-blocking calls and
rsvd_sync, CUDA-graph capture of a whole rsvd, the host-buffer entry point,
the workspace query, and the full rpca output set (Alg. 6 and the quantities
of PAPER.md:1239-1302, 1391-1402) plus predict() against the oracle."""
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


def _decay(m, n, seed, noise=1e-8):
    s = np.exp(-np.arange(min(m, n)) / 15.0)
    A, _ = synthetic.lowrank(m, n, torch.as_tensor(s), noise=noise, seed=seed)
    return A


def test_calls_do_not_block_and_sync_reports(rb):
    """rsvd_run only enqueues (sync=False); the results after Context.sync()
    equal the synchronous call's bit for bit; a non-finite input is reported
    by rsvd_sync as RSVD_ENUMERIC, not by the enqueueing call."""
    A = _decay(3000, 800, seed=3).cuda()
    ctx = rb.Context(0)
    r_async = rb.rsvd(A, 20, seed=5, ctx=ctx, sync=False)
    ctx.sync()
    r_sync = rb.rsvd(A, 20, seed=5, ctx=ctx)
    assert torch.equal(r_async.d, r_sync.d) and torch.equal(r_async.u, r_sync.u) and torch.equal(r_async.v, r_sync.v)
    B = A.clone()
    B[17, 3] = float("nan")
    rb.rsvd(B, 20, seed=5, ctx=ctx, sync=False)          # enqueued without complaint
    with pytest.raises(rb.RsvdError) as ei:
        ctx.sync()
    assert ei.value.status == 5
    r_after = rb.rsvd(A, 20, seed=5, ctx=ctx)             # the status was cleared by the sync
    assert torch.equal(r_after.d, r_sync.d)


@pytest.mark.parametrize("cfg_shape", [(10000, 5000, 50, "rademacher"), (1000, 500, 10, "normal")])
def test_whole_rsvd_captured_in_a_cuda_graph(rb, cfg_shape):
    """One rsvd (Omega, the 2q+2 passes, every orthonormalisation incl. the
    device-side TSQR fallback of the rank-deficient case, Jacobi, outputs)
    captured into a CUDA graph and replayed: same bits as the eager call."""
    m, n, k, sd = cfg_shape
    if m == 1000:
        A, meta = synthetic.make_config(1)
    else:
        A, meta = synthetic.make_config(2)
    A = A.cuda()
    st = torch.cuda.Stream()
    ctx = rb.Context(0, st)
    kw = dict(p=10, q=2, sdist=sd, seed=meta["seed_omega"], ctx=ctx)
    with torch.cuda.stream(st):
        ref = rb.rsvd(A, k, **kw)                         # warm-up: sizes every workspace
        d = torch.empty_like(ref.d)
        u = torch.empty_like(ref.u)
        v = torch.empty_like(ref.v)
        rb.rsvd(A, k, out=(d, u, v), sync=False, **kw)
        ctx.sync()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            rb.rsvd(A, k, out=(d, u, v), sync=False, **kw)
        d.zero_(); u.zero_(); v.zero_()
        g.replay()
        ctx.sync()
    assert torch.equal(d, ref.d) and torch.equal(u, ref.u) and torch.equal(v, ref.v)


def test_run_host_matches_device_run(rb):
    """rsvd_run_host (HOST buffers in and out, copies inside the call) gives
    the device call's bits and the oracle's values."""
    A = _decay(4000, 700, seed=12)
    Ah = A.pin_memory()
    r_h = rb.rsvd_host(Ah, 25, p=10, q=2, seed=9)
    r_d = rb.rsvd(A.cuda(), 25, p=10, q=2, seed=9)
    assert not r_h.d.is_cuda
    assert torch.equal(r_h.d, r_d.d.cpu()) and torch.equal(r_h.u, r_d.u.cpu()) and torch.equal(r_h.v, r_d.v.cpu())
    o = oracle.oracle_rsvd(A.numpy(), 25, p=10, q=2, seed=9)
    assert np.max(np.abs(_np(r_h.d) - o["d"]) / o["d"]) <= 1e-10


def test_workspace_bytes(rb):
    """rsvd_workspace_bytes sizes what rsvd_run then owns: at least the 7-byte
    Ozaki slices of an FP64 A plus the m x l panels, and the run fits in it."""
    A = _decay(8000, 2000, seed=4).cuda()
    ctx = rb.Context(0)
    need = ctx.workspace_bytes(A, 40, p=10, q=2)
    assert need >= 7 * 8000 * 2048 + 8 * 8000 * 64
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    free0 = torch.cuda.mem_get_info()[0]
    rb.rsvd(A, 40, ctx=ctx)
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 <= need + (64 << 20)            # library-owned growth within the query (+ slack)
    assert torch.cuda.memory_allocated() - before < (64 << 20)


@pytest.mark.parametrize("scale", [False, True])
def test_rpca_full_outputs_vs_oracle(rb, scale):
    """Every rpca output against the oracle on the same data and Omega:
    eigvals, sdev, rotation, scores x, center, scale, loadings W Lambda^1/2,
    whitened PCs, proportion / cumulative proportion of variance, total
    variance."""
    A = _decay(5000, 240, seed=31) * 3.0 + torch.linspace(-2, 7, 240, dtype=torch.float64)
    An = A.numpy()
    out = rb.rpca(A.cuda(), 18, center=True, scale=scale, p=10, q=2, sdist="unif", seed=8, loadings=True,
                  whiten=True, explained=True)
    o = oracle.oracle_rpca(An, 18, center=True, scale=scale, p=10, q=2, sdist="unif", seed=8)
    rel = lambda a, b: np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))  # noqa: E731
    assert rel(_np(out["eigvals"]), o["eigvals"]) < 2e-10
    assert rel(_np(out["sdev"]), o["sdev"]) < 1e-10
    assert rel(_np(out["var_ratio"]), o["var_ratio"]) < 2e-10
    assert rel(_np(out["var_cum"]), o["var_cum"]) < 2e-10
    assert abs(float(out["total_var"]) - o["total_var"]) < 1e-12 * o["total_var"]
    assert np.abs(_np(out["center"]) - o["center"]).max() < 1e-12
    if scale:
        assert rel(_np(out["scale"]), o["scale"]) < 1e-13
    for key in ("rotation", "loadings", "x", "x_white"):
        got, want = _np(out[key]), o[key]
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-9, key


def test_rpca_default_is_centered_and_scaled(rb):
    """rpca(A, k) defaults to center = TRUE, scale = TRUE."""
    A = _decay(2000, 100, seed=2) + torch.linspace(0, 3, 100, dtype=torch.float64)
    out = rb.rpca(A.cuda(), 8, seed=1)
    assert out["center"] is not None and out["scale"] is not None
    o = oracle.oracle_rpca(A.numpy(), 8, seed=1)
    assert np.max(np.abs(_np(out["eigvals"]) - o["eigvals"]) / o["eigvals"]) < 2e-10


@pytest.mark.parametrize("scale", [False, True])
def test_rpca_predict_vs_oracle(rb, scale):
    """predict() of new rows by the library's pass kernels, against
    the oracle's ((Anew - c) / s) W, and on the training rows of an exact-range
    fit (k = n) it reproduces the scores U Sigma (Eq. PCs)."""
    A = _decay(3000, 64, seed=5) + 1.5
    Anew = _decay(777, 64, seed=6) + 1.5
    fit = rb.rpca(A.cuda(), 12, center=True, scale=scale, p=10, q=2, seed=4)
    got = _np(rb.predict(fit, Anew.cuda()))
    want = oracle.oracle_rpca_predict(Anew.numpy(), _np(fit["rotation"]), _np(fit["center"]),
                                      _np(fit["scale"]) if scale else None)
    assert np.abs(got - want).max() < 1e-12 * np.abs(want).max()
    full = rb.rpca(A.cuda(), 64, center=True, scale=scale, p=0, q=1, seed=4)
    back = _np(rb.predict(full, A.cuda()))
    assert np.abs(back - _np(full["x"])).max() < 1e-10 * np.abs(_np(full["x"])).max()

"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same
seeded inputs.  Tolerances (BASELINE.json north_star):
singular values relative 1e-10 (FP64) / 1e-4 (FP32); reconstruction error
<= 1.0001 x the oracle's + 1e-13 floor (reading R24); ||U^T U - I||_max,
||V^T V - I||_max <= 1e-12 (FP64) / 1e-5 (FP32); Omega bit-exact for
uniform / Rademacher, <= 4 ulp for normal."""
import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

SD = ["normal", "unif", "rademacher"]


@pytest.fixture(scope="module")
def rb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1608_02148_b200 as rb
    return rb


def _np(t):
    return t.detach().cpu().numpy().astype(np.float64)


def _recon_err(A, d, U, V):
    return np.linalg.norm(A - (U * d) @ V.T) / np.linalg.norm(A)


def _cos_cols(X, Y):
    return np.abs(np.sum(X * Y, axis=0)) / (np.linalg.norm(X, axis=0) * np.linalg.norm(Y, axis=0))


def _clusters(dd, gap_tol):
    """Groups of consecutive singular values whose neighbours are closer than
    gap_tol * d_0 (singular vectors defined only up to a rotation inside a
    group, reading R29 / SURVEY c29)."""
    groups, cur = [], [0]
    for i in range(1, len(dd)):
        if abs(dd[i - 1] - dd[i]) <= gap_tol * dd[0]:
            cur.append(i)
        else:
            groups.append(cur)
            cur = [i]
    groups.append(cur)
    return groups


def _sin_max_angle(X, Y):
    """sin of the largest principal angle between span(X) and span(Y) (both
    with orthonormal columns): ||(I - Y Y^T) X||_2."""
    R = X - Y @ (Y.T @ X)
    return float(np.linalg.norm(R, 2)) if R.size else 0.0


def _check_vectors(Vg, Vo, dd, gap_tol, cos_tol, ang_tol):
    """Separated singular vectors column by column (|cos| > 1 - cos_tol, same
    sign, reading R9); clusters of near-equal values by principal angles
    (sin theta_max <= ang_tol); a cluster cut by the last compared column is
    not determined by the first columns alone and is skipped."""
    nv = min(Vg.shape[1], Vo.shape[1], len(dd))
    for grp in _clusters(dd, gap_tol):
        if grp[0] >= nv:
            break
        if len(grp) == 1:
            i = grp[0]
            c = abs(float(Vg[:, i] @ Vo[:, i])) / (np.linalg.norm(Vg[:, i]) * np.linalg.norm(Vo[:, i]))
            assert c > 1 - cos_tol, (i, c)
            assert float(Vg[:, i] @ Vo[:, i]) > 0, ("sign", i)
        elif grp[-1] < nv:
            sa = _sin_max_angle(Vg[:, grp], Vo[:, grp])
            assert sa <= ang_tol, (grp, sa)


def _check_parity(A, r, o, k, tol_d=1e-10, tol_orth=1e-12, floor=1e-13, gap_tol=1e-6, cos_tol=1e-8, ang_tol=1e-8):
    d, U, V = _np(r.d), _np(r.u), _np(r.v)
    assert np.all(np.isfinite(d)) and np.all(np.isfinite(U)) and np.all(np.isfinite(V))
    rel = np.abs(d - o["d"]) / np.maximum(np.abs(o["d"]), 1e-300)
    assert rel.max() <= tol_d, "singular values: max rel err %.3e" % rel.max()
    if U.shape[1]:
        assert np.abs(U.T @ U - np.eye(U.shape[1])).max() <= tol_orth
    if V.shape[1]:
        assert np.abs(V.T @ V - np.eye(V.shape[1])).max() <= tol_orth
    if U.shape[1] == k and V.shape[1] == k:
        e_gpu = _recon_err(A, d, U, V)
        e_or = _recon_err(A, o["d"], o["u"], o["v"])
        assert e_gpu <= 1.0001 * e_or + floor, (e_gpu, e_or)
    # singular vectors: column-wise where separated, principal angles in clusters (R29)
    if V.shape[1]:
        _check_vectors(V, o["v"], o["d"], gap_tol, cos_tol, ang_tol)
    if U.shape[1]:
        _check_vectors(U, o["u"], o["d"], gap_tol, cos_tol, ang_tol)


# ----------------------------------------------------------------------------- Omega (K1)
@pytest.mark.parametrize("sdist", SD)
@pytest.mark.parametrize("n,l", [(1, 1), (777, 13), (5000, 60)])
def test_omega_bits(rb, sdist, n, l):
    seed, stream = 0x0123456789ABCDEF, 0x00000002_00000007
    g = _np(rb.omega(n, l, sdist, seed, stream))
    o = oracle.omega(n, l, sdist, seed, stream)
    if sdist == "normal":
        ulp = np.abs(g - o) / np.spacing(np.maximum(np.abs(o), 1e-300))
        assert ulp.max() <= 4
    else:
        assert np.array_equal(g, o)
    g32 = rb.omega(n, l, sdist, seed, stream, dtype=torch.float32).cpu().numpy()
    o32 = oracle.omega(n, l, sdist, seed, stream, dtype=np.float32)
    if sdist == "normal":
        assert np.abs(g32.astype(np.float64) - o32).max() <= 2 * np.spacing(np.abs(o32).max())
    else:
        assert np.array_equal(g32.astype(np.float64), o32)


# ----------------------------------------------------------------------------- rsvd
def test_config1_exact_rank(rb):
    """Config 1 (J:7): exact rank 10, recovered singular values to 1e-12."""
    A, meta = synthetic.make_config(1)
    An = A.numpy()
    Ad = A.cuda()
    r = rb.rsvd(Ad, 10, p=10, q=2, sdist="normal", seed=meta["seed_omega"])
    s = meta["s"].numpy()
    assert np.max(np.abs(_np(r.d) - s) / s) <= 1e-12
    o = oracle.oracle_rsvd(An, 10, p=10, q=2, sdist="normal", seed=meta["seed_omega"])
    _check_parity(An, r, o, 10)


CASES = [
    # m, n, k, p, q, sdist, nu, nv
    (300, 200, 10, 10, 2, "normal", None, None),
    (1000, 257, 17, 5, 1, "unif", 5, 17),
    (2049, 300, 50, 10, 2, "rademacher", None, None),
    (4000, 1500, 40, 20, 3, "normal", None, 0),
    (173, 531, 12, 8, 2, "normal", None, None),         # wide: works on A^T
    (120, 90, 90, 10, 1, "unif", None, None),           # l = min(m,n): exact SVD
    (5000, 64, 1, 10, 0, "rademacher", None, None),     # k = 1, q = 0
    (3001, 777, 100, 20, 2, "unif", None, None),        # l = 120 (the build limit)
]


def _decay_matrix(m, n, seed, noise=1e-8):
    k = min(m, n)
    s = np.exp(-np.arange(k) / 15.0)
    A, _ = synthetic.lowrank(m, n, torch.as_tensor(s), noise=noise, seed=seed)
    return A


@pytest.mark.parametrize("m,n,k,p,q,sdist,nu,nv", CASES)
def test_rsvd_parity_cases(rb, m, n, k, p, q, sdist, nu, nv):
    A = _decay_matrix(m, n, seed=m + n)
    An = A.numpy()
    r = rb.rsvd(A.cuda(), k, nu=nu, nv=nv, p=p, q=q, sdist=sdist, seed=77, stream=3)
    o = oracle.oracle_rsvd(An, k, nu=nu, nv=nv, p=p, q=q, sdist=sdist, seed=77, stream=3)
    _check_parity(An, r, o, k)


@pytest.mark.parametrize("m,n,k,p,q", [(2, 2, 1, 0, 0), (17, 1, 1, 3, 1), (40, 33, 33, 0, 2),
                                         (33, 40, 5, 100, 1), (1, 9, 1, 2, 0), (129, 128, 120, 0, 1)])
def test_rsvd_tiny_and_degenerate_shapes(rb, m, n, k, p, q):
    """Degenerate shapes: 2 x 2, a single column / row, k = min(m, n) (exact
    SVD), oversampling clamped to min(m, n) (R10), a wide input worked on A^T,
    and l = 120 = k + 0 on a barely tall matrix."""
    g = torch.Generator().manual_seed(m * 131 + n)
    # column scales decay over at most e^-3, so every requested singular value is
    # well above eps * sigma_1 (relative parity is meaningful for all k of them)
    A = torch.randn(m, n, generator=g, dtype=torch.float64) * torch.exp(-torch.arange(n, dtype=torch.float64) / max(7.0, n / 3))
    An = A.numpy()
    r = rb.rsvd(A.cuda(), k, p=p, q=q, seed=2)
    o = oracle.oracle_rsvd(An, k, p=p, q=q, seed=2)
    _check_parity(An, r, o, k, tol_d=1e-10, gap_tol=1e-6, cos_tol=1e-8)


@pytest.mark.parametrize("k", [1, 40])
def test_rid_extreme_k(rb, k):
    """rid with a single column and with k = n (every column is a skeleton
    column: Z is a permutation of I and C Z = A exactly up to rounding)."""
    A = _decay_matrix(500, 40, seed=k + 9, noise=1e-3)
    An = A.numpy()
    r = rb.rid(A.cuda(), k, p=5, q=1, seed=4)
    o = oracle.oracle_rid(An, k, p=5, q=1, seed=4)
    J = r["J"].cpu().numpy()
    assert list(J) == list(o["J"])
    Z = _np(r["Z"])
    assert np.abs(Z - o["Z"]).max() < 1e-9 * max(1.0, np.abs(o["Z"]).max())
    if k == 40:
        assert np.abs(_np(r["C"]) @ Z - An).max() < 1e-12 * np.abs(An).max()


def test_rsvd_unaligned_lda(rb):
    """Odd leading dimension (non-16-byte rows) takes the element-wise staging path."""
    A = _decay_matrix(1001, 301, seed=5)
    big = torch.zeros(1001, 303, dtype=torch.float64)
    big[:, :301] = A
    view = big.cuda()[:, :301]
    r = rb.rsvd(view, 20, p=10, q=2, seed=1)
    o = oracle.oracle_rsvd(A.numpy(), 20, p=10, q=2, seed=1)
    _check_parity(A.numpy(), r, o, 20)


def test_rsvd_fp32(rb):
    A = _decay_matrix(3000, 700, seed=9).to(torch.float32)
    An = A.numpy()
    r = rb.rsvd(A.cuda(), 30, p=10, q=2, seed=4)
    assert r.d.dtype == torch.float32
    o = oracle.oracle_rsvd(An, 30, p=10, q=2, seed=4)
    _check_parity(An.astype(np.float64), r, o, 30, tol_d=1e-4, tol_orth=1e-5, floor=1e-6, cos_tol=1e-5, ang_tol=1e-3,
                  gap_tol=1e-3)


def test_rsvd_rank_deficient_large_panel(rb):
    """Exactly rank-5 input with a panel too tall for one CTA: CholeskyQR2 breaks
    down and the TSQR (Householder leaves) path must take over."""
    A, s = synthetic.lowrank(6000, 400, torch.as_tensor(10.0 ** (-np.arange(5) / 2)), seed=3)
    An = A.numpy()
    r = rb.rsvd(A.cuda(), 5, p=15, q=2, seed=2)
    assert np.max(np.abs(_np(r.d) - s.numpy()) / s.numpy()) <= 1e-11
    o = oracle.oracle_rsvd(An, 5, p=15, q=2, seed=2)
    _check_parity(An, r, o, 5)


@pytest.mark.timeout(300)
def test_rsvd_fallback_many_leaves_and_concurrent(rb):
    """The single-launch TSQR fallback with more leaves than SMs (200000 rows at
    l = 120: ~830 leaves, ~10 levels, grid-stride over the leaves) on an exactly
    rank-12 input, and two contexts on two streams running it at the same time
    (ticket-ordered work items: no wait depends on a CTA that is not running).
    Exact rank 12 < l: the top 12 singular values are the generator's."""
    s = torch.as_tensor(2.0 ** -np.arange(12.0))
    A, _ = synthetic.lowrank(200000, 300, s, seed=21)
    Ad = A.cuda()
    ctxs = [rb.Context(0, torch.cuda.Stream()) for _ in range(2)]
    ref = rb.rsvd(Ad, 100, p=20, q=1, seed=3, ctx=ctxs[0])
    assert ctxs[0].stats()["tsqr_fallback"]
    d = _np(ref.d)
    assert np.max(np.abs(d[:12] - s.numpy()) / s.numpy()) < 1e-11
    u = _np(ref.u)[:, :12]
    assert np.abs(u.T @ u - np.eye(12)).max() < 1e-12
    outs = [rb.rsvd(Ad, 100, p=20, q=1, seed=3, ctx=c, sync=False) for c in ctxs]
    for c in ctxs:
        c.sync()
    for o in outs:
        assert torch.equal(o.d, ref.d) and torch.equal(o.u, ref.u)


def test_rsvd_deterministic(rb):
    A = _decay_matrix(2000, 500, seed=1).cuda()
    r1 = rb.rsvd(A, 20, seed=5)
    r2 = rb.rsvd(A, 20, seed=5)
    assert torch.equal(r1.d, r2.d) and torch.equal(r1.u, r2.u) and torch.equal(r1.v, r2.v)


def test_rsvd_errors(rb):
    A = torch.randn(50, 40, dtype=torch.float64, device="cuda")
    for bad in (0, 41):
        with pytest.raises(rb.RsvdError) as ei:
            rb.rsvd(A, bad)
        assert ei.value.status == 1
    r = rb.rsvd(A, 5, nu=9, nv=9)           # clamped to k with a warning
    assert r.u.shape == (50, 5) and r.v.shape == (40, 5)


def test_config2_full_size(rb):
    """Config 2 (J:8) at full size: 10000 x 5000, k=50, p=10, q=2, Rademacher."""
    A, meta = synthetic.make_config(2)
    An = A.numpy()
    r = rb.rsvd(A.cuda(), 50, p=10, q=2, sdist="rademacher", seed=meta["seed_omega"])
    o = oracle.oracle_rsvd(An, 50, p=10, q=2, sdist="rademacher", seed=meta["seed_omega"])
    _check_parity(An, r, o, 50)


# ----------------------------------------------------------------------------- rqb
def test_rqb_parity(rb):
    A = _decay_matrix(2500, 400, seed=11)
    An = A.numpy()
    Q, B = rb.rqb(A.cuda(), 20, p=10, q=1, sdist="unif", seed=6)
    Qo, Bto = oracle.oracle_rqb(An, 30, 1, "unif", 6)
    Q, B = _np(Q), _np(B)
    assert np.abs(Q.T @ Q - np.eye(30)).max() < 1e-12
    # same projector Q Q^T A (and, for a full-rank sketch, the same Q up to rounding)
    assert np.linalg.norm(Q @ B - Qo @ Bto.T) / np.linalg.norm(An) < 1e-11
    assert np.abs(Q - Qo).max() < 1e-8


# ----------------------------------------------------------------------------- rpca
@pytest.mark.parametrize("scale", [False, True])
def test_rpca_parity(rb, scale):
    A = _decay_matrix(4000, 300, seed=21) + 3.0 * torch.arange(300, dtype=torch.float64)[None, :] / 300
    An = A.numpy()
    out = rb.rpca(A.cuda(), 25, center=True, scale=scale, p=10, q=2, sdist="unif", seed=8)
    o = oracle.oracle_rpca(An, 25, center=True, scale=scale, p=10, q=2, sdist="unif", seed=8)
    ev = _np(out["eigvals"])
    assert np.max(np.abs(ev - o["eigvals"]) / o["eigvals"]) < 1e-10
    assert np.abs(_np(out["center"]) - o["center"]).max() < 1e-13
    if scale:
        assert np.max(np.abs(_np(out["scale"]) - o["scale"]) / o["scale"]) < 1e-13
    c = _cos_cols(_np(out["rotation"]), o["rotation"])
    assert np.all(c > 1 - 1e-8)
    x = _np(out["x"])
    assert np.linalg.norm(x - o["x"]) / np.linalg.norm(o["x"]) < 1e-9


def test_rpca_large_offset_centring(rb):
    """In-tile centring keeps explicit-centring accuracy for large column means
    (offsets 1e2..1e4 x the rms)."""
    A = _decay_matrix(3000, 200, seed=2) * 1e-2 + 1e2
    An = A.numpy()
    out = rb.rpca(A.cuda(), 10, center=True, scale=False, p=10, q=2, seed=3)
    o = oracle.oracle_rpca(An, 10, center=True, scale=False, p=10, q=2, seed=3)
    ev = _np(out["eigvals"])
    assert np.max(np.abs(ev - o["eigvals"]) / o["eigvals"]) < 1e-9


@pytest.mark.parametrize("q", [1, 2])
def test_rsvd_direct_power_scheme_parity(rb, q):
    """Alg. 1 direct power scheme (power="direct") against the
    oracle's Alg. 1 on the same Omega: d within 1e-10 relative, V columns
    parallel, U orthonormal."""
    A = _decay_matrix(3000, 700, seed=41 + q, noise=1e-6)
    An = A.numpy()
    r = rb.rsvd(A.cuda(), 20, p=10, q=q, seed=5, power="direct")
    o = oracle.oracle_rsvd(An, 20, p=10, q=q, seed=5, power="direct")
    d = _np(r.d)
    assert np.max(np.abs(d - o["d"]) / o["d"]) < 1e-10
    c = _cos_cols(_np(r.v), o["v"])
    assert np.all(c[:15] > 1 - 1e-8)
    u = _np(r.u)
    assert np.abs(u.T @ u - np.eye(20)).max() < 1e-12


@pytest.mark.parametrize("m,n,k,p,q", [(3000, 700, 20, 10, 2), (2500, 900, 50, 14, 1)])
def test_rsvd_lu_power_scheme_parity(rb, m, n, k, p, q):
    """Alg. 3 normalized power iterations (power="lu"): GEPP on the
    GPU (cooperative, rows in place) against the oracle's Alg. 3 on the same
    Omega: d within 1e-10 relative, separated V columns parallel."""
    A = _decay_matrix(m, n, seed=m + 2 * k, noise=1e-6)
    An = A.numpy()
    r = rb.rsvd(A.cuda(), k, p=p, q=q, seed=5, power="lu")
    o = oracle.oracle_rsvd(An, k, p=p, q=q, seed=5, power="lu")
    d = _np(r.d)
    assert np.max(np.abs(d - o["d"]) / o["d"]) < 1e-10
    c = _cos_cols(_np(r.v), o["v"])
    assert np.all(c[: k // 2] > 1 - 1e-8)
    u = _np(r.u)
    assert np.abs(u.T @ u - np.eye(k)).max() < 1e-12


def test_rsvd_power_param_rejected(rb):
    A = torch.randn(50, 40, dtype=torch.float64).cuda()
    with pytest.raises(rb.RsvdError):
        rb.rsvd(A, 5, power=3)


@pytest.mark.timeout(300)
def test_rsvd_robust_tsqr_at_l120(rb):
    """CholeskyQR breakdown at the largest sketch width (l = 120): the robust
    Householder TSQR must reduce a 240-row stack of two R factors in one leaf
    (regression: it once looped forever there).  Exact rank 50 < l, so the
    top 50 singular values match the oracle's and U stays orthonormal."""
    g = torch.Generator().manual_seed(8)
    A = (torch.randn(3000, 50, generator=g, dtype=torch.float64) *
         torch.exp(-torch.arange(50, dtype=torch.float64) / 10)) @ torch.randn(50, 500, generator=g, dtype=torch.float64)
    An = A.numpy()
    ctx = rb.Context(0)
    r = rb.rsvd(A.cuda(), 100, p=20, q=1, seed=3, ctx=ctx)
    assert ctx.stats()["tsqr_fallback"]
    o = oracle.oracle_rsvd(An, 100, p=20, q=1, seed=3)
    d = _np(r.d)
    assert np.max(np.abs(d[:50] - o["d"][:50]) / o["d"][:50]) < 1e-10
    u = _np(r.u)[:, :50]
    assert np.abs(u.T @ u - np.eye(50)).max() < 1e-12


# ----------------------------------------------------------------------------- rid / rcur (§8(f) f3)
@pytest.mark.parametrize("m,n,k", [(3000, 500, 20), (2049, 777, 40)])
def test_rid_parity(rb, m, n, k):
    """Alg. rid with Alg. id on B, reading R31:
    the pivot order J equals the oracle's (distinct column norms), C = A(:, J)
    bit-exact, Z within 1e-9 of the oracle's, Z(:, J) = I, and the ID error
    matches the oracle's."""
    A = _decay_matrix(m, n, seed=m + k, noise=1e-6)
    An = A.numpy()
    r = rb.rid(A.cuda(), k, p=10, q=2, seed=7)
    o = oracle.oracle_rid(An, k, p=10, q=2, seed=7)
    J = r["J"].cpu().numpy()
    assert list(J) == list(o["J"])
    C, Z = _np(r["C"]), _np(r["Z"])
    assert np.array_equal(C, An[:, J])
    assert np.abs(Z - o["Z"]).max() < 1e-9 * max(1.0, np.abs(o["Z"]).max())
    assert np.abs(Z[:, J] - np.eye(k)).max() == 0.0
    e_gpu = np.linalg.norm(An - C @ Z) / np.linalg.norm(An)
    e_orc = np.linalg.norm(An - o["C"] @ o["Z"]) / np.linalg.norm(An)
    assert e_gpu <= 1.0001 * e_orc + 1e-13


def test_rid_exact_rank_and_rank_deficiency(rb):
    """Exact rank k: C Z = A to rounding (the ID is exact); asking for more
    columns than the rank is reported as RSVD_ENUMERIC (S(1:k,1:k) singular)."""
    g = torch.Generator().manual_seed(5)
    A = (torch.randn(1500, 12, generator=g, dtype=torch.float64) @
         torch.randn(12, 400, generator=g, dtype=torch.float64))
    r = rb.rid(A.cuda(), 12, p=8, q=1, seed=2)
    C, Z = _np(r["C"]), _np(r["Z"])
    An = A.numpy()
    assert np.abs(C @ Z - An).max() < 1e-11 * np.abs(An).max()
    with pytest.raises(rb.RsvdError):
        rb.rid(A.cuda(), 14, p=8, q=1, seed=2)


@pytest.mark.parametrize("m,n,k", [(2500, 400, 16), (4000, 1000, 30)])
def test_rcur_parity(rb, m, n, k):
    """Alg. rcur: J and I equal the oracle's, C = A(:, J) and
    R = A(I, :) bit-exact, U within 1e-8 relative, and the CUR error matches
    the oracle's."""
    A = _decay_matrix(m, n, seed=3 * m + k, noise=1e-6)
    An = A.numpy()
    r = rb.rcur(A.cuda(), k, p=10, q=2, seed=9)
    o = oracle.oracle_rcur(An, k, p=10, q=2, seed=9)
    J, I = r["J"].cpu().numpy(), r["I"].cpu().numpy()
    assert list(J) == list(o["J"]) and list(I) == list(o["I"])
    C, U, R = _np(r["C"]), _np(r["U"]), _np(r["R"])
    assert np.array_equal(C, An[:, J]) and np.array_equal(R, An[I, :])
    assert np.abs(U - o["U"]).max() < 1e-8 * np.abs(o["U"]).max()
    e_gpu = np.linalg.norm(An - C @ U @ R) / np.linalg.norm(An)
    e_orc = np.linalg.norm(An - o["C"] @ o["U"] @ o["R"]) / np.linalg.norm(An)
    assert e_gpu <= 1.0001 * e_orc + 1e-12


# ----------------------------------------------------------------------------- rrpca
def _rrpca_trajectory(out, o, margin=0.05):
    """Compare the GPU's per-iteration (l, k) of Alg. 7 with the oracle's.
    Returns the first iteration where they differ (None if never).  A
    difference is only accepted where it is ill-posed: every oracle singular
    value between the two counts lies within `margin` of the threshold 1/mu
    (the tail of a randomized SVD is not determined to rounding level, so a
    count can flip there; reading R30)."""
    nt = min(len(out["trace"]), len(o["trace"]))
    for t in range(nt):
        g, w = out["trace"][t], o["trace"][t]
        assert g[3] == w[3], ("target rank differs before any count did", t)
        if g[1] != w[1]:
            thr = 1.0 / w[2]
            lo, hi = sorted((g[1], w[1]))
            band = np.asarray(o["sigmas"][t][lo:hi])
            assert band.size and np.all(np.abs(band - thr) <= margin * thr), (t, g[1], w[1], band, thr)
            return t
    return None


def _rrpca_same_iterations(An, out, kw):
    """An oracle run of exactly the GPU's number of iterations (tol <= 0 never
    stops early), for the L / S comparison when the natural counts differ."""
    kw = dict(kw, maxiter=out["iters"], tol=0.0)
    return oracle.oracle_rrpca(An, **kw)


def _check_rrpca(rb, A, L0=None, S0=None, recover=True, **kw):
    """GPU rrpca vs the oracle on the same A and Omega streams: the rank
    trajectory, the residual trace (1e-6 relative), and L and S within 1e-10
    of an oracle run with the SAME number of iterations (rerun with maxiter =
    the GPU's count when the natural counts differ) whenever the trajectories
    agree; planted components recovered (1e-6, support 0.999)."""
    An = A.numpy()
    out = rb.rrpca(A.cuda(), trace=True, **{key: val for key, val in kw.items() if key != "kmax"})
    okw = {key: val for key, val in kw.items() if key != "rand"}
    o = oracle.oracle_rrpca(An, rand=kw.get("rand", True), **okw)
    div = _rrpca_trajectory(out, o)
    nt = min(out["iters"], o["iters"]) if div is None else div
    for t in range(nt):
        assert abs(out["trace"][t][0] - o["trace"][t][0]) <= 1e-6 * o["trace"][t][0] + 1e-15, t
    L, S = _np(out["L"]), _np(out["S"])
    if div is None:
        ref = o if out["iters"] == o["iters"] else _rrpca_same_iterations(An, out, dict(okw, rand=kw.get("rand", True)))
        assert np.linalg.norm(L - ref["L"]) / np.linalg.norm(ref["L"]) < 1e-10
        assert np.linalg.norm(S - ref["S"]) / np.linalg.norm(ref["S"]) < 1e-10
        assert abs(out["iters"] - o["iters"]) <= 1
    if recover and L0 is not None:
        L0n, S0n = L0.numpy(), S0.numpy()
        assert np.linalg.norm(L - L0n) / np.linalg.norm(L0n) < 1e-6
        assert ((np.abs(S) > 1e-6) == (S0n != 0)).mean() > 0.999
    assert out["residual"] < kw["tol"]
    return out, o, div


def test_rrpca_parity_small(rb):
    A, L0, S0 = synthetic.sparse_plus_lowrank(4000, 300, rank=5, frac=0.05, seed=12)
    _, _, div = _check_rrpca(rb, A, L0, S0, k=10, p=10, q=2, tol=1e-7, maxiter=100, seed=3)
    assert div is None


@pytest.mark.parametrize("m,n,rank,k", [(4000, 300, 5, 0), (3000, 400, 40, 0), (3000, 400, 40, 60)])
def test_rrpca_adaptive_and_large_rank_parity(rb, m, n, rank, k):
    """Alg. 7 with the adaptive target rank of steps (1), (7) (k = 0, R30) and a
    fixed rank above 32 (the R = 64 update kernel): the rank trajectory (l, k)
    per iteration matches the oracle's (a count may differ only where the
    oracle's values sit at 1/mu), L and S within 1e-10 of the oracle at the
    same iteration count, and the planted L0, S0 are recovered."""
    A, L0, S0 = synthetic.sparse_plus_lowrank(m, n, rank=rank, frac=0.05, seed=rank + 11)
    out, o, div = _check_rrpca(rb, A, L0, S0, k=k, p=10, q=2, tol=1e-7, maxiter=100, seed=4, kmax=min(m, n, 110))
    assert all(t[3] <= min(m, n) / 4 for t in o["trace"])          # no Remark-2 switch on either side
    if k == 0:
        assert out["trace"][0][3] == 2 and out["trace"][-1][3] == rank + 1
        assert div is None


@pytest.mark.parametrize("rank,k,rand", [(5, 10, False), (32, 0, True)])
def test_rrpca_deterministic_svd(rb, rank, k, rand):
    """rand = FALSE and Remark 2's switch (adaptive k >
    min(m, n)/4 -> deterministic SVD): the GPU's deterministic SVD (rsvd with
    l = min(m, n), q = 0) against the oracle's numpy SVD, same rank trajectory,
    L and S within 1e-10 at the same iteration count; the rank-5 case also
    recovers the planted L0 (rank 32 of 120 is beyond exact recovery)."""
    A, L0, S0 = synthetic.sparse_plus_lowrank(3000, 120, rank=rank, frac=0.05, seed=rank + 100)
    out, o, div = _check_rrpca(rb, A, L0, S0, recover=rank == 5, k=k, p=10, q=2, tol=1e-7, maxiter=100, seed=4,
                               rand=rand)
    if k == 0:
        assert any(t[3] > 120 / 4 for t in o["trace"])               # the switch is exercised
    assert div is None


# ----------------------------------------------------------------------------- full-size configs 3, 5
def test_config3_full_size_rpca(rb):
    """Config 3 (J:9): 200000 x 4000 column-centred PCA (scale = FALSE, reading
    R15), k=100, p=20, q=2, uniform Omega: eigenvalues (2e-10, the d^2 of the
    1e-10 d tolerance), column means, rotation and scores x = U Sigma
    (Alg. 6 step (3)) column-wise where separated and by principal angles in
    clusters, orthonormality, and the centred reconstruction error within
    1.0001 x the oracle's (computed in row chunks on the device)."""
    A, meta = synthetic.make_config(3)
    Ad = A.cuda()
    out = rb.rpca(Ad, 100, center=True, scale=False, p=20, q=2, sdist="unif", seed=meta["seed_omega"])
    An = A.numpy()
    o = oracle.oracle_rpca(An, 100, center=True, scale=False, p=20, q=2, sdist="unif", seed=meta["seed_omega"])
    ev = _np(out["eigvals"])
    assert np.max(np.abs(ev - o["eigvals"]) / o["eigvals"]) < 2e-10
    assert np.abs(_np(out["center"]) - o["center"]).max() < 1e-12
    rot, x = _np(out["rotation"]), _np(out["x"])
    assert np.abs(rot.T @ rot - np.eye(100)).max() < 1e-12
    d = np.sqrt(o["eigvals"] * (An.shape[0] - 1))
    _check_vectors(rot, o["rotation"], d, 1e-6, 1e-8, 1e-8)
    U, Uo = x / d[None, :], o["x"] / d[None, :]
    assert np.abs(U.T @ U - np.eye(100)).max() < 1e-11
    _check_vectors(U, Uo, d, 1e-6, 1e-8, 1e-8)
    # centred reconstruction error ||X - x W^T||_F / ||X||_F, X = A - 1 c^T
    c = torch.as_tensor(o["center"], device="cuda")
    xg, rg = out["x"], out["rotation"]
    xo, ro = torch.as_tensor(o["x"], device="cuda"), torch.as_tensor(o["rotation"], device="cuda")
    num_g = num_o = den = 0.0
    for r0 in range(0, A.shape[0], 20000):
        X = Ad[r0:r0 + 20000] - c[None, :]
        den += float((X * X).sum())
        num_g += float(((X - xg[r0:r0 + 20000] @ rg.T) ** 2).sum())
        num_o += float(((X - xo[r0:r0 + 20000] @ ro.T) ** 2).sum())
    eg, eo = np.sqrt(num_g / den), np.sqrt(num_o / den)
    assert eg <= 1.0001 * eo + 1e-13, (eg, eo)


@pytest.mark.timeout(1200)
def test_config4_full_size_properties(rb):
    """Config 4 (J:10) at full size -- 10^6 x 10^4 FP32 (40 GB), k = 100,
    p = 20, q = 3, Gaussian Omega, the launch configuration bench.py times --
    checked on properties that hold at any size (the oracle cannot run it).
    B^T = A^T Q, so A^T u_i = d_i v_i (Alg. 5 / Eq. UQU) up to the FP32
    accumulation of the pass over 10^6 rows (R12): for sampled i the FP64
    matvec w = A^T u_i (chunked, on the device) gives ||w|| = d_i within the
    J:5 FP32 tolerance 1e-4 and a direction within 1e-4 of v_i; the vector
    residual ||w - d_i v_i|| / d_i stays below 1e-2 (FP32 sums of 10^6
    products).  U, V orthonormal to 1e-5; d descending."""
    A, meta = synthetic.make_config(4, device="cuda")
    r = rb.rsvd(A, 100, p=20, q=3, sdist=meta["sdist"], seed=meta["seed_omega"])
    d = r.d.double()
    assert bool(torch.all(d[:-1] >= d[1:]))
    U, V = r.u, r.v
    eye = torch.eye(100, dtype=torch.float64, device="cuda")
    assert float((U.double().T @ U.double() - eye).abs().max()) < 1e-5
    assert float((V.double().T @ V.double() - eye).abs().max()) < 1e-5
    idx = [0, 1, 10, 50, 99]
    W = torch.zeros(A.shape[1], len(idx), dtype=torch.float64, device="cuda")
    Us = U[:, idx].double()
    for r0 in range(0, A.shape[0], 100000):
        W += A[r0:r0 + 100000].double().T @ Us[r0:r0 + 100000]
    for j, i in enumerate(idx):
        w, v = W[:, j], V[:, i].double()
        nw = float(torch.linalg.norm(w))
        assert abs(nw - float(d[i])) / float(d[i]) < 1e-4, (i, nw, float(d[i]))
        assert 1.0 - float(w @ v) / nw < 1e-4, (i, float(w @ v) / nw)
        assert float(torch.linalg.norm(w - d[i] * v)) / float(d[i]) < 1e-2
    del A


@pytest.mark.timeout(1800)
def test_config4_full_size_vs_oracle(rb):
    """Config 4 (J:10) at full size against the oracle's FP64 rsvd of the same
    FP32 A (tests/golden/cfg4_oracle.npz, written on the GPU box's host by
    tools/make_cfg4_golden.py, which calls only oracle/ and synthetic/):
    d within the FP32 tolerance 1e-4 (J:5), V column-wise / by principal
    angles within 1e-3 (reading R29 FP32), U and V orthonormal to 1e-5, and
    the reconstruction error (row chunks, FP64, on the device) within
    1.0001 x the oracle's + 1e-6 (R24)."""
    import os
    gold = os.path.join(os.path.dirname(__file__), "golden", "cfg4_oracle.npz")
    g = np.load(gold)
    A, meta = synthetic.make_config(4, device="cuda")
    r = rb.rsvd(A, 100, p=20, q=3, sdist=meta["sdist"], seed=meta["seed_omega"])
    d, V = _np(r.d), _np(r.v)
    assert np.max(np.abs(d - g["d"]) / g["d"]) <= 1e-4
    _check_vectors(V, g["v"], g["d"], 1e-3, 1e-4, 1e-3)
    eye = torch.eye(100, dtype=torch.float64, device="cuda")
    Ud = r.u.double()
    assert float((Ud.T @ Ud - eye).abs().max()) < 1e-5
    assert np.abs(V.T @ V - np.eye(100)).max() < 1e-5
    ur = g["u_rows"]                                   # the oracle's first 2000 rows of U
    ug = _np(r.u[:ur.shape[0]])
    for grp in _clusters(g["d"], 1e-3):               # separated columns: same direction and sign
        if len(grp) == 1:
            i = grp[0]
            c = float(ug[:, i] @ ur[:, i]) / (np.linalg.norm(ug[:, i]) * np.linalg.norm(ur[:, i]))
            assert c > 1 - 1e-2, (i, c)
    num = den = 0.0
    Vd, dd = r.v.double(), r.d.double()
    for r0 in range(0, A.shape[0], 50000):
        X = A[r0:r0 + 50000].double()
        den += float((X * X).sum())
        num += float(((X - (Ud[r0:r0 + 50000] * dd[None, :]) @ Vd.T) ** 2).sum())
    err = np.sqrt(num / den)
    assert err <= 1.0001 * float(g["recon_err"]) + 1e-6, (err, float(g["recon_err"]))
    del A


def test_config5_full_size_rrpca(rb):
    """Config 5 (J:11): 100000 x 1000 robust PCA by IALM, rsvd(k=20, p=10, q=2),
    tol 1e-7: the residual trace of every iteration, L and S against the oracle
    run of the SAME number of iterations (unconditionally: an oracle rerun
    with maxiter = the GPU's count when the natural counts differ), and the
    planted L0, S0 (ground truth, R21 / SURVEY X5)."""
    A, meta = synthetic.make_config(5)
    out, o, div = _check_rrpca(rb, A, meta["L0"], meta["S0"], k=20, p=10, q=2, tol=1e-7, maxiter=100,
                               seed=meta["seed_omega"])
    assert div is None                       # fixed rank 20 of a rank-20 signal: no borderline counts


# ----------------------------------------------------------------------------- FP32 on tcgen05
def _ctx_fp32_path(rb, path):
    import os
    old = os.environ.get("RSVD_FP32_PATH")
    os.environ["RSVD_FP32_PATH"] = path
    try:
        return rb.Context(0)
    finally:
        if old is None:
            del os.environ["RSVD_FP32_PATH"]
        else:
            os.environ["RSVD_FP32_PATH"] = old


@pytest.mark.parametrize("path", ["ozaki", "tf32"])
@pytest.mark.parametrize("m,n,k,p,q", [(3000, 700, 30, 10, 2), (5000, 1200, 100, 20, 3), (777, 2000, 20, 12, 1),
                                       (4099, 1030, 50, 14, 2), (4900, 1030, 100, 20, 2), (1100, 3000, 100, 20, 1)])
def test_rsvd_fp32_tcgen05_parity(rb, m, n, k, p, q, path):
    """FP32 A through the tcgen05 passes -- 3-digit Ozaki int8 slices (default)
    or 3xTF32 (RSVD_FP32_PATH=tf32): singular values within 1e-4 of the FP64
    oracle on the same FP32 data (J:5), orthonormality 1e-5.  (4099, 1030):
    ragged row block and a row length that is not a multiple of 4 (the
    warp-per-row slicer).  l = 120 runs the row-pair (cta_group::2) kernel:
    (4900, 1030) has 39 row blocks of A.X (the last pair's second CTA entirely
    out of range) and 9 of A^T.X; (1100, 3000) is wide (the roles swapped)."""
    A = _decay_matrix(m, n, seed=m + 3 * n, noise=1e-5).to(torch.float32)
    An = A.numpy()
    ctx = _ctx_fp32_path(rb, path)
    r = rb.rsvd(A.cuda(), k, p=p, q=q, seed=12, ctx=ctx)
    assert (ctx.stats()["ozaki_passes"] > 0) == (path == "ozaki")
    o = oracle.oracle_rsvd(An, k, p=p, q=q, seed=12)
    _check_parity(An.astype(np.float64), r, o, k, tol_d=1e-4, tol_orth=1e-5, floor=1e-6, gap_tol=1e-3, cos_tol=1e-5,
                  ang_tol=1e-3)


def test_rsvd_fp32_ozaki_matches_fp64(rb):
    """The 3-digit slices of FP32 A keep 24 bits per element relative to its
    row maximum and the X panel 22 bits: the FP32 run agrees with the FP64
    Ozaki run on the exactly upcast matrix to ~1e-6 (far inside J:5's 1e-4),
    including rows spanning four decades."""
    A = _decay_matrix(2600, 900, seed=77, noise=1e-5).numpy()
    A = A * (10.0 ** np.random.default_rng(3).uniform(-4, 0, size=(A.shape[0], 1)))
    A32 = torch.from_numpy(A).to(torch.float32)
    r32 = rb.rsvd(A32.cuda(), 40, p=10, q=2, seed=5)
    r64 = rb.rsvd(A32.double().cuda(), 40, p=10, q=2, seed=5)
    d32, d64 = _np(r32.d).astype(np.float64), _np(r64.d)
    assert np.max(np.abs(d32 - d64) / d64) < 2e-6


def test_rsvd_fp32_ozaki_top_binade(rb):
    """Elements within half a unit below the row's power of two (|a| = 2^E (1 -
    2^-24)) round to 2^23 at 24 bits: the slicer clamps instead of wrapping
    the two's-complement top digit.  Rows of +-0.99999994 * 2^e_r plus a
    rank-3 signal; d within 1e-4 of the oracle."""
    rng = np.random.default_rng(11)
    m, n = 2048, 768
    top = np.float32(1.0) - np.float32(2.0 ** -24)
    A = np.where(rng.random((m, n)) < 0.5, -top, top).astype(np.float32)
    A *= (2.0 ** rng.integers(-3, 4, size=(m, 1))).astype(np.float32)
    A[:, :3] *= np.float32(0.5)
    r = rb.rsvd(torch.from_numpy(A).cuda(), 10, p=10, q=1, seed=2)
    o = oracle.oracle_rsvd(A.astype(np.float64), 10, p=10, q=1, seed=2)
    assert np.max(np.abs(_np(r.d).astype(np.float64) - o["d"]) / o["d"]) < 1e-4


def test_rpca_fp32_centred_ozaki(rb):
    """FP32 rpca: the centring / scaling is applied in FP64 to the upcast FP32
    elements inside the 3-digit slicer; eigenvalues within 1e-4 of the oracle."""
    A = (_decay_matrix(3000, 500, seed=8, noise=1e-4).numpy() + 3.0).astype(np.float32)
    for scale in (False, True):
        r = rb.rpca(torch.from_numpy(A).cuda(), 20, center=True, scale=scale, p=10, q=2, seed=3)
        o = oracle.oracle_rpca(A.astype(np.float64), 20, center=True, scale=scale, p=10, q=2, seed=3)
        ev, eo = _np(r["eigvals"]).astype(np.float64), o["eigvals"]
        assert np.max(np.abs(ev - eo) / eo) < 1e-4


# ----------------------------------------------------------------------------- FP64 pass paths
def _ctx_with_path(rb, path):
    import os
    old = os.environ.get("RSVD_FP64_PATH")
    os.environ["RSVD_FP64_PATH"] = path
    try:
        return rb.Context(0)
    finally:
        if old is None:
            del os.environ["RSVD_FP64_PATH"]
        else:
            os.environ["RSVD_FP64_PATH"] = old


@pytest.mark.parametrize("m,n,k,p", [(3000, 1100, 50, 10), (2500, 900, 100, 20)])
def test_ozaki_and_dmma_paths_agree(rb, m, n, k, p):
    """The Ozaki int8 tensor-core passes and the FP64 DMMA passes compute the
    same products to FP64 accuracy: both match the oracle and each other."""
    A = _decay_matrix(m, n, seed=21)
    Ad = A.cuda()
    c_oz, c_dm = _ctx_with_path(rb, "ozaki"), _ctx_with_path(rb, "dmma")
    r_oz = rb.rsvd(Ad, k, p=p, q=2, seed=4, ctx=c_oz)
    r_dm = rb.rsvd(Ad, k, p=p, q=2, seed=4, ctx=c_dm)
    assert c_oz.stats()["ozaki_passes"] > 0 and c_dm.stats()["ozaki_passes"] == 0
    d_oz, d_dm = _np(r_oz.d), _np(r_dm.d)
    assert np.max(np.abs(d_oz - d_dm) / d_dm) <= 1e-11
    o = oracle.oracle_rsvd(A.numpy(), k, p=p, q=2, seed=4)
    _check_parity(A.numpy(), r_oz, o, k)
    _check_parity(A.numpy(), r_dm, o, k)


def test_rsvd_heterogeneous_row_scales(rb):
    """Rows spanning six decades inside one exponent super-tile of the Ozaki
    slices (the exponent is shared by 1024 x 1024 elements): parity holds."""
    A = _decay_matrix(2200, 800, seed=33).numpy()
    rng = np.random.default_rng(7)
    A = A * (10.0 ** rng.uniform(-6, 0, size=(A.shape[0], 1)))
    r = rb.rsvd(torch.from_numpy(A).cuda(), 30, p=10, q=2, seed=9)
    o = oracle.oracle_rsvd(A, 30, p=10, q=2, seed=9)
    _check_parity(A, r, o, 30)


@pytest.mark.parametrize("e", [-450, 450])
def test_rsvd_power_of_two_scaling(rb, e):
    """ADVICE r1 (Ozaki exponent range): A scaled by 2^e far from 1.  Every step
    is equivariant under a power-of-two scaling (the slices keep their digits,
    the row exponents shift; Gram and Cholesky factors scale exactly while no
    value leaves the normal range), so d(2^e A) = 2^e d(A) and U, V are the same
    -- checked to 1e-14, and 2^-e d against the oracle on A to 1e-10.  (|A| beyond about
    2^±500 squares out of range in the Gram of CholeskyQR: DESIGN.md R35.)"""
    A = _decay_matrix(3000, 700, seed=31)
    r0 = rb.rsvd(A.cuda(), 40, p=10, q=2, seed=5)
    As = A * (2.0 ** e)
    r1 = rb.rsvd(As.cuda(), 40, p=10, q=2, seed=5)
    d0, d1 = _np(r0.d), _np(r1.d)
    assert np.max(np.abs(d1 * 2.0 ** -e - d0) / d0) < 1e-14
    assert np.abs(_np(r1.v) - _np(r0.v)).max() < 1e-12
    assert np.abs(_np(r1.u) - _np(r0.u)).max() < 1e-12
    # the oracle's Jacobi test squares alpha * beta too (it is written for data near
    # unit scale): it runs on the unscaled A, and 2^e d(A) is the scaled answer
    o = oracle.oracle_rsvd(A.numpy(), 40, p=10, q=2, seed=5)
    assert np.max(np.abs(d1 * 2.0 ** -e - o["d"]) / o["d"]) < 1e-10


def test_rsvd_repeated_calls_bitwise(rb):
    """Race check by repetition (compute-sanitizer is closed on the GPU pool):
    200 config-2 calls (Np = 64 stream-K passes with fix-up flags, the Jacobi
    rotation log replayed by other CTAs) and 100 calls at l = 120 (2-CTA paired
    passes) enqueued back to back with no host synchronisation; every result
    must equal the first call's bit for bit (tools/stress_determinism.py runs
    the longer version over every kernel family)."""
    A, meta = synthetic.make_config(2)
    Ad = A.cuda()
    for k, p, q, n_rep in ((50, 10, 2, 200), (100, 20, 1, 100)):
        ref = rb.rsvd(Ad, k, p=p, q=q, sdist="rademacher", seed=meta["seed_omega"])
        ref = [t.clone() for t in ref]
        bad = torch.zeros((), dtype=torch.int64, device="cuda")
        for _ in range(n_rep):
            r = rb.rsvd(Ad, k, p=p, q=q, sdist="rademacher", seed=meta["seed_omega"], sync=False)
            for a, b in zip(r, ref):
                bad += (a != b).sum()
        torch.cuda.synchronize()
        assert int(bad.item()) == 0

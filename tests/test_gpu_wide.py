"""GPU parity of wide plans, l = k + p > 120 (reading R34 of DESIGN.md): the
DMMA column-block passes, CholeskyQR2 with the cooperative Cholesky
(wide.cu chol_wide_kernel) and the round-robin Jacobi (jacobi_wide_kernel)
against the CPU oracle on the same seeded inputs, with the tolerances of
test_gpu_parity.py (singular values 1e-10 relative, orthonormality 1e-12,
reconstruction <= 1.0001 x the oracle's).  The interface allows any
k <= min(m, n) (Alg. 4 input P:590); rrpca's Remark 2
switches to the deterministic SVD at k > min(m, n)/4 whatever min(m, n) is."""
import numpy as np
import pytest
import torch

import oracle
import synthetic
from test_gpu_parity import _check_parity, _check_rrpca, _check_vectors, _np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1608_02148_b200 as rb
    return rb


def _slow_decay(m, n, seed, tau=100.0, noise=1e-8):
    s = np.exp(-np.arange(min(m, n)) / tau)
    A, _ = synthetic.lowrank(m, n, torch.as_tensor(s), noise=noise, seed=seed)
    return A


WIDE = [
    # m, n, k, p, q, sdist
    (2000, 600, 150, 20, 2, "normal"),       # l = 170: one full and one partial column block
    (3000, 1000, 240, 16, 1, "unif"),        # l = 256: two full column blocks
    (400, 1500, 130, 10, 1, "rademacher"),   # wide input: worked on A^T, l = 140
    (700, 300, 300, 0, 0, "normal"),         # l = k = min(m, n): the exact SVD (Jacobi at l = 300)
    (1500, 257, 200, 57, 2, "unif"),         # l = 257 = min(m, n) (odd: a bye in every Jacobi round)
]


@pytest.mark.parametrize("m,n,k,p,q,sdist", WIDE)
def test_rsvd_wide_parity(rb, m, n, k, p, q, sdist):
    A = _slow_decay(m, n, seed=m + 3 * n)
    An = A.numpy()
    r = rb.rsvd(A.cuda(), k, p=p, q=q, sdist=sdist, seed=91, stream=2)
    o = oracle.oracle_rsvd(An, k, p=p, q=q, sdist=sdist, seed=91, stream=2)
    _check_parity(An, r, o, k)


def test_rsvd_wide_exact_svd_vs_lapack(rb):
    """k = min(m, n), p = q = 0 on a well-conditioned square-ish input: Q Q^T A = A,
    so the result is the exact SVD (SURVEY §8(c) special case (ii)) -- checked
    against numpy's LAPACK SVD directly, not only against the oracle."""
    g = torch.Generator().manual_seed(5)
    A = torch.randn(600, 200, generator=g, dtype=torch.float64)
    r = rb.rsvd(A.cuda(), 200, p=0, q=0, seed=1)
    s = np.linalg.svd(A.numpy(), compute_uv=False)
    assert np.max(np.abs(_np(r.d) - s) / s) < 1e-12
    U, V = _np(r.u), _np(r.v)
    assert np.abs(U.T @ U - np.eye(200)).max() < 1e-12
    assert np.abs(V.T @ V - np.eye(200)).max() < 1e-12
    assert np.linalg.norm(A.numpy() - (U * _np(r.d)) @ V.T) / np.linalg.norm(A.numpy()) < 1e-13


def test_rsvd_wide_fp32(rb):
    """FP32 A in a wide plan (DMMA column blocks on the FP32 rows, FP64 panels):
    singular values within the FP32 tolerance 1e-4 of the FP64 oracle on the
    same FP32 input and FP32-rounded Omega (reading R12)."""
    A = _slow_decay(2500, 800, seed=17).float()
    r = rb.rsvd(A.cuda(), 140, p=20, q=2, seed=3)
    o = oracle.oracle_rsvd(A.numpy(), 140, p=20, q=2, seed=3)
    d = _np(r.d)
    assert np.max(np.abs(d - o["d"]) / o["d"]) < 1e-4
    U, V = _np(r.u), _np(r.v)
    assert np.abs(U.T @ U - np.eye(140)).max() < 1e-5
    assert np.abs(V.T @ V - np.eye(140)).max() < 1e-5


def test_rpca_wide(rb):
    """rpca (centre + scale, Alg. 6) at k = 150, l = 170: eigenvalues, rotation and
    scores against the oracle."""
    A = _slow_decay(3000, 400, seed=8, noise=1e-6) + 3.0
    An = A.numpy()
    out = rb.rpca(A.cuda(), 150, center=True, scale=True, p=20, q=2, seed=6)
    o = oracle.oracle_rpca(An, 150, center=True, scale=True, p=20, q=2, seed=6)
    ev = _np(out["eigvals"])
    assert np.max(np.abs(ev - o["eigvals"]) / o["eigvals"]) < 2e-10
    d = np.sqrt(o["eigvals"] * (An.shape[0] - 1))
    _check_vectors(_np(out["rotation"]), o["rotation"], d, 1e-6, 1e-8, 1e-8)
    _check_vectors(_np(out["x"]) / d[None, :], o["x"] / d[None, :], d, 1e-6, 1e-8, 1e-8)


def test_rsvd_wide_rank_deficient(rb):
    """An exactly rank-10 input with l = 160: the sketch is rank-deficient to
    working precision, the CholeskyQR of the wide plan breaks down and the
    device-side Householder fallback (wide.cu hqr_wide_kernel, reading R34)
    orthonormalises the panel: the 10 planted singular values to 1e-12 and
    against the oracle, the rest at rounding level, U and V orthonormal over
    all 150 columns, and the fallback reported in the context's stats."""
    s = 10.0 ** (-np.arange(10) / 5.0)
    A, _ = synthetic.lowrank(1000, 400, torch.as_tensor(s), seed=2)
    ctx = rb.Context()
    r = rb.rsvd(A.cuda(), 150, p=10, q=1, seed=1, ctx=ctx)
    d, U, V = _np(r.d), _np(r.u), _np(r.v)
    assert np.max(np.abs(d[:10] - s) / s) < 1e-12
    assert d[10:].max() < 1e-13
    assert np.abs(U.T @ U - np.eye(150)).max() < 1e-12
    assert np.abs(V.T @ V - np.eye(150)).max() < 1e-12
    assert ctx.stats()["tsqr_fallback"]
    o = oracle.oracle_rsvd(A.numpy(), 150, p=10, q=1, seed=1)
    assert np.max(np.abs(d[:10] - o["d"][:10]) / o["d"][:10]) < 1e-10
    assert np.linalg.norm(A.numpy() - (U * d) @ V.T) / np.linalg.norm(A.numpy()) < 1e-13


def test_rrpca_remark2_switch_above_120(rb):
    """adaptive rank with 120 < min(m, n) < 440 whose rank crosses
    min(m, n)/4: the deterministic SVD (l = min(m, n) = 200, a wide plan) runs
    instead of failing or capping k; trajectory, L and S against the oracle."""
    A, L0, S0 = synthetic.sparse_plus_lowrank(3000, 200, rank=60, frac=0.05, seed=71)
    out, o, div = _check_rrpca(rb, A, L0, S0, recover=False, k=0, p=10, q=2, tol=1e-7, maxiter=100, seed=4)
    assert any(t[3] > 200 / 4 for t in o["trace"])                  # the switch is exercised
    assert div is None


def test_rrpca_rank_above_128_dense_update(rb):
    """rand = FALSE at k = 150 on a 2500 x 300 input: the deterministic SVD at
    l = 300 and the IALM update with L materialised by gemm_pass (rank > 128,
    wide.cu ialm_dense_kernel) against the oracle."""
    A, L0, S0 = synthetic.sparse_plus_lowrank(2500, 300, rank=150, frac=0.05, seed=72)
    _, _, div = _check_rrpca(rb, A, L0, S0, recover=False, k=150, p=10, q=2, tol=1e-7, maxiter=100, seed=4,
                             rand=False)
    assert div is None


def test_wide_lu_power_scheme_rejected_before_launch(rb):
    """Alg. 3's cooperative GEPP is limited to l <= 128: a wide Alg. 3 request is
    refused with RSVD_EUNSUPPORTED before any launch (not a CUDA error mid-call);
    the context stays usable."""
    A = _slow_decay(600, 300, seed=3)
    with pytest.raises(rb.RsvdError) as ei:
        rb.rsvd(A.cuda(), 150, p=10, q=1, seed=1, power="lu")
    assert ei.value.status == 6
    r = rb.rsvd(A.cuda(), 20, p=10, q=1, seed=1)
    assert np.all(np.isfinite(_np(r.d)))

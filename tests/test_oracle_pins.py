"""Pins for the CPU oracle (oracle/), checked against things other than itself:
worked examples (tests/golden/), closed forms, textbook special cases, an
independent Philox (cuRAND, host-compiled), numpy/LAPACK on tiny inputs and
brute force.  CPU only."""
import json
import math
import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle
from oracle.linalg import hqr, jacobi_svd_bt, soft_threshold
from oracle.philox import omega, omega_words, philox4x32_10
from oracle.rsvd import oracle_rpca_predict
from oracle.rsvd import oracle_rpca, oracle_rqb, oracle_rrpca, oracle_rsvd, predict_rank, resolve_params

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "worked_examples.json")))


def error_bound_factor(k, p, q, m, n):
    """Expected-error bound factor, PAPER.md:665-669 (§3.4):
    [1 + sqrt(k/(p-1)) + e sqrt(k+p)/p * sqrt(min(m,n)-k)]^(1/(2q+1))."""
    t = 1.0 + math.sqrt(k / (p - 1)) + math.e * math.sqrt(k + p) / p * math.sqrt(min(m, n) - k)
    return t ** (1.0 / (2 * q + 1))


# ----------------------------------------------------------------------------- Philox / Omega
@pytest.fixture(scope="module")
def curand_kat(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available for the cuRAND host KAT")
    out = str(tmp_path_factory.mktemp("kat") / "philox_kat")
    src = os.path.join(os.path.dirname(HERE), "tools", "philox_kat.cu")
    subprocess.check_call([nvcc, "-o", out, src], stderr=subprocess.DEVNULL)

    def run(rows):
        txt = "\n".join(" ".join("%08x" % v for v in r) for r in rows) + "\n"
        res = subprocess.run([out], input=txt, capture_output=True, text=True, check=True)
        return [[int(w, 16) for w in line.split()] for line in res.stdout.strip().splitlines()]
    return run


def test_philox_golden_kat():
    for case in GOLD["philox_kat"]["cases"]:
        c = [np.array([int(x, 16)], dtype=np.uint32) for x in case["c"]]
        k = [int(x, 16) for x in case["k"]]
        w = philox4x32_10(*c, *k)
        assert [int(x[0]) for x in w] == [int(x, 16) for x in case["w"]]


def test_philox_matches_curand_random(curand_kat):
    rng = np.random.default_rng(7)
    rows = rng.integers(0, 2 ** 32, size=(200, 6), dtype=np.uint64).astype(np.uint32)
    ref = np.array(curand_kat(rows.tolist()), dtype=np.uint64)
    for r in range(rows.shape[0]):
        w = philox4x32_10(*[rows[r:r + 1, i] for i in range(4)], int(rows[r, 4]), int(rows[r, 5]))
        assert [int(x[0]) for x in w] == [int(v) for v in ref[r]]


def test_omega_counter_mapping_matches_curand(curand_kat):
    """Entry (i, j) uses counter (lo(e), hi(e), lo(stream), hi(stream)), e = j*n+i,
    key (lo(seed), hi(seed)); a = w1<<32|w0, b = w3<<32|w2 (reading R1)."""
    n, l = 37, 5
    seed = 0x123456789ABCDEF0
    stream = 0x0000000500000003
    a, b = omega_words(n, l, seed, stream)
    rows = []
    idx = [(0, 0), (36, 0), (0, 4), (17, 3), (36, 4)]
    for i, j in idx:
        e = j * n + i
        rows.append([e & 0xFFFFFFFF, e >> 32, stream & 0xFFFFFFFF, stream >> 32,
                     seed & 0xFFFFFFFF, seed >> 32])
    ref = curand_kat(rows)
    for (i, j), w in zip(idx, ref):
        assert int(a[i, j]) == (w[1] << 32) | w[0]
        assert int(b[i, j]) == (w[3] << 32) | w[2]


def test_omega_distributions():
    n, l = 20000, 5     # 1e5 samples: mean within 0.02, variance within 0.03 (S:212, 5 sigma)
    g = omega(n, l, "normal", seed=11, stream=0).ravel()
    assert abs(g.mean()) < 0.02 and abs(g.var() - 1.0) < 0.03
    from scipy import stats
    # Kolmogorov-Smirnov against N(0,1) (library CDF): catches a wrong Box-Muller factor.
    assert stats.kstest(g, "norm").pvalue > 1e-4
    u = omega(n, l, "unif", seed=11, stream=0).ravel()
    assert u.min() > -1.0 and u.max() < 1.0
    assert abs(u.mean()) < 0.01 and abs(u.var() - 1.0 / 3.0) < 0.01
    assert stats.kstest(u, "uniform", args=(-1, 2)).pvalue > 1e-4
    r = omega(n, l, "rademacher", seed=11, stream=0).ravel()
    assert set(np.unique(r).tolist()) == {-1.0, 1.0}      # P:429 "+1 and -1"
    assert abs(r.mean()) < 0.02
    # distinct streams / seeds give different matrices; same inputs identical
    assert not np.array_equal(omega(50, 3, "normal", 1, 0), omega(50, 3, "normal", 1, 1))
    assert not np.array_equal(omega(50, 3, "normal", 1, 0), omega(50, 3, "normal", 2, 0))
    assert np.array_equal(omega(50, 3, "normal", 1, 0), omega(50, 3, "normal", 1, 0))
    # nested sketches share leading columns (column-major counter)
    assert np.array_equal(omega(50, 3, "unif", 4, 0), omega(50, 6, "unif", 4, 0)[:, :3])


def test_omega_fp32_rounding():
    g64 = omega(100, 4, "normal", 3, 0)
    g32 = omega(100, 4, "normal", 3, 0, dtype=np.float32)
    assert np.array_equal(g32, g64.astype(np.float32).astype(np.float64))


def test_gaussian_test_matrix_full_rank():
    """'random vectors are linearly independent with high probability'."""
    for s in range(20):
        Om = omega(200, 20, "normal", seed=s)
        assert np.linalg.svd(Om, compute_uv=False).min() > 1e-3


# ----------------------------------------------------------------------------- Householder QR
def test_hqr_worked_examples():
    ex = GOLD["qr_column_3_4"]
    Q, R = hqr(np.array(ex["Y"]))
    assert np.allclose(Q, ex["Q"], atol=1e-15, rtol=0) and np.allclose(R, ex["R"], atol=1e-15, rtol=0)
    Q, R = hqr(np.array(GOLD["qr_identity"]["Y"], dtype=float))
    assert np.allclose(Q, np.eye(3), atol=1e-15) and np.allclose(R, np.eye(3), atol=1e-15)


@pytest.mark.parametrize("m,l", [(50, 8), (200, 20), (61, 61), (300, 1)])
def test_hqr_invariants_and_lapack(m, l):
    Y = np.random.default_rng(m * 100 + l).standard_normal((m, l))
    Q, R = hqr(Y)
    assert np.abs(Q.T @ Q - np.eye(l)).max() < 1e-14
    assert np.linalg.norm(Q @ R - Y) / np.linalg.norm(Y) < 1e-14
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) >= 0)
    Qn, Rn = np.linalg.qr(Y)                      # LAPACK, sign-normalised
    sg = np.sign(np.diag(Rn))
    assert np.abs(Q - Qn * sg).max() < 1e-12 and np.abs(R - Rn * sg[:, None]).max() < 1e-12


def test_hqr_rank_deficient():
    rng = np.random.default_rng(5)
    G = rng.standard_normal((40, 3))
    Y = np.concatenate([G, G @ rng.standard_normal((3, 3)), np.zeros((40, 2))], axis=1)
    Q, R = hqr(Y)
    assert np.abs(Q.T @ Q - np.eye(8)).max() < 1e-14
    assert np.linalg.norm(Q @ R - Y) / np.linalg.norm(Y) < 1e-14


# ----------------------------------------------------------------------------- Jacobi SVD
def test_jacobi_worked_examples():
    ex = GOLD["svd_diag_3_1_2"]
    d, Ut, V, _ = jacobi_svd_bt(np.array(ex["B"], dtype=float).T)
    assert np.allclose(d, ex["d"], rtol=0, atol=1e-15)
    Qo, _ = np.linalg.qr(np.random.default_rng(3).standard_normal((30, 7)))
    d, Ut, V, _ = jacobi_svd_bt(Qo)              # isometry: all singular values 1
    assert np.abs(d - 1.0).max() < 1e-14


@pytest.mark.parametrize("n,l", [(12, 9), (9, 9), (500, 20), (60, 30)])
def test_jacobi_vs_lapack(n, l):
    rng = np.random.default_rng(n + 7 * l)
    Bt = rng.standard_normal((n, l)) * np.logspace(0, -6, l)[None, :]
    d, Ut, V, sweeps = jacobi_svd_bt(Bt)
    dn = np.linalg.svd(Bt, compute_uv=False)
    assert np.abs(d - dn).max() / dn.max() < 1e-13 and np.all(np.abs(d - dn) / dn < 1e-11)
    assert np.abs(Ut.T @ Ut - np.eye(l)).max() < 1e-13
    assert np.abs(V.T @ V - np.eye(l)).max() < 1e-12
    B = Bt.T
    assert np.linalg.norm(Ut @ np.diag(d) @ V.T - B) / np.linalg.norm(B) < 1e-14
    assert np.all(np.diff(d) <= 0) and sweeps < 30


def test_eckart_young_12x9():
    """||A - A_k||_2 = sigma_{k+1}, ||A - A_k||_F = sqrt(sum_{j>k} sigma_j^2)."""
    A = np.random.default_rng(12).standard_normal((12, 9))
    d, Ut, V, _ = jacobi_svd_bt(A)       # A = (B^T) with B = A^T: A = V diag(d) Ut^T
    for k in range(1, 9):
        Ak = (V[:, :k] * d[:k]) @ Ut[:, :k].T
        assert abs(np.linalg.norm(A - Ak, 2) - d[k]) < 1e-12
        assert abs(np.linalg.norm(A - Ak) - np.sqrt(np.sum(d[k:] ** 2))) < 1e-12


def test_jacobi_rank_deficient():
    rng = np.random.default_rng(2)
    Bt = rng.standard_normal((50, 3)) @ rng.standard_normal((3, 6))
    d, Ut, V, _ = jacobi_svd_bt(Bt)
    assert np.all(d[3:] < 1e-13 * d[0])
    assert np.abs(Ut.T @ Ut - np.eye(6)).max() < 1e-13


def test_soft_threshold_and_dual_norm_examples():
    ex = GOLD["soft_threshold"]
    assert np.array_equal(soft_threshold(ex["x"], ex["tau"]), np.array(ex["y"]))
    x = np.random.default_rng(1).standard_normal(100)
    assert np.array_equal(soft_threshold(x, 0.0), x)
    ex = GOLD["dual_norm_diag_3_0"]
    A = np.array(ex["A"], dtype=float)
    J = max(np.linalg.norm(A, 2), np.abs(A).max() / ex["lam"])
    assert J == ex["J"]


# ----------------------------------------------------------------------------- rsvd
def test_resolve_params():
    assert resolve_params(100, 50, 10) == (10, 10, 10, 20)
    assert resolve_params(100, 50, 45, p=10) == (45, 45, 45, 50)       # l clamped (R10)
    assert resolve_params(100, 50, 10, nu=20, nv=0) == (10, 10, 0, 20)  # clamp / not formed
    for bad in (0, 51):
        with pytest.raises(ValueError):
            resolve_params(100, 50, bad)


def test_rsvd_worked_example_diag():
    ex = GOLD["rsvd_diag_5_3_1"]
    r = oracle_rsvd(np.array(ex["A"], dtype=float), ex["k"], p=ex["p"], q=ex["q"], seed=1)
    assert np.allclose(r["d"], ex["d"], rtol=1e-12, atol=0)


def test_rsvd_config1_exact_rank_planted():
    """Config 1 (J:7): exact rank 10, s_i = 10^(-i/5): recovered to 1e-12 (reading R25)."""
    import synthetic
    A, meta = synthetic.make_config(1)
    A = A.numpy()
    r = oracle_rsvd(A, 10, p=10, q=2, sdist="normal", seed=meta["seed_omega"])
    s = meta["s"].numpy()
    assert np.max(np.abs(r["d"] - s) / s) < 1e-12
    assert np.abs(r["u"].T @ r["u"] - np.eye(10)).max() < 1e-12
    assert np.abs(r["v"].T @ r["v"] - np.eye(10)).max() < 1e-12
    R = A - (r["u"] * r["d"]) @ r["v"].T
    assert np.linalg.norm(R) / np.linalg.norm(A) < 1e-13


@pytest.mark.parametrize("m,n", [(60, 40), (40, 60), (33, 33)])
def test_rsvd_full_sketch_is_exact_svd(m, n):
    """l = min(m,n) => Q Q^T A = A => rsvd equals the deterministic SVD."""
    A = np.random.default_rng(m * n).standard_normal((m, n))
    k = min(m, n)
    r = oracle_rsvd(A, k, p=10, q=1, sdist="unif", seed=3)
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    assert np.abs(r["d"] - s).max() / s[0] < 1e-13
    # singular vectors agree up to sign with LAPACK's
    cu = np.abs(np.sum(r["u"] * U, axis=0))
    cv = np.abs(np.sum(r["v"] * Vt.T, axis=0))
    assert np.all(np.abs(cu - 1) < 1e-9) and np.all(np.abs(cv - 1) < 1e-9)
    # sign convention (R9): the largest-|.| entry of each V column is >= 0
    idx = np.argmax(np.abs(r["v"]), axis=0)
    assert np.all(r["v"][idx, np.arange(k)] > 0)


def test_rsvd_power_scheme_matches_Aq_sketch():
    """Alg. 2 sub_iterations spans range((A A^T)^q A Omega) (Eq. Aq):
    compare with a direct Y = A^(q) Omega on a well-conditioned input."""
    rng = np.random.default_rng(9)
    m, n, l, q = 80, 50, 6, 2
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.linspace(2.0, 1.0, n)
    A = (U * s) @ V.T
    Aq = (U * s ** (2 * q + 1)) @ V.T          # closed form of (A A^T)^q A
    Om = omega(n, l, "normal", seed=4)
    Qd, _ = np.linalg.qr(Aq @ Om)
    Q, Bt = oracle_rqb(A, l, q, "normal", seed=4)
    cosines = np.linalg.svd(Qd.T @ Q, compute_uv=False)
    assert cosines.min() > 1 - 1e-10
    assert np.abs(Bt - A.T @ Q).max() < 1e-13


def test_direct_power_scheme_is_Aq_sketch():
    """Alg. 1 (direct): the sketch after q iterations is exactly
    A^(q) Omega = U S^(2q+1) V^T Omega (Eq. Aq), and on a
    well-conditioned input the whole rsvd agrees with the Alg. 2 path."""
    rng = np.random.default_rng(19)
    m, n, l, q = 90, 60, 8, 2
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.linspace(2.0, 1.0, n)
    A = (U * s) @ V.T
    Aq = (U * s ** (2 * q + 1)) @ V.T
    Om = omega(n, l, "normal", seed=6)
    Qd, _ = np.linalg.qr(Aq @ Om)
    Q, Bt = oracle_rqb(A, l, q, "normal", seed=6, power="direct")
    assert np.linalg.svd(Qd.T @ Q, compute_uv=False).min() > 1 - 1e-12
    assert np.abs(Bt - A.T @ Q).max() < 1e-13
    r1 = oracle_rsvd(A, 5, p=3, q=q, seed=6, power="direct")
    r2 = oracle_rsvd(A, 5, p=3, q=q, seed=6)
    assert np.abs(r1["d"] - r2["d"]).max() < 1e-12
    assert np.abs(np.abs(np.sum(r1["v"] * r2["v"], axis=0)) - 1).max() < 1e-9


def test_rsvd_wide_input_transposes():
    A = np.random.default_rng(4).standard_normal((30, 70))
    r = oracle_rsvd(A, 5, nu=5, nv=3, p=5, q=1, seed=2)
    assert r["u"].shape == (30, 5) and r["v"].shape == (70, 3)
    rt = oracle_rsvd(A.T, 5, p=5, q=1, seed=2)
    assert np.abs(r["d"] - rt["d"]).max() < 1e-12


def _lowrank_decay(m, n, seed, decay=0.7, noise=0.0):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = decay ** np.arange(n)
    return (U * s) @ V.T, s


def test_rsvd_expected_error_bound():
    """E||A - A_k||_2 <= factor * sigma_{k+1}, mean over 50 seeds."""
    m, n, k, p = 120, 60, 8, 4
    A, s = _lowrank_decay(m, n, 21, decay=0.85)
    for q in (0, 1):
        errs = []
        for seed in range(50):
            r = oracle_rsvd(A, k, p=p, q=q, sdist="normal", seed=seed)
            errs.append(np.linalg.norm(A - (r["u"] * r["d"]) @ r["v"].T, 2))
        assert np.mean(errs) <= error_bound_factor(k, p, q, m, n) * s[k]
        assert min(errs) >= s[k] * (1 - 1e-10)                  # Eckart-Young


def test_rsvd_error_nonincreasing_in_q():
    A, s = _lowrank_decay(150, 80, 8, decay=0.93)
    k = 10
    means = []
    for q in (0, 1, 2, 3):
        e = [np.linalg.norm(A - (lambda r: (r["u"] * r["d"]) @ r["v"].T)(
            oracle_rsvd(A, k, p=5, q=q, seed=sd))) for sd in range(10)]
        means.append(np.mean(e))
    assert all(means[i + 1] <= means[i] * (1 + 1e-12) for i in range(3))
    assert means[-1] >= np.sqrt(np.sum(s[k:] ** 2)) * (1 - 1e-12)


def test_rsvd_fp32_input_semantics():
    A = np.random.default_rng(0).standard_normal((40, 20)).astype(np.float32)
    r32 = oracle_rsvd(A, 5, p=5, q=1, seed=1)
    Om = omega(20, 10, "normal", 1, 0, dtype=np.float32)
    Q, Bt = oracle_rqb(A.astype(np.float64), 10, 1, "normal", 1, 0, omega_dtype=np.float32)
    d = np.linalg.svd(Bt, compute_uv=False)
    assert np.abs(r32["d"] - d[:5]).max() < 1e-12 * d[0]
    assert Om.dtype == np.float64


# ----------------------------------------------------------------------------- rpca
def test_rpca_eigenvalues_are_covariance_eigenvalues():
    """Lambda = Sigma^2 / (m-1) equal the covariance eigenvalues (Eq. P:1322)."""
    rng = np.random.default_rng(6)
    X = rng.standard_normal((90, 12)) @ rng.standard_normal((12, 12)) + 5.0
    out = oracle_rpca(X, 12, center=True, scale=False, p=5, q=1, seed=2)
    ev = np.sort(np.linalg.eigvalsh(np.cov(X, rowvar=False)))[::-1]
    assert np.abs(out["eigvals"] - ev).max() / ev[0] < 1e-12
    assert np.abs(out["center"] - X.mean(axis=0)).max() < 1e-13
    Xc = X - X.mean(axis=0)
    assert np.abs(out["x"] - Xc @ out["rotation"]).max() < 1e-11   # scores = X W
    out_s = oracle_rpca(X, 12, center=True, scale=True, p=5, q=1, seed=2)
    evs = np.sort(np.linalg.eigvalsh(np.corrcoef(X, rowvar=False)))[::-1]
    assert np.abs(out_s["eigvals"] - evs).max() < 1e-12


@pytest.mark.parametrize("scale", [False, True])
def test_rpca_loadings_whitening_explained_variance(scale):
    """Full-rank case k = n (l = min(m, n): the exact SVD), checked against what
    the paper and linear algebra fix, not against the oracle's own formulas:
    * loadings L = W Lambda^1/2 factor the covariance (correlation) matrix,
      C = L L^T, the squared column sums are the eigenvalues and the squared
      row sums the variables' variances;
    * the whitened PCs have unit variance and are uncorrelated (P:1262-1266,
      Fig. 4b "uncorrelated and have unit variance"): cov(Z_white) = I;
    * the proportions of variance sum to 1 over all n components, and the
      total variance is the trace of np.cov / np.corrcoef."""
    rng = np.random.default_rng(17)
    X = rng.standard_normal((120, 9)) @ rng.standard_normal((9, 9)) * np.arange(1, 10) + 3.0
    out = oracle_rpca(X, 9, center=True, scale=scale, p=0, q=1, seed=4)
    C = np.corrcoef(X, rowvar=False) if scale else np.cov(X, rowvar=False)
    L = out["loadings"]
    assert np.abs(L @ L.T - C).max() < 1e-11 * np.abs(C).max()
    assert np.abs((L * L).sum(axis=0) - out["eigvals"]).max() < 1e-11 * out["eigvals"][0]
    assert np.abs((L * L).sum(axis=1) - np.diag(C)).max() < 1e-11 * np.abs(C).max()
    Zw = out["x_white"]
    assert np.abs(np.cov(Zw, rowvar=False) - np.eye(9)).max() < 1e-10
    assert abs(out["total_var"] - np.trace(C)) < 1e-12 * np.trace(C)
    assert abs(out["var_cum"][-1] - 1.0) < 1e-12
    assert np.all(np.diff(out["var_cum"]) >= 0)
    assert np.abs(out["var_ratio"] - np.linalg.eigvalsh(C)[::-1] / np.trace(C)).max() < 1e-12


def test_rpca_predict_reproduces_training_scores():
    """predict() on the training rows gives back the scores of Alg. 6
    step (3), Z = U Sigma, when the range is captured exactly (k = n, so
    Q Q^T X = X and X W = U Sigma V^T W = U Sigma, Eq. PCs); rows equal to
    the column means map to the origin."""
    rng = np.random.default_rng(23)
    X = rng.standard_normal((200, 30)) @ np.diag(np.exp(-np.arange(30) / 6.0)) + 2.0
    for scale in (False, True):
        out = oracle_rpca(X, 30, center=True, scale=scale, p=0, q=1, seed=7)
        P = oracle_rpca_predict(X, out["rotation"], out["center"], out["scale"])
        assert np.abs(P - out["x"]).max() < 1e-10 * np.abs(out["x"]).max()
        origin = oracle_rpca_predict(out["center"][None, :], out["rotation"], out["center"], out["scale"])
        assert np.abs(origin).max() == 0.0


# ----------------------------------------------------------------------------- rrpca
def test_rrpca_recovers_planted_low_rank_plus_sparse():
    """Scaled analogue of the paper's synthetic study with the
    config-5 construction; ground truth pins the mu reading (R17)."""
    import synthetic
    A, L0, S0 = synthetic.sparse_plus_lowrank(2000, 200, rank=5, frac=0.05, seed=31)
    A, L0, S0 = A.numpy(), L0.numpy(), S0.numpy()
    out = oracle_rrpca(A, k=10, p=10, q=2, tol=1e-7, maxiter=100, seed=5)
    assert out["residual"] < 1e-7 and out["iters"] < 100
    assert np.linalg.norm(out["L"] - L0) / np.linalg.norm(L0) < 1e-5
    supp = (np.abs(out["S"]) > 1e-6) == (S0 != 0)
    assert supp.mean() > 0.999
    assert abs(out["lam"] - 1 / np.sqrt(2000)) < 1e-16


def test_predict_rank_rule():
    """Alg. 7 step (7) predict_rank (Remark 1 P:1716), reading R30:
    worked cases of the stated rule (SPEC predict_rank examples)."""
    assert predict_rank([5, 3, 0.1], 1.0, 2, 100) == (7, 2)       # l == k: grow by ceil(5% of 100)
    assert predict_rank([0.5, 0.2], 1.0, 2, 100) == (2, 1)        # nothing above 1/mu: l floored to 1
    assert predict_rank([5, 3, 0.1], 1.0, 10, 100) == (3, 2)      # l < k: shrink to l + 1
    assert predict_rank([9, 8, 7], 1.0, 3, 3) == (3, 3)           # growth capped at min(m, n)
    assert predict_rank([9, 8, 7], 1.0, 3, 41) == (6, 3)          # ceil(0.05 * 41) = 3
    assert predict_rank([2.0, 1.0], 1.0, 2, 10) == (2, 1)         # strict '>' at the threshold


def test_rrpca_adaptive_rank_settles_at_rank_plus_one():
    """k = 0: k starts at 2 (step (1)) and predict_rank grows it until the
    thresholded rank l stops at the planted rank 5, after which k = l + 1 = 6;
    the planted L0, S0 are recovered (ground truth, not the oracle itself)."""
    import synthetic
    A, L0, S0 = synthetic.sparse_plus_lowrank(2000, 200, rank=5, frac=0.05, seed=31)
    A, L0, S0 = A.numpy(), L0.numpy(), S0.numpy()
    out = oracle_rrpca(A, k=0, p=10, q=2, tol=1e-7, maxiter=100, seed=5)
    tr = out["trace"]
    assert tr[0][3] == 2                                   # step (1): k = 2
    assert all(t[3] <= 200 // 4 for t in tr)               # stays randomized (Remark 2)
    assert tr[-1][1] == 5 and tr[-1][3] == 6               # l = rank, k = l + 1
    assert out["residual"] < 1e-7
    assert np.linalg.norm(out["L"] - L0) / np.linalg.norm(L0) < 1e-5
    assert ((np.abs(out["S"]) > 1e-6) == (S0 != 0)).mean() > 0.999


# ----------------------------------------------------------------------------- id / rid / rcur (§8(f) f3)
def test_qrcp_matches_lapack_geqp3():
    """Pivoted QR (Alg. id step (1)) against LAPACK's geqp3 (scipy):
    same pivot order on inputs with distinct column norms, |diag S| equal,
    and A(:, P) = Q S reconstructed with the oracle's own factor."""
    import scipy.linalg as sl
    from oracle.linalg import qrcp
    rng = np.random.default_rng(21)
    for m, n in [(40, 30), (25, 60), (9, 9)]:
        A = rng.standard_normal((m, n)) * np.exp(-np.arange(n) / 10.0)[None, :]
        S, P = qrcp(A)
        _q, R, P2 = sl.qr(A, pivoting=True)
        assert (P == P2).all()
        r = min(m, n)
        assert np.abs(np.abs(np.diag(S[:r, :r])) - np.abs(np.diag(R[:r, :r]))).max() < 1e-12
        assert np.abs(np.tril(S[:r, :r], -1)).max() == 0.0
        # orthogonal invariance: S^T S = A(:,P)^T A(:,P)
        assert np.abs(S.T @ S - A[:, P].T @ A[:, P]).max() < 1e-12 * np.abs(A).max() ** 2 * m


def test_id_worked_example_and_exact_rank():
    """Alg. id.  Hand case: diag(1, 3, 2) pivots the columns by
    norm (P = [1, 2, 0]), k = 2 gives J = [1, 2] and Z = [[0, 1, 0], [0, 0, 1]].
    Exact rank k: C Z = A (the ID is exact), Z(:, J) = I_k."""
    from oracle.rsvd import oracle_id
    r = oracle_id(np.diag([1.0, 3.0, 2.0]), 2)
    assert list(r["J"]) == [1, 2]
    assert np.abs(r["Z"] - np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])).max() < 1e-15
    rng = np.random.default_rng(22)
    A = rng.standard_normal((150, 9)) @ rng.standard_normal((9, 80))
    r = oracle_id(A, 9)
    assert np.abs(r["C"] @ r["Z"] - A).max() < 1e-12 * np.abs(A).max()
    assert np.abs(r["Z"][:, r["J"]] - np.eye(9)).max() < 1e-15
    assert np.abs(r["C"] - A[:, r["J"]]).max() == 0.0


def test_rid_rcur_exact_rank_reconstruct():
    """Alg. rid and rcur on an exactly rank-k
    input: C Z = A and C U R = A to rounding (C and R span the column and row
    spaces), the randomized ID picks the same columns as the deterministic ID
    of A when l = min(m, n) (Q Q^T A = A, so B = Q^T A has A's pivots)."""
    from oracle.rsvd import oracle_id, oracle_rid, oracle_rcur
    rng = np.random.default_rng(23)
    A = rng.standard_normal((300, 12)) @ rng.standard_normal((12, 90))
    r = oracle_rid(A, 12, p=6, q=1, seed=3)
    assert np.abs(r["C"] @ r["Z"] - A).max() < 1e-11 * np.abs(A).max()
    c = oracle_rcur(A, 12, p=6, q=1, seed=3)
    assert np.abs(c["C"] @ c["U"] @ c["R"] - A).max() < 1e-10 * np.abs(A).max()
    assert np.abs(c["R"] - A[c["I"], :]).max() == 0.0
    small = rng.standard_normal((40, 25))
    full = oracle_rid(small, 5, p=20, q=0, seed=1)     # l = 25 = min(m, n)
    det = oracle_id(small, 5)
    assert list(full["J"]) == list(det["J"])


def test_lu_pp_matches_scipy_and_normalized_iterations():
    """Alg. 3: the pivoted LU written out equals scipy's (LAPACK
    getrf) permuted L on random inputs; the normalized power iterations span
    the same space as Alg. 2 (Eq. Aq), so rsvd agrees on a well-conditioned
    input."""
    import scipy.linalg as sl
    from oracle.linalg import lu_pp
    rng = np.random.default_rng(24)
    Y = rng.standard_normal((50, 8))
    L, piv = lu_pp(Y)
    PL, U = sl.lu(Y, permute_l=True)
    assert np.abs(L - PL).max() < 1e-13
    Ut = np.triu(np.linalg.solve(L[piv, :], Y[piv, :]))
    assert np.abs(L @ Ut - Y).max() < 1e-12
    U_, _ = np.linalg.qr(rng.standard_normal((90, 60)))
    V_, _ = np.linalg.qr(rng.standard_normal((60, 60)))
    A = (U_ * np.linspace(2.0, 1.0, 60)) @ V_.T
    r1 = oracle_rsvd(A, 5, p=3, q=2, seed=6, power="lu")
    r2 = oracle_rsvd(A, 5, p=3, q=2, seed=6)
    assert np.abs(r1["d"] - r2["d"]).max() < 1e-12

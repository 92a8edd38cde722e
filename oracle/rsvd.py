"""rqb / rsvd / rpca / rrpca, step by step in the paper's order (oracle, FP64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

``oracle_rsvd`` follows Alg. 4 ``rqb``, Alg. 2
``sub_iterations`` and Alg. 5 ``rsvd``:

  (1) l = k + p                      (Alg. 4 step 1; clamp l <= min(m,n), reading R10)
  (2) Omega = rnorm(n, l)            (step 2; counter spec, oracle/philox.py)
  (3) Y = A Omega                    (step 3, Eq. YAQ)
  (4) for j = 1..q:                  (Alg. 2)
        [Q,~] = qr(Y); [Q,~] = qr(A^T Q); Y = A Q
  (9) [Q,~] = qr(Y)                  (step 9; reading R3: the last QR follows the loop)
  (10) B = Q^T A                     (step 10, Eq. BQA) -- formed as B^T = A^T Q
  Alg. 5 (2) [U~, Sigma, V] = svd(B)  (economic; jacobi_svd_bt on B^T)
  Alg. 5 (3) U = Q U~                (Eq. UQU)
  return U(:,1:nu), d = diag(Sigma)(1:k), V(:,1:nv)
  plus the sign convention of reading R9 (largest-|.| entry of each V column >= 0).

Matrix products use numpy's ``@`` (a library primitive, as the task allows);
the QR and SVD are written out in oracle/linalg.py.
"""
import numpy as np

from .linalg import hqr, jacobi_svd_bt, lu_pp, qrcp, soft_threshold
from .philox import omega


def resolve_params(m, n, k, nu=None, nv=None, p=10, q=2):
    """Parameter resolution (step a1; readings R10, R11).

    1 <= k <= min(m, n) else ValueError; p >= 0, q >= 0; l = min(k+p, min(m,n));
    nu, nv default k, values > k are clamped to k, 0 means "not formed".
    """
    mn = min(m, n)
    if not (1 <= k <= mn):
        raise ValueError("k must satisfy 1 <= k <= min(m, n)")
    if p < 0 or q < 0:
        raise ValueError("p and q must be >= 0")
    nu = k if nu is None else min(max(int(nu), 0), k)
    nv = k if nv is None else min(max(int(nv), 0), k)
    l = min(k + p, mn)
    return k, nu, nv, l


def sign_fix(U, V):
    """Reading R9: for every column i, if the largest-|.| entry of V(:,i)
    (lowest index on ties) is negative, negate V(:,i) and U(:,i)."""
    U = U.copy()
    V = V.copy()
    for i in range(V.shape[1]):
        idx = int(np.argmax(np.abs(V[:, i])))
        if V[idx, i] < 0:
            V[:, i] = -V[:, i]
            if U is not None and i < U.shape[1]:
                U[:, i] = -U[:, i]
    return U, V


def _prepare(A, center=False, scale=False):
    """Upcast exactly to FP64; optional column centring/scaling (Alg. 6)."""
    X = np.array(A, dtype=np.float64)
    m = X.shape[0]
    c = None
    s = None
    if center:
        c = X.sum(axis=0) / m
        X = X - c[None, :]
    if scale:
        s = np.sqrt((X * X).sum(axis=0) / (m - 1))
        s = np.where(s > 0, s, 1.0)
        X = X / s[None, :]
    return X, c, s


def oracle_rqb(A, l, q=2, sdist="normal", seed=0, stream=0, omega_dtype=np.float64,
               power="subspace"):
    """Alg. 4 rqb with Alg. 2 sub_iterations (power="subspace"), the direct
    power scheme of Alg. 1 (power="direct") or the normalized power
    iterations of Alg. 3 (power="lu"): returns Q (m x l), B^T (n x l)."""
    X = np.asarray(A, dtype=np.float64)
    m, n = X.shape
    Om = omega(n, l, sdist, seed, stream, dtype=omega_dtype)   # step (2)
    Y = X @ Om                                                  # step (3)
    for _ in range(q):                                          # step (4)
        if power == "direct":                                   # Alg. 1
            Y = X.T @ Y                                         #   (2)
            Y = X @ Y                                           #   (3)
            continue
        if power == "lu":                                       # Alg. 3
            Lq, _p = lu_pp(Y)                                   #   (2) [L,~] = lu(Y)
            Lz, _p = lu_pp(X.T @ Lq)                            #   (3) [L,~] = lu(A^T L)
            Y = X @ Lz                                          #   (4)
            continue
        Q, _r = hqr(Y)                                          # Alg. 2 (2)
        Qz, _r = hqr(X.T @ Q)                                   #   (3)
        Y = X @ Qz                                              #   (4)
    Q, _r = hqr(Y)                                              # step (9)
    Bt = X.T @ Q                                                # step (10), B^T = A^T Q
    return Q, Bt


def oracle_rsvd(A, k, nu=None, nv=None, p=10, q=2, sdist="normal", seed=0,
                stream=0, center=False, scale=False, full=False, power="subspace"):
    """Alg. 5 rsvd with the interface of P:708.

    Returns dict(d, u, v, l, center, scale) -- d: (k,), u: m x nu, v: n x nv.
    ``full=True`` additionally returns the untruncated l-column factors.
    FP32 ``A`` -> Omega rounded to FP32 (reading R12), arithmetic in FP64.
    """
    A = np.asarray(A)
    omega_dtype = np.float32 if A.dtype == np.float32 else np.float64
    X, c, s = _prepare(A, center, scale)
    m, n = X.shape
    k, nu, nv, l = resolve_params(m, n, k, nu, nv, p, q)
    transposed = m < n
    W = X.T if transposed else X
    Q, Bt = oracle_rqb(W, l, q, sdist, seed, stream, omega_dtype, power=power)
    sigma, Ut, V, sweeps = jacobi_svd_bt(Bt)                    # Alg. 5 (2)
    U = Q @ Ut                                                  # Alg. 5 (3), Eq. UQU
    if transposed:
        U, V = V, U
    U, V = sign_fix(U, V)
    out = dict(d=sigma[:k].copy(), u=U[:, :nu].copy(), v=V[:, :nv].copy(), l=l,
               center=c, scale=s, sweeps=sweeps)
    if full:
        out.update(d_full=sigma, u_full=U, v_full=V)
    return out


def oracle_rpca(A, k, center=True, scale=True, retx=True, p=10, q=2,
                sdist="normal", seed=0, stream=0):
    """Alg. 6 rpca / interface P:1381-1398 (defaults
    center = TRUE, scale = TRUE as in P:1381).

    rsvd on the centred (and optionally scaled) X; eigenvalues
    Lambda = Sigma^2 / (m-1) (Eq. P:1322), rotation W = V, sdev = sqrt(Lambda)
    (P:1396), scores x = U Sigma (= X W, Eq. PCs).  Also the quantities of
    Sections 4.1-4.2 and summary():
      loadings  L = W Lambda^{1/2}
      x_white   z_i / sqrt(lambda_i), i.e. Z Lambda^{-1/2} (
                reading R32: the printed "X L" contradicts the line after it,
                which whitening by 1/sqrt(lambda_i) defines)
      total_var sum of ALL n eigenvalues = trace of the covariance
                (correlation) matrix = sum of the column variances of X
      var_ratio lambda_i / total_var, var_cum its cumulative sum
    """
    r = oracle_rsvd(A, k, p=p, q=q, sdist=sdist, seed=seed, stream=stream,
                    center=center, scale=scale)
    X, _c, _s = _prepare(A, center, scale)
    m = X.shape[0]
    eig = r["d"] ** 2 / (m - 1)
    sdev = np.sqrt(eig)
    total = float(np.sum(X * X) / (m - 1))          # the column variances of X, summed
    out = dict(rotation=r["v"], eigvals=eig, sdev=sdev, center=r["center"],
               scale=r["scale"], d=r["d"], loadings=r["v"] * sdev[None, :],
               total_var=total, var_ratio=eig / total, var_cum=np.cumsum(eig) / total)
    if retx:
        out["x"] = r["u"] * r["d"][None, :]
        out["x_white"] = out["x"] / sdev[None, :]
    return out


def oracle_rpca_predict(Anew, rotation, center=None, scale=None):
    """predict() of an rpca object: the new rows centred and
    scaled with the training statistics, then rotated: ((Anew - c) / s) W."""
    X = np.array(Anew, dtype=np.float64)
    if center is not None:
        X = X - np.asarray(center, dtype=np.float64)[None, :]
    if scale is not None:
        X = X / np.asarray(scale, dtype=np.float64)[None, :]
    return X @ np.asarray(rotation, dtype=np.float64)


def predict_rank(d, mu_inv, k, minmn):
    """Alg. 7 step (7) "k, l = predict_rank(Sigma, mu^-1)"; the paper
    defers the rule to Lin et al. (Remark 1).  Reading R30:
      l = max(1, #{d_i > mu^-1})
      k_next = l + 1                                if l < k
               min(l + ceil(0.05 minmn), minmn)    otherwise
    Returns (k_next, l)."""
    l = max(1, int(np.sum(np.asarray(d) > mu_inv)))
    if l < k:
        return l + 1, l
    return min(l + int(np.ceil(0.05 * minmn)), minmn), l


def oracle_rrpca(A, lam=None, maxiter=100, tol=1e-7, k=20, p=10, q=2,
                 sdist="normal", seed=0, trace=False, kmax=None, det_switch=True, rand=True):
    """Alg. 7 rrpca, the inexact ALM loop, readings R17-R23, R30.

    lambda = max(m,n)^-1/2;  ||A||_2 = sigma_1 of rsvd(A, 1, p, q,
    stream 0) (R18);  mu_0 = 1.25 / ||A||_2 (R17);  Z = A / J(A) with
    J(A) = max(||A||_2, ||A||_max / lambda) (R19);  S = 0.  Then repeat:
      (6)  [U, Sigma, V] = rsvd(A - S + Z/mu, k, p, q)   (fresh Omega: stream t, R23)
      (7)  l = #{sigma_i > 1/mu}                         (fixed k > 0, R22)
           k, l = predict_rank(Sigma, 1/mu)              (k = 0: adaptive, k starts at 2, R30)
      (8)  Sigma_l = soft_thres(sigma(1:l), 1/mu)
      (9)  L = U(:,1:l) Sigma_l V(:,1:l)^T
      (10) S = soft_thres(A - L + Z/mu, lambda/mu)
      (11) Z = Z + (A - L - S) mu
      (12) mu = min(1.5 mu, 1e7 mu_0)                    (R20)
      until ||A - L - S||_F / ||A||_F < tol  (R21; evaluated after step 11)
    Adaptive mode: predicted k is capped at kmax (default min(m, n)); with
    det_switch the truncated SVD of step (6) is the deterministic one (numpy
    SVD) whenever k > min(m, n)/4 (Remark 2).  rand=False: the
    deterministic truncated SVD in every iteration.
    Returns dict(L, S, iters, residual, trace=[(res, l, mu, k)...],
    sigmas=[the step-(6) singular values of every iteration]).  tol <= 0 runs
    exactly maxiter iterations.
    """
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    minmn = min(m, n)
    adaptive = k == 0
    if kmax is None:
        kmax = minmn
    if adaptive:
        k = min(2, kmax)
    if lam is None or lam <= 0:
        lam = 1.0 / np.sqrt(max(m, n))
    norm2 = oracle_rsvd(A, 1, p=p, q=q, sdist=sdist, seed=seed, stream=0)["d"][0]
    mu0 = 1.25 / norm2
    mu = mu0
    dual = max(norm2, np.max(np.abs(A)) / lam)
    Z = A / dual
    S = np.zeros_like(A)
    normF = np.sqrt(np.sum(A * A))
    hist = []
    sigmas = []
    L = np.zeros_like(A)
    res = np.inf
    it = 0
    for it in range(1, maxiter + 1):
        M = A - S + Z / mu
        if (not rand) or (adaptive and det_switch and k > minmn / 4):
            uu, dd, vt = np.linalg.svd(M, full_matrices=False)
            r = dict(u=uu[:, :k], d=dd[:k], v=vt[:k].T)
        else:
            r = oracle_rsvd(M, k, p=p, q=q, sdist=sdist, seed=seed, stream=it)
        d = r["d"]
        sigmas.append(np.array(d, copy=True))
        nl = int(np.sum(d > 1.0 / mu))
        kused = k
        if adaptive:
            k, _ = predict_rank(d, 1.0 / mu, k, minmn)
            k = min(k, kmax)
        dl = soft_threshold(d[:nl], 1.0 / mu)
        L = (r["u"][:, :nl] * dl[None, :]) @ r["v"][:, :nl].T
        S = soft_threshold(A - L + Z / mu, lam / mu)
        E = A - L - S
        Z = Z + E * mu
        res = np.sqrt(np.sum(E * E)) / normF
        hist.append((res, nl, mu, kused))
        mu = min(1.5 * mu, 1e7 * mu0)
        if res < tol:
            break
    return dict(L=L, S=S, iters=it, residual=res, trace=hist, lam=lam, mu0=mu0,
                norm2=norm2, sigmas=sigmas)


def _triu_solve(S, B):
    """X = S^-1 B for upper-triangular nonsingular S (back substitution)."""
    k = S.shape[0]
    X = np.zeros_like(B, dtype=np.float64)
    for i in range(k - 1, -1, -1):
        X[i] = (B[i] - S[i, i + 1:] @ X[i + 1:]) / S[i, i]
    return X


def oracle_id(A, k):
    """Alg. id, column interpolative decomposition A ~ C Z:
      (1) [~, S, P] = qr(A)  pivoted QR, k steps
      (2) S^+ = pinv(S(1:k, 1:k))      -- S(1:k,1:k) is upper triangular; for
                                         rank >= k it is invertible and pinv = the
                                         inverse (back substitution, reading R31)
      (3) T = S^+ S(1:k, (k+1):n)
      (4)-(5) Z = 0 (k x n); Z(:, P) = [I_k, T]
      (6) J = P(1:k);  (7) C = A(:, J)
    Returns dict(C, Z, J, S, P)."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    S, P = qrcp(A, k)
    d = np.abs(np.diag(S[:k, :k]))
    if not d[0] > 0 or np.any(d[1:] <= m * 2.0 ** -52 * d[0]):
        raise ValueError("numerical rank < k: S(1:k,1:k) singular (reading R31)")
    T = _triu_solve(S[:k, :k], S[:k, k:])
    Z = np.zeros((k, n))
    Z[:, P] = np.hstack([np.eye(k), T])
    J = P[:k].copy()
    return dict(C=A[:, J].copy(), Z=Z, J=J, S=S, P=P)


def oracle_rid(A, k, p=10, q=2, sdist="normal", seed=0, stream=0):
    """Alg. rid: (1) [~, B] = rqb(A, k, q, p) (Alg. 4; the
    argument order in the listing is a typo, reading R27); (2) [~, Z, J] =
    id(B, k); (3) C = A(:, J).  Returns dict(C, Z, J)."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    k, _, _, l = resolve_params(m, n, k, 0, 0, p, q)
    Q, Bt = oracle_rqb(A, l, q, sdist, seed, stream)
    r = oracle_id(Bt.T, k)
    return dict(C=A[:, r["J"]].copy(), Z=r["Z"], J=r["J"])


def oracle_rcur(A, k, p=10, q=2, sdist="normal", seed=0, stream=0):
    """Alg. rcur:
      (1) [C, Z, J] = rid(A, k, p, q)
      (2) [~, S, P] = qr(C^T)  pivoted QR;  (3) I = P(1:k)
      (4) R = A(I, :);  (5) R^+ = pinv(R);  (6) U = Z R^+
    pinv(R) for the full-row-rank R (k x n): R^+ = Q_R S_R^-T from the
    Householder QR R^T = Q_R S_R (reading R31).  Returns dict(C, U, R, J, I)."""
    A = np.asarray(A, dtype=np.float64)
    r = oracle_rid(A, k, p, q, sdist, seed, stream)
    k = r["C"].shape[1]
    _S, P = qrcp(r["C"].T, k)
    I = P[:k].copy()
    R = A[I, :].copy()
    Qr, Sr = hqr(R.T)
    Rpinv = Qr @ _triu_solve(Sr, np.eye(k)).T          # Q_R S_R^-T
    U = r["Z"] @ Rpinv
    return dict(C=r["C"], U=U, R=R, J=r["J"], I=I, Z=r["Z"])

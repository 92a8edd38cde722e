"""Deterministic kernels the randomized algorithms call (oracle side, FP64).

* ``hqr``: economic QR by Householder reflections, explicit thin Q, diag(R)>=0.
  Paper: "[Q,~] = qr(Y)  economic QR" (Alg. 2 steps (2)-(3), PAPER.md:377-378;
  Alg. 4 step (9); "QR-decomposition Y =: QR").
* ``jacobi_svd_bt``: economic SVD of B (l x n) by one-sided (Hestenes) Jacobi
  applied to the columns of B^T.  Paper: "[U~, Sigma, V] = svd(B)  compute
  economic SVD" (Alg. 5 step (2)) -- "any exact-arithmetic-equivalent
  economic SVD" (reading R7).
* ``soft_threshold``: shrink(x, tau) = sign(x) max(|x| - tau, 0)
  (Alg. 7 steps (8) and (10)).
* ``lu_pp``: LU with partial pivoting, "[L, ~] = lu(Y)  pivoted LU" (Alg. 3
  norm_iterations steps (2)-(3)): returns the permuted unit lower
  factor L (Y = L U with L = P^T L_unit).
* ``qrcp``: QR with column pivoting, "[~, S, P] = qr(A)  pivoted QR
  decomposition" (Alg. id step (1); "stopped after k iterations to
  obtain only the k dominant pivots"): Businger-Golub largest
  remaining column norm, ties to the lowest index (reading R31).

Plain loops over columns / column pairs with numpy vector operations; no
blocking, no reordering beyond the textbook algorithms.
"""
import numpy as np


def _sign(x):
    """sign with sign(0) = +1 (reading R6)."""
    return 1.0 if x >= 0 else -1.0


def hqr(Y):
    """Householder QR of Y (m x l, m >= l): returns Q (m x l), R (l x l).

    For each column j: x = R(j:, j); alpha = -sign(x_0) ||x||; v = x - alpha e_1;
    H_j = I - 2 v v^T / (v^T v) applied to the trailing columns.  A column with
    ||x|| == 0 is skipped (H_j = I, R_jj = 0), so exactly rank-deficient Y still
    yields an orthonormal Q.  Q = H_1 ... H_l [I_l; 0] by back-accumulation.
    Finally columns of Q / rows of R are flipped so that diag(R) >= 0.
    """
    Y = np.array(Y, dtype=np.float64)
    m, l = Y.shape
    if m < l:
        raise ValueError("hqr needs m >= l")
    R = Y.copy()
    vs = []
    for j in range(l):
        x = R[j:, j]
        nx = np.sqrt(np.dot(x, x))
        if nx == 0.0:
            vs.append(None)
            continue
        alpha = -_sign(x[0]) * nx
        v = x.copy()
        v[0] -= alpha
        vtv = np.dot(v, v)
        w = v @ R[j:, j:]
        R[j:, j:] -= np.outer(v, w) * (2.0 / vtv)
        R[j + 1:, j] = 0.0
        R[j, j] = alpha
        vs.append((v, vtv))
    Q = np.zeros((m, l))
    Q[:l, :l] = np.eye(l)
    for j in range(l - 1, -1, -1):
        if vs[j] is None:
            continue
        v, vtv = vs[j]
        w = v @ Q[j:, :]
        Q[j:, :] -= np.outer(v, w) * (2.0 / vtv)
    R = np.triu(R[:l, :])
    for j in range(l):
        if R[j, j] < 0:
            R[j, :] = -R[j, :]
            Q[:, j] = -Q[:, j]
    return Q, R


def jacobi_svd_bt(Bt, max_sweeps=30):
    """Economic SVD of B from B^T (n x l) by one-sided Jacobi on its columns.

    Cyclic row-by-row pair order (p < q).  For columns b_p, b_q:
    alpha = ||b_p||^2, beta = ||b_q||^2, gamma = b_p . b_q; rotate iff
    |gamma| > tau sqrt(alpha beta), tau = l 2^-52 (reading R8).
    zeta = (beta - alpha) / (2 gamma), t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)),
    c = 1/sqrt(1 + t^2), s = c t;  b_p <- c b_p - s b_q, b_q <- s b_p + c b_q
    (old b_p in both), and the same on columns p, q of J (l x l, J0 = I).
    Stop after a sweep without rotations (cap ``max_sweeps``: RuntimeError).

    Then B^T J = W Sigma with W = [b_i / sigma_i]:  B = J Sigma W^T, i.e.
    U~ = J and V = W.  Sorted by sigma descending (stable).
    Returns (sigma (l,), Ut (l x l), V (n x l), sweeps).
    """
    X = np.array(Bt, dtype=np.float64)
    n, l = X.shape
    J = np.eye(l)
    tau = l * 2.0 ** -52
    sweeps = 0
    for sweep in range(max_sweeps + 1):
        rotated = False
        for p in range(l - 1):
            for q in range(p + 1, l):
                bp = X[:, p]
                bq = X[:, q]
                alpha = np.dot(bp, bp)
                beta = np.dot(bq, bq)
                gamma = np.dot(bp, bq)
                if not abs(gamma) > tau * np.sqrt(alpha * beta):
                    continue
                rotated = True
                zeta = (beta - alpha) / (2.0 * gamma)
                t = _sign(zeta) / (abs(zeta) + np.sqrt(1.0 + zeta * zeta))
                c = 1.0 / np.sqrt(1.0 + t * t)
                s = c * t
                xp = X[:, p].copy()
                X[:, p] = c * xp - s * X[:, q]
                X[:, q] = s * xp + c * X[:, q]
                jp = J[:, p].copy()
                J[:, p] = c * jp - s * J[:, q]
                J[:, q] = s * jp + c * J[:, q]
        if not rotated:
            break
        sweeps += 1
        if sweeps > max_sweeps:
            raise RuntimeError("one-sided Jacobi did not converge in %d sweeps" % max_sweeps)
    sigma = np.sqrt(np.einsum("ij,ij->j", X, X))
    V = X.copy()
    nz = sigma > 0
    V[:, nz] = X[:, nz] / sigma[nz]
    order = np.argsort(-sigma, kind="stable")
    return sigma[order], J[:, order], V[:, order], sweeps


def soft_threshold(x, tau):
    """shrink(x, tau) = sign(x) * max(|x| - tau, 0), entrywise."""
    x = np.asarray(x, dtype=np.float64)
    return np.sign(x) * np.maximum(np.abs(x) - tau, 0.0)


def qrcp(A, steps=None):
    """Householder QR with column pivoting (Businger-Golub), `steps` pivots.

    At step j the column with the largest 2-norm of rows j.. among the not yet
    pivoted columns is swapped to position j (first one on ties, reading R31),
    then reflected with the hqr convention (alpha = -sign(x_0) ||x||,
    H = I - 2 v v^T / v^T v).  Returns S (min(m, steps) x n, upper trapezoidal
    in the pivoted column order; rows >= steps hold the un-reduced remainder
    when steps < min(m, n)) and the permutation P (column j of S is column
    P[j] of A)."""
    R = np.array(A, dtype=np.float64)
    m, n = R.shape
    steps = min(m, n) if steps is None else min(int(steps), m, n)
    P = np.arange(n)
    for j in range(steps):
        norms = np.sum(R[j:, j:] * R[j:, j:], axis=0)
        pj = j + int(np.argmax(norms))
        if pj != j:
            R[:, [j, pj]] = R[:, [pj, j]]
            P[[j, pj]] = P[[pj, j]]
        x = R[j:, j]
        nx = np.sqrt(np.dot(x, x))
        if nx == 0.0:
            continue
        alpha = -_sign(x[0]) * nx
        v = x.copy()
        v[0] -= alpha
        vtv = np.dot(v, v)
        w = v @ R[j:, j + 1:]
        R[j:, j + 1:] -= np.outer(v, w) * (2.0 / vtv)
        R[j + 1:, j] = 0.0
        R[j, j] = alpha
    return R, P


def lu_pp(Y):
    """Gaussian elimination with partial pivoting on Y (m x l, m >= l).

    Step j: the unpivoted row with the largest |y_ij| (first on ties) is the
    pivot p_j; every other unpivoted row i gets l_ij = y_ij / y_pj and
    y_i,c -= l_ij y_pj,c for c > j.  Returns L (m x l) with L[p_j, j] = 1,
    L[p_j, c] = 0 for c > j and the multipliers elsewhere (so Y = L U with U
    the pivot rows' upper triangle; L is unit lower triangular up to the row
    permutation), and the pivot rows.  A zero pivot column is skipped
    (multipliers 0)."""
    W = np.array(Y, dtype=np.float64)
    m, l = W.shape
    done = np.zeros(m, dtype=bool)
    piv = np.zeros(l, dtype=np.int64)
    L = np.zeros((m, l))
    for j in range(l):
        cand = np.where(~done)[0]
        p = cand[int(np.argmax(np.abs(W[cand, j])))]
        piv[j] = p
        done[p] = True
        L[p, j] = 1.0
        u = W[p, j]
        rest = np.where(~done)[0]
        if u == 0.0:
            continue
        lij = W[rest, j] / u
        L[rest, j] = lij
        W[np.ix_(rest, np.arange(j + 1, l))] -= np.outer(lij, W[p, j + 1:])
    return L, piv

"""Seeded synthetic inputs shaped like the paper's workloads (shared by tests,
bench and smoke; holds none of the method's arithmetic).

The five BASELINE.json configs:

  1  FP64 1000 x 500,  A = U diag(s) V^T, exact rank 10, s_i = 10^(-i/5),
     Haar U, V;                       k=10,  p=10, q=2, Gaussian Omega
  2  FP64 10000 x 5000, s_i = exp(-i/20) (r = 800 terms, the rest < 1e-17 s_1)
     + N(0, (1e-6)^2);                k=50,  p=10, q=2, Rademacher Omega
     (stands in for the paper's dense 10000 x 5000 test, Fig. 8)
  3  FP64 200000 x 4000, rank-200, s_i = 1/i, + N(0, (1e-3)^2), column-centred
     (randomized PCA);                k=100, p=20, q=2, uniform Omega
     (stands in for the tiger image / digits PCA workloads)
  4  FP32 1e6 x 1e4 (40 GB), rank-500, s_i = exp(-i/50), + N(0, (1e-4)^2);
                                      k=100, p=20, q=3, Gaussian Omega
  5  FP64 100000 x 1000, A = G1 G2^T + S: G1, G2 i.i.d. N(0,1) (rank 20),
     S 5% Bernoulli support, |S_ij| ~ U[5,10], random sign; rrpca with
     rsvd(k=20, p=10, q=2) per iteration, tol 1e-7
     (scaled-up analogue of the paper's synthetic RPCA study)

"N(0, x)" is read as standard deviation x (reading R13).  Haar
factors: QR of a Gaussian matrix with diag(R) > 0 (torch.linalg.qr is used as
a data-generation library call; it is not part of the method).  Data seed =
1000 + cfg; Omega seed = 2000 + cfg.
"""
import math

import torch

CONFIGS = {
    1: dict(name="cfg1_exact_rank_1000x500", m=1000, n=500, dtype="f64", k=10, p=10, q=2,
            sdist="normal", center=False, rank=10, spectrum="pow10", noise=0.0),
    2: dict(name="cfg2_dense_10000x5000", m=10000, n=5000, dtype="f64", k=50, p=10, q=2,
            sdist="rademacher", center=False, rank=800, spectrum="exp20", noise=1e-6),
    3: dict(name="cfg3_pca_200000x4000", m=200000, n=4000, dtype="f64", k=100, p=20, q=2,
            sdist="unif", center=True, rank=200, spectrum="inv", noise=1e-3),
    4: dict(name="cfg4_f32_1000000x10000", m=1000000, n=10000, dtype="f32", k=100, p=20, q=3,
            sdist="normal", center=False, rank=500, spectrum="exp50", noise=1e-4),
    5: dict(name="cfg5_rrpca_100000x1000", m=100000, n=1000, dtype="f64", k=20, p=10, q=2,
            sdist="normal", center=False, rank=20, spectrum=None, noise=0.0, rrpca=True,
            sparse_frac=0.05, sparse_lo=5.0, sparse_hi=10.0, tol=1e-7),
}


def spectrum(kind, r, dtype=torch.float64):
    i = torch.arange(1, r + 1, dtype=torch.float64)
    if kind == "pow10":
        s = 10.0 ** (-i / 5.0)
    elif kind == "exp20":
        s = torch.exp(-i / 20.0)
    elif kind == "exp50":
        s = torch.exp(-i / 50.0)
    elif kind == "inv":
        s = 1.0 / i
    else:
        raise ValueError(kind)
    return s.to(dtype)


def _gen(device, seed):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def haar(m, r, gen, device):
    """m x r matrix with orthonormal columns, Haar-distributed (QR with diag(R) > 0)."""
    G = torch.randn(m, r, generator=gen, device=device, dtype=torch.float64)
    Q, R = torch.linalg.qr(G)
    sgn = torch.sign(torch.diagonal(R))
    sgn[sgn == 0] = 1
    return Q * sgn[None, :]


def lowrank(m, n, s, noise=0.0, seed=0, device="cpu", dtype=torch.float64, chunk_rows=None):
    """A = U diag(s) V^T + noise * N(0,1) with Haar U (m x r), V (n x r); assembled
    in FP64 then rounded to ``dtype``.  Returns (A, s)."""
    s = torch.as_tensor(s, dtype=torch.float64, device=device)
    r = s.numel()
    g = _gen(device, seed)
    U = haar(m, r, g, device)
    V = haar(n, r, g, device)
    if chunk_rows is None:
        A = (U * s[None, :]) @ V.T
        if noise:
            A += noise * torch.randn(m, n, generator=g, device=device, dtype=torch.float64)
        return A.to(dtype), s
    A = torch.empty(m, n, dtype=dtype, device=device)
    Vs = (V * s[None, :]).T.contiguous()
    for r0 in range(0, m, chunk_rows):
        r1 = min(m, r0 + chunk_rows)
        blk = U[r0:r1] @ Vs
        if noise:
            blk += noise * torch.randn(r1 - r0, n, generator=g, device=device, dtype=torch.float64)
        A[r0:r1] = blk.to(dtype)
    return A, s


def sparse_plus_lowrank(m, n, rank=20, frac=0.05, lo=5.0, hi=10.0, seed=0, device="cpu"):
    """Config-5 construction (reading R16): L0 = G1 G2^T, S0 Bernoulli(frac) support,
    magnitudes U[lo, hi], signs +-1; returns (A, L0, S0)."""
    g = _gen(device, seed)
    G1 = torch.randn(m, rank, generator=g, device=device, dtype=torch.float64)
    G2 = torch.randn(n, rank, generator=g, device=device, dtype=torch.float64)
    L0 = G1 @ G2.T
    supp = torch.rand(m, n, generator=g, device=device, dtype=torch.float64) < frac
    mag = lo + (hi - lo) * torch.rand(m, n, generator=g, device=device, dtype=torch.float64)
    sgn = torch.where(torch.rand(m, n, generator=g, device=device, dtype=torch.float64) < 0.5, -1.0, 1.0)
    S0 = torch.where(supp, mag * sgn, torch.zeros((), dtype=torch.float64, device=device))
    return L0 + S0, L0, S0


def make_config(cfg, device="cpu", scale_rows=None):
    """Build config ``cfg``'s input A on ``device`` (optionally with fewer rows,
    for reduced-size tests).  Returns (A, meta) where meta carries the rsvd
    parameters and the planted ground truth."""
    c = dict(CONFIGS[cfg])
    m = c["m"] if scale_rows is None else scale_rows
    n = c["n"]
    seed = 1000 + cfg
    dtype = torch.float32 if c["dtype"] == "f32" else torch.float64
    meta = dict(c, m=m, seed_data=seed, seed_omega=2000 + cfg)
    if c.get("rrpca"):
        A, L0, S0 = sparse_plus_lowrank(m, n, c["rank"], c["sparse_frac"], c["sparse_lo"],
                                        c["sparse_hi"], seed=seed, device=device)
        meta.update(L0=L0, S0=S0)
        return A, meta
    r = min(c["rank"], n)
    s = spectrum(c["spectrum"], r)
    chunk = 65536 if m * n > 2e8 else None
    A, s = lowrank(m, n, s, c["noise"], seed=seed, device=device, dtype=dtype, chunk_rows=chunk)
    meta.update(s=s)
    return A, meta


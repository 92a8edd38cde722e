"""Random test matrix Omega from a counter-based generator (oracle side).

Paper: "we seek a matrix with independent identically distributed (i.i.d.)
entries from some distribution" -- Gaussian N(0,1), uniform U(-1,1) or
Rademacher +-1 (§2.3 "Random test matrices"; Alg. 4 step (2)
``Omega = rnorm(n, l)``).  The paper draws with R's RNG and fixes no
seed semantics; reading R1 fixes a counter spec (Philox4x32-10,
Salmon et al. SC'11) so the oracle and the GPU draw the *same* Omega:

  entry (i, j) of the n x l matrix, 0 <= i < n, 0 <= j < l:
    e       = j*n + i                                   (column-major counter)
    counter = (lo32(e), hi32(e), lo32(stream), hi32(stream))
    key     = (lo32(seed), hi32(seed))
    (w0,w1,w2,w3) = Philox4x32-10(counter, key)
    a = w1<<32 | w0 ;  b = w3<<32 | w2                  (uint64)
    U01(x) = (2*(x>>12) + 1) * 2^-53                    (exact, in (0,1))
    normal:     sqrt(-2 ln U01(a)) * cos(2 pi U01(b))
    unif:       2*U01(a) - 1
    rademacher: +1 if (a>>63) == 0 else -1

This module is written independently of the CUDA generator and is pinned
against cuRAND's ``curand_Philox4x32_10`` (tests/test_oracle_pins.py).
"""
import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint32(0x9E3779B9)
_W1 = np.uint32(0xBB67AE85)
_MASK32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)

SDIST = {"normal": 0, "unif": 1, "rademacher": 2}


def _mulhilo(m, x):
    prod = m * x.astype(np.uint64)
    return (prod & _MASK32).astype(np.uint32), (prod >> _S32).astype(np.uint32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds on uint32 arrays (Salmon et al., SC'11).

    One round: (lo0,hi0) = M0*c0, (lo1,hi1) = M1*c2,
    out = (hi1^c1^k0, lo1, hi0^c3^k1, lo0); the key is bumped by the Weyl
    constants (W0, W1) between rounds.
    """
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint32) for c in (c0, c1, c2, c3))
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    with np.errstate(over="ignore"):
        for r in range(10):
            lo0, hi0 = _mulhilo(_M0, c0)
            lo1, hi1 = _mulhilo(_M1, c2)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            if r < 9:
                k0 = np.uint32(k0 + _W0)
                k1 = np.uint32(k1 + _W1)
    return c0, c1, c2, c3


def u01(x):
    """U01(x) = (2*(x>>12)+1) * 2^-53 for uint64 x: exact in FP64, in (0,1)."""
    x = np.asarray(x, dtype=np.uint64)
    return ((x >> np.uint64(12)).astype(np.float64) * 2.0 + 1.0) * 2.0 ** -53


def omega_words(n, l, seed, stream):
    """The two uint64 words (a, b) for every entry, shaped (n, l)."""
    i = np.arange(n, dtype=np.uint64)[:, None]
    j = np.arange(l, dtype=np.uint64)[None, :]
    e = j * np.uint64(n) + i
    seed = np.uint64(seed)
    stream = np.uint64(stream)
    w0, w1, w2, w3 = philox4x32_10(
        (e & _MASK32).astype(np.uint32), (e >> _S32).astype(np.uint32),
        np.full(e.shape, np.uint32(int(stream) & 0xFFFFFFFF), dtype=np.uint32),
        np.full(e.shape, np.uint32(int(stream) >> 32), dtype=np.uint32),
        int(seed) & 0xFFFFFFFF, int(seed) >> 32)
    a = (w1.astype(np.uint64) << _S32) | w0.astype(np.uint64)
    b = (w3.astype(np.uint64) << _S32) | w2.astype(np.uint64)
    return a, b


def omega(n, l, sdist="normal", seed=0, stream=0, dtype=np.float64):
    """Omega (n x l) per the counter spec above.

    ``dtype=np.float32`` rounds each FP64 value to nearest FP32 (DESIGN.md
    reading R12); the result is returned upcast to float64 exactly.
    """
    if isinstance(sdist, str):
        sdist = SDIST[sdist]
    a, b = omega_words(n, l, seed, stream)
    if sdist == 0:
        val = np.sqrt(-2.0 * np.log(u01(a))) * np.cos(6.283185307179586 * u01(b))
    elif sdist == 1:
        val = 2.0 * u01(a) - 1.0
    elif sdist == 2:
        val = np.where((a >> np.uint64(63)) == 0, 1.0, -1.0)
    else:
        raise ValueError("sdist must be normal, unif or rademacher")
    if dtype == np.float32:
        val = val.astype(np.float32).astype(np.float64)
    return val

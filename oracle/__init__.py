"""CPU oracle for the randomized SVD hot path of arXiv 1608.02148 (rsvd package).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path may import this package:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
leg / ``--impl reference`` arm use it.  It shares no code with the CUDA path
(``paper_1608_02148_b200/csrc``): it has its own Philox4x32-10 generator written
from the counter spec (DESIGN.md §Ω), its own Householder QR and its own
one-sided Jacobi SVD (applied to B^T directly, a different derivation from the
GPU's QR(B^T)+Jacobi(R^T) route).

Precision: float64 throughout (the paper: "full double precision", PAPER.md:681,
§3.5).  FP32 inputs are upcast exactly; FP32-rounded Omega is upcast exactly.

Passages followed (PAPER.md line numbers, "P:n"):
  * Alg. 4 ``rqb``                 P:585-615 (§3.3)
  * Alg. 2 ``sub_iterations``      P:366-387 (§2.2.2)
  * Alg. 5 ``rsvd``                P:616-637, Eq. UQU
  * random test matrices          P:417-430 (§2.3)
  * ``rsvd()`` interface           P:706-724 (§3.6)
  * Alg. 6 ``rpca``                P:1336-1361, Eq. P:1322 (§4.2); loadings,
                                  whitening, explained variance P:1239-1302;
                                  predict() P:1570
  * Alg. 7 ``rrpca`` (IALM)        P:1655-1723 (§5.3)
  * Alg. id / rid / rcur           P:2059-2127, Alg. rcur P:1975-2010 (§6)

Pins: every function here is pinned by ``tests/test_oracle_pins.py`` against
closed forms, textbook special cases, an independent Philox implementation
(cuRAND's host-compiled ``curand_Philox4x32_10``) and brute force on tiny
inputs.  Parity unpinned: the paper's printed Table 1-3 numbers (their datasets
are not available), see DESIGN.md §Readings.
"""
from .philox import philox4x32_10, omega, u01
from .linalg import hqr, jacobi_svd_bt, qrcp, soft_threshold
from .rsvd import (oracle_rqb, oracle_rsvd, oracle_rpca, oracle_rpca_predict, oracle_rrpca, oracle_id, oracle_rid,
                   oracle_rcur, predict_rank, resolve_params, sign_fix)

__all__ = ["philox4x32_10", "omega", "u01", "hqr", "jacobi_svd_bt",
           "soft_threshold", "oracle_rqb", "oracle_rsvd", "oracle_rpca", "oracle_rpca_predict",
           "oracle_rrpca", "resolve_params", "sign_fix"]

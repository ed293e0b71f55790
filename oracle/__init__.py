"""CPU fp64 ORACLE for the sparse-aware truncated-SVD update of arXiv 2401.09703.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import anything under oracle/.  The product
path (paper_2401_09703_b200 + libtsvd.so) never imports it and shares no code with it:
no kernels, helpers, constants or pre/post-processing.  Only the seeded input
generators in synth/ (no method arithmetic) feed both sides.

What it computes: by Def 2 and Theorem 1
 every update returns SVD_k of the update applied to the
*maintained* approximation Ã = U_k Σ_k V_k^T.  The oracle reaches it the plain way,
with Zha–Simon's dense augmented projection (Eq (1), Eq (2)
PAPER.md:118-160): dense Householder QR (numpy.linalg.qr) of the densified augmented
matrix (I - U U^T) E and a dense LAPACK SVD (scipy gesdd) of the core.  It never uses
SV-LCOV, Cholesky-QR, deflation or the extended decomposition — those are the
method's, and live only in the CUDA path.

Modules
  zha_simon  exact add rows / add columns / update weights (dense Eq (1)/(2)).
  variants   dense GKL (Alg 5) and dense RPI (Alg 7)
             plus the App D.3 cores.
  svlcov     Def 1 / Lemma 2 tuple algebra, Alg 1 (dense MGS) and Alg 2 (SV-LCOV QR)
             written out step by step, for pinning Lemma 3 and the orthogonaliser's R.
  steps      plain definitions of the intermediate quantities of the path (lift,
             sparse Gram, Cholesky with deflation, cores) for kernel-level parity.
  metrics    parity metrics: sin of the largest principal angle (never via
             sqrt(1-cos^2)), relative singular-value error, gap guard.

Pins: tests/test_oracle_pins.py (-m "not gpu").  Every function here is pinned by
at least one check that does not re-run it (brute force, exactness, energy, worked
examples, closed forms); see DESIGN.md §"Oracle pins".
"""

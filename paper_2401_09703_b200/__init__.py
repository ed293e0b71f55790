"""B200-native sparse-aware truncated-SVD update (arXiv 2401.09703).

The product is libtsvd.so (C-ABI in include/tsvd.h, sm_100a CUDA in csrc/); this
package is its thin Python binding.  See DESIGN.md.
"""
from .tsvd import (  # noqa: F401
    EXACT, GKL, RPI, EXPORTED, LIB_PATH, TSVD, Sparse, TsvdError, make_opts, version,
    k_chol_deflate, k_dgemm, k_gather_spmm, k_inverse, k_jacobi_svd, k_materialize,
    k_scatter_add, k_sparse_gram, k_trsm_upper,
)

"""B200-native sparse-aware truncated-SVD update (arXiv 2401.09703).

The product is libtsvd.so (C-ABI in include/tsvd.h, sm_100a CUDA in csrc/); this
package is its thin Python binding.  See DESIGN.md.

The binding is loaded on first attribute access, so that `python -m
paper_2401_09703_b200.build` works before the library exists.  Accessing any name
without a built libtsvd.so raises ImportError: there is no CPU fallback.
"""
_NAMES = ("EXACT", "GKL", "RPI", "EXPORTED", "LIB_PATH", "TSVD", "Sparse", "TsvdError", "make_opts",
          "version", "k_chol_deflate", "k_dgemm", "k_gather_spmm", "k_inverse", "k_norm2_est", "k_jacobi_svd",
          "k_materialize", "k_scatter_add", "k_sparse_gram", "k_trsm_upper", "k_gaussian", "k_core_svd", "k_cholqr", "k_chol_rinv",
          "nccl_unique_id", "state_info", "shard_owner", "shard_split_host",
          "k_approx_basis", "dag_order", "dag_check")


def __getattr__(name):
    if name in _NAMES:
        from . import tsvd as _t
        return getattr(_t, name)
    raise AttributeError(name)


__all__ = list(_NAMES)

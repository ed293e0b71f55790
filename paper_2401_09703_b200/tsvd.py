"""Thin ctypes binding of libtsvd.so (include/tsvd.h, include/tsvd_kernels.h).

Argument marshalling only: every step of the update runs in the library's CUDA
kernels.  There is no Python or CPU fallback — if libtsvd.so is missing, importing
this module raises.  Arrays may be torch tensors (CUDA or CPU) or numpy arrays; the
library detects host vs device pointers itself (tsvd.h conventions).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSVD_LIB", os.path.join(_HERE, "libtsvd.so"))
if not os.path.exists(LIB_PATH):
    raise ImportError(f"libtsvd.so not found at {LIB_PATH}: build it with "
                      f"`python -m paper_2401_09703_b200.build` (there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

# ----------------------------------------------------------------------------- C types
STATUS = {0: "OK", 1: "E_SHAPE", 2: "E_NOT_ORTHONORMAL", 3: "E_BAD_SIGMA", 4: "E_NUMERIC",
          5: "E_SVD_FAIL", 6: "E_OOB", 7: "E_INVALID", 8: "E_OOM", 9: "E_CUDA", 10: "E_NCCL",
          11: "E_UNSUPPORTED", 12: "E_NOT_LOCAL", 13: "E_STATE_VERSION", 14: "E_IO"}
EXACT, GKL, RPI = 0, 1, 2
KERNEL_CLASSES = ("gather_spmm", "sparse_gram", "dgemm_dmma", "chol_panel", "small_chol", "core_jacobi",
                  "scatter_add", "approx_sparse")


class tsvd_opts(C.Structure):
    _fields_ = [("mode", C.c_int32), ("l", C.c_int32), ("t", C.c_int32), ("flags", C.c_int32),
                ("sketch", C.c_void_p), ("seed", C.c_uint64), ("reset_cond", C.c_double), ("defl_tol", C.c_double)]


class tsvd_sparse(C.Structure):
    _fields_ = [("s", C.c_int64), ("dim", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("val", C.c_void_p)]


class tsvd_stats(C.Structure):
    _fields_ = [("s", C.c_int64), ("nnz", C.c_int64), ("s_eff", C.c_int64), ("rank", C.c_int64 * 2), ("touched", C.c_int64 * 2),
                ("theta_next", C.c_double), ("energy", C.c_double), ("cond", C.c_double * 2),
                ("reset", C.c_int32 * 2), ("jacobi_sweeps", C.c_int32), ("core_iters", C.c_int32),
                ("core_path", C.c_int32), ("core_rows", C.c_int32),
                ("core_cols", C.c_int32), ("total_resets", C.c_int32), ("ms_pre", C.c_float),
                ("ms_svd", C.c_float), ("ms_post", C.c_float), ("ms_total", C.c_float),
                ("launches", C.c_int32), ("kern_ms", C.c_float * 8), ("kern_flops", C.c_double * 8),
                ("kern_bytes", C.c_double * 8), ("kern_launches", C.c_int32 * 8), ("top_class", C.c_int32),
                ("top_launches", C.c_int32), ("top_ms", C.c_float),
                ("top_flops", C.c_double), ("top_bytes", C.c_double)]

    def as_dict(self):
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            d[name] = list(v) if hasattr(v, "__len__") else v
        return d


class tsvd_shard_opts(C.Structure):
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("virtual_shards", C.c_int32), ("block", C.c_int32),
                ("nccl_id", C.c_void_p)]


_P = C.c_void_p
_SIGS = {
    "tsvd_create": (C.c_int, [C.POINTER(_P), C.c_int32, C.c_int64, C.c_int64, C.c_int32]),
    "tsvd_create_sharded": (C.c_int, [C.POINTER(_P), C.c_int32, C.POINTER(tsvd_shard_opts), C.c_int64, C.c_int64,
                                      C.c_int32]),
    "tsvd_nccl_unique_id": (C.c_int, [_P]),
    "tsvd_shard_owner": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    "tsvd_shard_split_host": (C.c_int, [C.POINTER(tsvd_sparse), C.c_int32, C.c_int32, C.c_int32, _P, _P, _P,
                                        C.POINTER(C.c_int64)]),
    "tsvd_destroy": (None, [_P]),
    "tsvd_last_error": (C.c_char_p, [_P]),
    "tsvd_version": (C.c_char_p, []),
    "tsvd_init": (C.c_int, [_P, C.c_int64, C.c_int64, _P, _P, _P, _P]),
    "tsvd_init_sparse": (C.c_int, [_P, C.POINTER(tsvd_sparse), C.c_int32, C.c_int32, C.c_uint64, _P]),
    "tsvd_update_rows": (C.c_int, [_P, C.POINTER(tsvd_sparse), C.POINTER(tsvd_opts), _P]),
    "tsvd_update_cols": (C.c_int, [_P, C.POINTER(tsvd_sparse), C.POINTER(tsvd_opts), _P]),
    "tsvd_update_weights": (C.c_int, [_P, C.POINTER(tsvd_sparse), C.POINTER(tsvd_sparse),
                                      C.POINTER(tsvd_opts), _P]),
    "tsvd_get_U": (C.c_int, [_P, _P, _P]),
    "tsvd_get_V": (C.c_int, [_P, _P, _P]),
    "tsvd_get_S": (C.c_int, [_P, _P, _P]),
    "tsvd_query_row": (C.c_int, [_P, C.c_int32, C.c_int64, _P, _P]),
    "tsvd_query_row_local": (C.c_int, [_P, C.c_int32, C.c_int64, _P, _P]),
    "tsvd_score_pairs": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P]),
    "tsvd_residual_fro": (C.c_int, [_P, C.POINTER(tsvd_sparse), _P, _P]),
    "tsvd_get_U_shard": (C.c_int, [_P, C.c_int32, _P, _P, C.POINTER(C.c_int64), _P]),
    "tsvd_get_V_shard": (C.c_int, [_P, C.c_int32, _P, _P, C.POINTER(C.c_int64), _P]),
    "tsvd_materialize": (C.c_int, [_P, _P]),
    "tsvd_dims": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "tsvd_last_stats": (C.c_int, [_P, C.POINTER(tsvd_stats)]),
    "tsvd_last_stats_nowait": (C.c_int, [_P, C.POINTER(tsvd_stats)]),
    "tsvd_reserve": (C.c_int, [_P, C.c_int64, _P]),
    "tsvd_dag_order": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32, _P, C.c_int64]),
    "tsvd_dag_check": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "tsvd_k_dgemm": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_double, _P,
                               C.c_int64, _P, C.c_int64, C.c_double, _P, C.c_int64, C.c_int32, _P]),
    "tsvd_k_gather_spmm": (C.c_int, [C.POINTER(tsvd_sparse), _P, C.c_int32, _P, _P]),
    "tsvd_k_sparse_gram": (C.c_int, [C.POINTER(tsvd_sparse), _P, _P]),
    "tsvd_k_chol_deflate": (C.c_int, [_P, C.c_int64, _P, C.c_double, _P, C.POINTER(C.c_int64), _P]),
    "tsvd_k_trsm_upper": (C.c_int, [_P, C.c_int64, _P, _P, C.c_int32, _P]),
    "tsvd_k_jacobi_svd": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int32, _P, _P, _P, C.POINTER(C.c_int32), _P]),
    "tsvd_k_cholqr": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int32, C.c_double, _P, _P]),
    "tsvd_save": (C.c_int, [_P, C.c_char_p, _P]),
    "tsvd_load": (C.c_int, [_P, C.c_char_p, _P]),
    "tsvd_state_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "tsvd_k_chol_rinv": (C.c_int, [_P, C.c_int64, _P, C.c_double, _P, _P, _P]),
    "tsvd_k_core_svd": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int32, _P, _P, _P, _P, _P]),
    "tsvd_k_inverse": (C.c_int, [_P, C.c_int32, _P, _P, _P]),
    "tsvd_k_norm2_est": (C.c_int, [_P, C.c_int32, _P, _P]),
    "tsvd_k_scatter_add": (C.c_int, [C.POINTER(tsvd_sparse), _P, C.c_int32, _P, _P]),
    "tsvd_k_materialize": (C.c_int, [_P, C.c_int64, C.c_int32, _P, _P]),
    "tsvd_k_gaussian": (C.c_int, [C.c_uint64, C.c_int32, C.c_int64, C.c_int64, _P, _P]),
    "tsvd_k_approx_basis": (C.c_int, [C.POINTER(tsvd_sparse), _P, C.c_int32, C.POINTER(tsvd_opts), C.c_int32,
                                      _P, _P, _P, _P]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


class TsvdError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {msg}")


# ----------------------------------------------------------------------------- helpers
def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr() if a.numel() else None
    if isinstance(a, np.ndarray):
        return a.ctypes.data if a.size else None
    raise TypeError(type(a))


def _stream(stream=None) -> Optional[int]:
    if stream is not None:
        return stream if isinstance(stream, int) else stream.cuda_stream
    try:
        import torch
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            return torch.cuda.current_stream().cuda_stream
    except ImportError:  # pragma: no cover
        pass
    return None


@dataclass
class Sparse:
    """s sparse update vectors of length dim as CSR rows (tsvd_sparse).  Arrays are
    numpy (host) or torch (host or CUDA): int64 row_ptr, int32 col_idx, float64 val."""
    s: int
    dim: int
    row_ptr: object
    col_idx: object
    val: object

    @property
    def nnz(self) -> int:
        return int(len(self.col_idx))

    @classmethod
    def from_scipy(cls, A, device=None, pin=False):
        A = A.tocsr()
        rp = np.ascontiguousarray(A.indptr, dtype=np.int64)
        ci = np.ascontiguousarray(A.indices, dtype=np.int32)
        v = np.ascontiguousarray(A.data, dtype=np.float64)
        if device is not None or pin:
            import torch
            rp, ci, v = (torch.from_numpy(x) for x in (rp, ci, v))
            if pin:
                rp, ci, v = rp.pin_memory(), ci.pin_memory(), v.pin_memory()
            if device is not None:
                rp, ci, v = rp.to(device), ci.to(device), v.to(device)
        return cls(A.shape[0], A.shape[1], rp, ci, v)

    def c(self) -> tsvd_sparse:
        return tsvd_sparse(self.s, self.dim, self.nnz, _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(self.val))


def make_opts(mode=EXACT, l=10, t=3, sketch=None, seed=0, reset_cond=1e4, defl_tol=1e-12, flags=0) -> tsvd_opts:
    """tsvd_opts (include/tsvd.h).  Keep `sketch` alive while the options are in use."""
    o = tsvd_opts(mode, l, t, flags, _ptr(sketch), seed, reset_cond, defl_tol)
    o._keep = sketch
    return o


def state_info(path: str):
    """(k, m, n) from a state file's header (no context, no GPU)."""
    k, m, n = C.c_int32(), C.c_int64(), C.c_int64()
    _k(_lib.tsvd_state_info(os.fsencode(path), C.byref(k), C.byref(m), C.byref(n)), "state_info")
    return k.value, m.value, n.value


def version() -> str:
    return _lib.tsvd_version().decode()


# ----------------------------------------------------------------------------- the data structure
def _nccl_env():
    # single-node bootstrap over loopback (the box's other interfaces may refuse connections);
    # set before NCCL reads it, overridable by the caller's environment
    os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for a NCCL-sharded context (call on rank 0, share the bytes)."""
    _nccl_env()
    buf = C.create_string_buffer(128)
    _k(_lib.tsvd_nccl_unique_id(buf), "nccl_unique_id")
    return buf.raw


def shard_owner(i: int, world: int, block: int):
    g, li = C.c_int32(), C.c_int64()
    _k(_lib.tsvd_shard_owner(i, world, block, C.byref(g), C.byref(li)), "shard_owner")
    return g.value, li.value


def shard_split_host(E: "Sparse", world: int, block: int, shard: int):
    """Host CSR split of E by the owner of its columns (tsvd_shard_split_host)."""
    e = E.c()
    nnz = C.c_int64()
    _k(_lib.tsvd_shard_split_host(C.byref(e), world, block, shard, None, None, None, C.byref(nnz)), "split")
    rp = np.empty(E.s + 1, np.int64)
    ci = np.empty(max(nnz.value, 1), np.int32)
    v = np.empty(max(nnz.value, 1), np.float64)
    _k(_lib.tsvd_shard_split_host(C.byref(e), world, block, shard, rp.ctypes.data, ci.ctypes.data, v.ctypes.data,
                                  C.byref(nnz)), "split")
    return rp, ci[:nnz.value], v[:nnz.value]


class TSVD:
    """Theorem 1's data structure on one GPU, optionally row-sharded:
    shard=dict(world=W, rank=r, nccl_id=bytes) (NCCL mode, one process per GPU) or
    shard=dict(world=W, virtual=True) (all W shards on this GPU)."""

    def __init__(self, k: int, m_capacity: int = 0, n_capacity: int = 0, device: int = 0, shard=None):
        h = _P()
        if shard is None:
            st = _lib.tsvd_create(C.byref(h), device, m_capacity, n_capacity, k)
        else:
            W = int(shard["world"])
            virt = bool(shard.get("virtual", False))
            self._id = C.create_string_buffer(shard["nccl_id"], 128) if shard.get("nccl_id") else None
            if self._id is not None:
                _nccl_env()
            so = tsvd_shard_opts(W, int(shard.get("rank", 0)), W if virt else 1, int(shard.get("block", 0)),
                                 C.cast(self._id, C.c_void_p) if self._id is not None else None)
            st = _lib.tsvd_create_sharded(C.byref(h), device, C.byref(so), m_capacity, n_capacity, k)
        if st:
            raise TsvdError(st, "tsvd_create: " + (_lib.tsvd_last_error(None) or b"").decode())
        self._h = h
        self.k = k
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            _lib.tsvd_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what):
        if st:
            raise TsvdError(st, f"{what}: {_lib.tsvd_last_error(self._h).decode()}")

    def init(self, U, S, V, stream=None):
        m, n = U.shape[0], V.shape[0]
        self._check(_lib.tsvd_init(self._h, m, n, _ptr(U), _ptr(S), _ptr(V), _stream(stream)), "init")

    def init_sparse(self, A: Sparse, oversample: int = 32, power_iters: int = 2, seed: int = 0, stream=None):
        """Initial truncated SVD of the sparse A computed on the GPU (tsvd_init_sparse)."""
        a = A.c()
        self._check(_lib.tsvd_init_sparse(self._h, C.byref(a), oversample, power_iters, seed, _stream(stream)),
                    "init_sparse")

    def update_rows(self, Er: Sparse, opts: Optional[tsvd_opts] = None, stream=None):
        e = Er.c()
        self._check(_lib.tsvd_update_rows(self._h, C.byref(e), C.byref(opts) if opts else None, _stream(stream)),
                    "update_rows")

    def update_cols(self, EcT: Sparse, opts: Optional[tsvd_opts] = None, stream=None):
        e = EcT.c()
        self._check(_lib.tsvd_update_cols(self._h, C.byref(e), C.byref(opts) if opts else None, _stream(stream)),
                    "update_cols")

    def update_weights(self, DT: Sparse, EmT: Sparse, opts: Optional[tsvd_opts] = None, stream=None):
        d, e = DT.c(), EmT.c()
        self._check(_lib.tsvd_update_weights(self._h, C.byref(d), C.byref(e), C.byref(opts) if opts else None,
                                             _stream(stream)), "update_weights")

    def update(self, kind: str, E: Sparse, D: Optional[Sparse] = None, opts=None, stream=None):
        if kind == "rows":
            return self.update_rows(E, opts, stream)
        if kind == "cols":
            return self.update_cols(E, opts, stream)
        return self.update_weights(D, E, opts, stream)

    def dims(self):
        m, n, k = C.c_int64(), C.c_int64(), C.c_int32()
        _lib.tsvd_dims(self._h, C.byref(m), C.byref(n), C.byref(k))
        return m.value, n.value, k.value

    def get_U(self, out=None, stream=None):
        m, _, k = self.dims()
        out = np.empty((m, k)) if out is None else out
        self._check(_lib.tsvd_get_U(self._h, _ptr(out), _stream(stream)), "get_U")
        return out

    def get_V(self, out=None, stream=None):
        _, n, k = self.dims()
        out = np.empty((n, k)) if out is None else out
        self._check(_lib.tsvd_get_V(self._h, _ptr(out), _stream(stream)), "get_V")
        return out

    def get_S(self, out=None, stream=None):
        out = np.empty(self.k) if out is None else out
        self._check(_lib.tsvd_get_S(self._h, _ptr(out), _stream(stream)), "get_S")
        return out

    def query_row(self, side: int, i: int, out=None, stream=None):
        out = np.empty(self.k) if out is None else out
        self._check(_lib.tsvd_query_row(self._h, side, i, _ptr(out), _stream(stream)), "query_row")
        return out

    def query_row_local(self, side: int, i: int, out=None, stream=None):
        """Row i of U / V computed by this process alone; TsvdError(E_NOT_LOCAL) if another
        process's shard owns it."""
        out = np.empty(self.k) if out is None else out
        self._check(_lib.tsvd_query_row_local(self._h, side, i, _ptr(out), _stream(stream)), "query_row_local")
        return out

    def get_shard(self, side: int, local_shard: int = 0, out=None, stream=None):
        """(rows, global_row_ids) of the U (side 0) or V (side 1) rows held by a local shard."""
        fn = _lib.tsvd_get_U_shard if side == 0 else _lib.tsvd_get_V_shard
        nr = C.c_int64()
        self._check(fn(self._h, local_shard, None, None, C.byref(nr), _stream(stream)), "get_shard")
        ids = np.empty(max(nr.value, 1), np.int64)
        out = np.empty((nr.value, self.k)) if out is None else out
        self._check(fn(self._h, local_shard, _ptr(out), ids.ctypes.data, C.byref(nr), _stream(stream)), "get_shard")
        return out, ids[:nr.value]

    def score_pairs(self, rows, cols, out=None, stream=None):
        """Ã[rows[p], cols[p]] = U[i] Σ V[j]^T for each pair (tsvd_score_pairs)."""
        rows = np.ascontiguousarray(rows, dtype=np.int64) if isinstance(rows, (list, np.ndarray)) else rows
        cols = np.ascontiguousarray(cols, dtype=np.int64) if isinstance(cols, (list, np.ndarray)) else cols
        n = len(rows)
        out = np.empty(n) if out is None else out
        self._check(_lib.tsvd_score_pairs(self._h, n, _ptr(rows), _ptr(cols), _ptr(out), _stream(stream)),
                    "score_pairs")
        return out

    def residual_fro(self, A: Sparse, stream=None):
        """(||A - Ã||_F, <A, Ã>, ||A||_F^2) for a sparse A with m rows (tsvd_residual_fro)."""
        a = A.c()
        out = np.zeros(3)
        self._check(_lib.tsvd_residual_fro(self._h, C.byref(a), out.ctypes.data, _stream(stream)), "residual_fro")
        return tuple(out)

    def save(self, path: str, stream=None):
        """Write the state (U', U'', Sigma, V', V'') to `path` atomically (tsvd.h "State persistence")."""
        self._check(_lib.tsvd_save(self._h, os.fsencode(path), _stream(stream)), "save")

    def load(self, path: str, stream=None):
        """Replace this context's state with the file's (same k)."""
        self._check(_lib.tsvd_load(self._h, os.fsencode(path), _stream(stream)), "load")

    @classmethod
    def from_file(cls, path: str, device: int = 0, m_capacity: int = 0, n_capacity: int = 0, stream=None):
        """A new context holding the state saved in `path` (capacities at least the file's dims)."""
        k, m, n = state_info(path)
        t = cls(k, m_capacity=max(m, m_capacity), n_capacity=max(n, n_capacity), device=device)
        t.load(path, stream=stream)
        return t

    def materialize(self, stream=None):
        self._check(_lib.tsvd_materialize(self._h, _stream(stream)), "materialize")

    def reserve(self, nbytes: int, stream=None):
        """Pre-grow the stream-ordered scratch pool (tsvd_reserve)."""
        self._check(_lib.tsvd_reserve(self._h, int(nbytes), _stream(stream)), "reserve")

    def stats(self, wait: bool = True) -> dict:
        """Statistics of the last update (tsvd_last_stats; wait=False: tsvd_last_stats_nowait,
        no device synchronisation, phase times possibly stale)."""
        s = tsvd_stats()
        (_lib.tsvd_last_stats if wait else _lib.tsvd_last_stats_nowait)(self._h, C.byref(s))
        return s.as_dict()


# ----------------------------------------------------------------------------- step-level entry points
def _k(st, what):
    if st:
        raise TsvdError(st, what)


def k_dgemm(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, Cm, ldc, uplo=0, stream=None):
    _k(_lib.tsvd_k_dgemm(int(transA), int(transB), M, N, K, alpha, _ptr(A), lda, _ptr(B), ldb, beta, _ptr(Cm), ldc,
                         uplo, _stream(stream)), "k_dgemm")


def k_gather_spmm(E: Sparse, X, k, W, stream=None):
    e = E.c()
    _k(_lib.tsvd_k_gather_spmm(C.byref(e), _ptr(X), k, _ptr(W), _stream(stream)), "k_gather_spmm")


def k_sparse_gram(E: Sparse, G, stream=None):
    e = E.c()
    _k(_lib.tsvd_k_sparse_gram(C.byref(e), _ptr(G), _stream(stream)), "k_sparse_gram")


def k_chol_deflate(G, s, enorm2, tau, keep, stream=None) -> int:
    r = C.c_int64()
    _k(_lib.tsvd_k_chol_deflate(_ptr(G), s, _ptr(enorm2), tau, _ptr(keep), C.byref(r), _stream(stream)),
       "k_chol_deflate")
    return r.value


def k_trsm_upper(R, s, keep, X, k, stream=None):
    _k(_lib.tsvd_k_trsm_upper(_ptr(R), s, _ptr(keep), _ptr(X), k, _stream(stream)), "k_trsm_upper")


def k_jacobi_svd(K, m, n, kk, theta, F, G, stream=None) -> int:
    sw = C.c_int32()
    _k(_lib.tsvd_k_jacobi_svd(_ptr(K), m, n, kk, _ptr(theta), _ptr(F), _ptr(G), C.byref(sw), _stream(stream)),
       "k_jacobi_svd")
    return sw.value


def k_cholqr(X, rows, l, passes=2, tau=1e-14, R=None, stream=None):
    _k(_lib.tsvd_k_cholqr(_ptr(X), rows, l, passes, tau, _ptr(R), _stream(stream)), "k_cholqr")


def k_chol_rinv(G, l, en, tau, keep, T, stream=None):
    _k(_lib.tsvd_k_chol_rinv(_ptr(G), l, _ptr(en), tau, _ptr(keep), _ptr(T), _stream(stream)), "k_chol_rinv")


def k_core_svd(K, m, n, kk, theta, F, G, stream=None):
    info = np.zeros(4)
    _k(_lib.tsvd_k_core_svd(_ptr(K), m, n, kk, _ptr(theta), _ptr(F), _ptr(G), info.ctypes.data, _stream(stream)),
       "k_core_svd")
    return dict(path=int(info[0]), iters=int(info[1]), sweeps=int(info[2]), energy=float(info[3]))


def k_inverse(M, k, Minv, cond, stream=None):
    _k(_lib.tsvd_k_inverse(_ptr(M), k, _ptr(Minv), _ptr(cond), _stream(stream)), "k_inverse")


def k_norm2_est(M, k, out, stream=None):
    _k(_lib.tsvd_k_norm2_est(_ptr(M), k, _ptr(out), _stream(stream)), "k_norm2_est")


def k_scatter_add(E: Sparse, Z, k, X, stream=None):
    e = E.c()
    _k(_lib.tsvd_k_scatter_add(C.byref(e), _ptr(Z), k, _ptr(X), _stream(stream)), "k_scatter_add")


def k_materialize(X, rows, k, M, stream=None):
    _k(_lib.tsvd_k_materialize(_ptr(X), rows, k, _ptr(M), _stream(stream)), "k_materialize")


def k_gaussian(seed, side, s, l, out, stream=None):
    _k(_lib.tsvd_k_gaussian(seed, side, s, l, _ptr(out), _stream(stream)), "k_gaussian")


def k_approx_basis(E: Sparse, X, k, opts, side, BJfull, Cp, Pm, stream=None):
    e = E.c()
    _k(_lib.tsvd_k_approx_basis(C.byref(e), _ptr(X), k, C.byref(opts), side, _ptr(BJfull), _ptr(Cp), _ptr(Pm),
                                _stream(stream)), "k_approx_basis")


def dag_order(kind: int, nt: int, nkb: int = 1):
    """Host task order of the tile-DAG kernels (tsvd_dag_order): list of (type, q, i, c)."""
    n = _lib.tsvd_dag_order(kind, nt, nkb, None, 0)
    if n < 0:
        raise ValueError("tsvd_dag_order: invalid arguments")
    buf = (C.c_int32 * (4 * n))()
    _lib.tsvd_dag_order(kind, nt, nkb, C.cast(buf, C.c_void_p), n)
    return [tuple(buf[4 * i:4 * i + 4]) for i in range(n)]


def dag_check(kind: int, nt: int, nkb: int = 1) -> int:
    """Mismatches between the device task generator and the host order (tsvd_dag_check)."""
    return int(_lib.tsvd_dag_check(kind, nt, nkb))


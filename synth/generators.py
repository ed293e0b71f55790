"""Seeded generators for the BASELINE.json configs (SURVEY.md §8(d) table "Synthetic inputs").

Every function is deterministic in its seed.  Sparse matrices are scipy CSR (scipy's own
index dtypes; paper_2401_09703_b200.Sparse.from_scipy converts to the C-ABI's int64 row
pointers / int32 column indices) with float64 values, rows sorted, no duplicates, no
explicit zeros.  An update batch is always handed over as *s sparse
update vectors stored as CSR rows* (the C-ABI's tsvd_sparse, include/tsvd.h):

  kind "rows"    : E_r            (s x n)   PAPER.md:53-56, Alg 9
  kind "cols"    : E_c^T          (s x m)   PAPER.md:53-58, Alg 3
  kind "weights" : D^T (s x m) and E_m^T (s x n), A + D E_m^T   PAPER.md:60, Alg 4
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import scipy.sparse as sp


# --------------------------------------------------------------------------- containers
@dataclass
class Batch:
    kind: str                      # "rows" | "cols" | "weights"
    E: sp.csr_matrix               # rows: E_r; cols: E_c^T; weights: E_m^T
    D: Optional[sp.csr_matrix] = None   # weights only: D^T (s x m)

    @property
    def s(self) -> int:
        return self.E.shape[0]

    @property
    def nnz(self) -> int:
        return int(self.E.nnz + (self.D.nnz if self.D is not None else 0))


@dataclass
class Workload:
    name: str
    k: int
    U0: np.ndarray
    S0: np.ndarray
    V0: np.ndarray
    batches: List[Batch]
    meta: dict = field(default_factory=dict)

    @property
    def m0(self) -> int:
        return self.U0.shape[0]

    @property
    def n0(self) -> int:
        return self.V0.shape[0]

    def final_dims(self):
        m, n = self.m0, self.n0
        for b in self.batches:
            if b.kind == "rows":
                m += b.s
            elif b.kind == "cols":
                n += b.s
        return m, n


def _csr(A) -> sp.csr_matrix:
    A = sp.csr_matrix(A, dtype=np.float64)
    A.sum_duplicates()
    A.eliminate_zeros()
    A.sort_indices()
    return A


# --------------------------------------------------------------------------- small helpers
def random_orthonormal(n: int, k: int, seed: int) -> np.ndarray:
    """n x k matrix with orthonormal columns (QR of a Gaussian matrix)."""
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.standard_normal((n, k)))
    return q * np.sign(np.diag(r))


def random_sparse(rows: int, cols: int, density: float, seed: int, values="uniform") -> sp.csr_matrix:
    rng = np.random.default_rng(seed)
    nnz = int(round(density * rows * cols))
    cells = rng.choice(rows * cols, size=nnz, replace=False) if nnz else np.zeros(0, np.int64)
    r, c = np.divmod(cells, cols)
    if values == "uniform":
        v = rng.uniform(0.0, 1.0, size=nnz)
    elif values == "normal":
        v = rng.standard_normal(nnz)
    else:
        v = np.ones(nnz)
    return _csr(sp.coo_matrix((v, (r, c)), shape=(rows, cols)))


def gaussian_sketch(seed: int, s: int, l: int) -> np.ndarray:
    """s x l standard-normal sketch Omega for RPI. Row-major."""
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(rng.standard_normal((s, l)))


def unit_vector(seed: int, s: int) -> np.ndarray:
    """Unit-norm start vector p1 for GKL ('Choose p1, ||p1|| = 1')."""
    rng = np.random.default_rng(seed)
    p = rng.standard_normal(s)
    return p / np.linalg.norm(p)


def _par_matmul(A, X, threads: int = 0):
    """A @ X for a scipy CSR A and dense X, row blocks on a thread pool (scipy's sparse
    product runs single-threaded and releases the GIL).  Harness plumbing only."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    m = A.shape[0]
    nt = threads or min(os.cpu_count() or 1, 32)
    if nt <= 1 or m < 100_000:
        return np.asarray(A @ X)
    step = (m + 4 * nt - 1) // (4 * nt)
    blocks = [(i, min(m, i + step)) for i in range(0, m, step)]
    out = np.empty((m, X.shape[1]))

    def one(b):
        out[b[0]:b[1]] = A[b[0]:b[1]] @ X

    with ThreadPoolExecutor(nt) as ex:
        list(ex.map(one, blocks))
    return out


def _orth(Y, want_r: bool = False):
    """Orthonormal basis of range(Y) for the harness's randomized SVD: Householder QR for
    small Y, Cholesky-QR2 (Gram, Cholesky, multiply by the triangular inverse — BLAS-3,
    fast on tall Y) for tall ones, falling back to Householder QR when the Gram is not
    positive definite.  want_r: also return R with Y = Q R."""
    import scipy.linalg as sla
    if Y.shape[0] >= 200_000:
        Q, Rt = Y, np.eye(Y.shape[1])
        for _ in range(2):
            try:
                R = sla.cholesky(Q.T @ Q, lower=False)
            except np.linalg.LinAlgError:
                break
            Q = Q @ sla.solve_triangular(R, np.eye(R.shape[0]), lower=False)
            Rt = R @ Rt
        else:
            Q = np.ascontiguousarray(Q)
            return (Q, Rt) if want_r else Q
    Q, R = np.linalg.qr(Y)
    return (Q, R) if want_r else Q


def init_truncated_svd(A, k: int, seed: int = 0, method: str = "auto", power_iters: int = 6):
    """Initial rank-k truncated SVD the stream starts from (harness work).

    dense LAPACK for small A, randomized subspace iteration otherwise.  Def 2
     makes the update result depend only on the (U, S, V) given,
    so this only has to return orthonormal U, V and a descending S >= 0."""
    m, n = A.shape
    if method == "auto":
        method = "dense" if m * n <= 4_000_000 else "randomized"
    if method == "dense":
        Ad = A.toarray() if sp.issparse(A) else np.asarray(A, dtype=np.float64)
        u, s, vt = np.linalg.svd(Ad, full_matrices=False)
        U, S, V = u[:, :k], s[:k], vt[:k].T
    else:
        rng = np.random.default_rng(seed)
        A = sp.csr_matrix(A)
        At = A.T.tocsr()
        p = min(k + 16, min(m, n))
        Y = _par_matmul(A, rng.standard_normal((n, p)))
        Q = _orth(Y)
        for _ in range(power_iters):
            Z = _orth(_par_matmul(At, Q))
            Q = _orth(_par_matmul(A, Z))
        # Q^T A = (A^T Q)^T = (Qb Rb)^T; Rb = u s vt gives A ~ (Q vt^T) s (Qb u)^T
        Qb, Rb = _orth(_par_matmul(At, Q), want_r=True)
        u, s, vt = np.linalg.svd(Rb)
        U = Q @ vt[:k].T
        S = s[:k]
        V = Qb @ u[:, :k]
    return (np.ascontiguousarray(U, dtype=np.float64), np.ascontiguousarray(S, dtype=np.float64),
            np.ascontiguousarray(V, dtype=np.float64))


# --------------------------------------------------------------------------- C1
def tiny_rowappend(seed: int = 1, m: int = 2000, n: int = 1000, nnz: int = 10_000, k: int = 16,
                   m_init: int = 1000, batch: int = 100, n_batches: int = 10) -> Workload:
    """BASELINE.json configs[0]: 2000 x 1000, i.i.d. uniform positions at 0.5 % density
    (exactly nnz cells drawn without replacement), values U(0,1), k = 16; SVD_16 of the
    first 1000 rows (LAPACK), then 10 batches of 100 appended rows."""
    A = random_sparse(m, n, nnz / (m * n), seed)
    U0, S0, V0 = init_truncated_svd(A[:m_init], k, method="dense")
    batches = [Batch("rows", _csr(A[m_init + b * batch: m_init + (b + 1) * batch]))
               for b in range(n_batches)]
    return Workload("C1-tiny-rowappend", k, U0, S0, V0, batches,
                    meta=dict(m=m, n=n, nnz=A.nnz, seed=seed))


# --------------------------------------------------------------------------- Chung-Lu
def _sample_sorted_cdf(rng, cdf, M):
    """M i.i.d. draws from the discrete distribution with cumulative weights cdf, via
    sorted uniforms (normalised exponential spacings — no sort) and a merge-like
    searchsorted, then a random permutation (i.i.d. order)."""
    u = np.cumsum(rng.exponential(size=M + 1))
    u = u[:-1] / u[-1]
    return rng.permutation(np.searchsorted(cdf, u))


def chung_lu(N: int, avg_deg: float, beta: float, seed: int, calib_rounds: int = 4) -> sp.csr_matrix:
    """Symmetric 0/1 Chung-Lu power-law adjacency (SURVEY §8(d) C2/C4 recipe): weights
    w_i ∝ i^(-1/(beta-1)); M endpoint pairs drawn i.i.d. ∝ w; self-loops and duplicates
    dropped; symmetrised; M calibrated so the realised mean degree is avg_deg; then a
    seeded random node permutation."""
    rng = np.random.default_rng(seed)
    w = np.arange(1, N + 1, dtype=np.float64) ** (-1.0 / (beta - 1.0))
    p = w / w.sum()
    cdf = np.cumsum(p)
    cdf[-1] = 1.0
    M = int(N * avg_deg / 2)
    U = None
    for _ in range(calib_rounds):
        r = _sample_sorted_cdf(rng, cdf, M)
        c = _sample_sorted_cdf(rng, cdf, M)
        keep = r != c
        r, c = r[keep], c[keep]
        lo, hi = np.minimum(r, c), np.maximum(r, c)
        # duplicates merged by the CSR conversion (upper triangle, one entry per edge)
        U = sp.csr_matrix((np.ones(len(lo)), (lo, hi)), shape=(N, N))
        U.sum_duplicates()
        deg = 2.0 * U.nnz / N
        if abs(deg - avg_deg) <= 0.02 * avg_deg:
            break
        M = int(M * avg_deg / max(deg, 1e-9))
    U.sort_indices()
    coo = U.tocoo()
    perm = rng.permutation(N)
    lo, hi = perm[coo.row], perm[coo.col]
    rows = np.concatenate([lo, hi])
    cols = np.concatenate([hi, lo])
    return _csr(sp.coo_matrix((np.ones(len(rows)), (rows, cols)), shape=(N, N)))


def graph_nodeappend(seed: int = 2, N: int = 100_000, avg_deg: float = 10.0, beta: float = 2.1,
                     k: int = 64, n_init: int = 50_000, batch: int = 5_000, n_batches: int = 10) -> Workload:
    """BASELINE.json configs[1]: Chung-Lu graph, SVD_64 of A[:n_init, :n_init], then
    per batch a row update A[c:c+b, :c] followed by a column update A[:c+b, c:c+b]
    (rows-then-columns)."""
    A = chung_lu(N, avg_deg, beta, seed)
    U0, S0, V0 = init_truncated_svd(A[:n_init, :n_init], k, seed=seed + 100)
    batches = []
    for b in range(n_batches):
        c = n_init + b * batch
        batches.append(Batch("rows", _csr(A[c:c + batch, :c])))
        # E_c^T = A[:c+b, c:c+b]^T = A[c:c+b, :c+b] (A symmetric)
        batches.append(Batch("cols", _csr(A[c:c + batch, :c + batch])))
    return Workload("C2-graph-nodeappend", k, U0, S0, V0, batches,
                    meta=dict(N=N, avg_deg=avg_deg, beta=beta, nnz=A.nnz, seed=seed))


# --------------------------------------------------------------------------- C3
def ratings_matrix(users: int, items: int, nnz: int, seed: int, zipf: float = 1.0,
                   mu: float = 4.0, sigma: float = 1.0) -> sp.csr_matrix:
    """User x item ratings: activity a_u ∝ LogNormal(mu, sigma) rescaled
    to sum nnz, clipped to [1, items]; items per user drawn without replacement ∝
    Zipf(zipf) over a seeded item permutation; values uniform on {0.5, 1.0, ..., 5.0}."""
    rng = np.random.default_rng(seed)
    a = rng.lognormal(mu, sigma, size=users)
    a = np.clip(np.round(a * nnz / a.sum()), 1, items).astype(np.int64)
    perm = rng.permutation(items)
    pop = np.empty(items)
    pop[perm] = np.arange(1, items + 1, dtype=np.float64) ** (-zipf)
    g = np.log(pop)
    indptr = np.zeros(users + 1, np.int64)
    indptr[1:] = np.cumsum(a)
    cols = np.empty(indptr[-1], np.int32)
    # Gumbel-top-a sampling without replacement, in user chunks
    order = np.argsort(-a, kind="stable")
    chunk = 256
    for c0 in range(0, users, chunk):
        us = order[c0:c0 + chunk]
        keys = g[None, :] + rng.gumbel(size=(len(us), items))
        for t, u in enumerate(us):
            au = a[u]
            sel = np.argpartition(-keys[t], au - 1)[:au] if au < items else np.arange(items)
            cols[indptr[u]:indptr[u + 1]] = np.sort(sel)
    vals = rng.integers(1, 11, size=indptr[-1]) * 0.5
    return _csr(sp.csr_matrix((vals, cols, indptr), shape=(users, items)))


def ratings_rowappend(seed: int = 3, users: int = 70_000, items: int = 10_000, nnz: int = 10_000_000,
                      k: int = 64, u_init: int = 35_000, batch: int = 3_500, n_batches: int = 10) -> Workload:
    """BASELINE.json configs[2]: SVD_64 of the first 35k users, then 10 x 3.5k users appended."""
    A = ratings_matrix(users, items, nnz, seed)
    U0, S0, V0 = init_truncated_svd(A[:u_init], k, seed=seed + 100)
    batches = [Batch("rows", _csr(A[u_init + b * batch: u_init + (b + 1) * batch]))
               for b in range(n_batches)]
    return Workload("C3-ratings-rowappend", k, U0, S0, V0, batches,
                    meta=dict(users=users, items=items, nnz=A.nnz, seed=seed))


# --------------------------------------------------------------------------- C4
def weights_rpi(seed: int = 4, N: int = 1_000_000, avg_deg: float = 20.0, beta: float = 2.1,
                k: int = 128, changes: int = 100_000, n_batches: int = 10) -> Workload:
    """BASELINE.json configs[3]: weight updates A + D E^T on a Chung-Lu graph.  Per batch
    changes/2 deletions (uniform over current edges) and changes/2 insertions (endpoints
    ∝ w, rejecting existing edges / self-loops), applied symmetrically as ΔA (±1);
    D = one-hot columns of the distinct touched rows R, E = ΔA[R, :]^T."""
    rng = np.random.default_rng(seed + 7)
    A = chung_lu(N, avg_deg, beta, seed)
    U0, S0, V0 = init_truncated_svd(A, k, seed=seed + 100, method="randomized", power_iters=3)
    w = np.arange(1, N + 1, dtype=np.float64) ** (-1.0 / (beta - 1.0))
    cdf = np.cumsum(w / w.sum())
    cdf[-1] = 1.0
    cur = sp.triu(A, k=1).tocoo()
    edges = set(zip(cur.row.tolist(), cur.col.tolist())) if N <= 20_000 else None
    elist_r, elist_c = cur.row.astype(np.int64), cur.col.astype(np.int64)
    batches = []
    for _ in range(n_batches):
        nd = changes // 2
        di = rng.choice(len(elist_r), size=min(nd, len(elist_r)), replace=False)
        dr, dc = elist_r[di], elist_c[di]
        ir = np.searchsorted(cdf, rng.random(nd * 2))
        ic = np.searchsorted(cdf, rng.random(nd * 2))
        ok = ir != ic
        ir, ic = np.minimum(ir[ok], ic[ok]), np.maximum(ir[ok], ic[ok])
        existing = A[ir, ic].A1 != 0 if edges is None else np.array([(a, b) in edges for a, b in zip(ir, ic)])
        key = ir * N + ic
        _, first = np.unique(key, return_index=True)
        keep = np.zeros(len(ir), bool)
        keep[first] = True
        keep &= ~existing
        ir, ic = ir[keep][:nd], ic[keep][:nd]
        r = np.concatenate([dr, dc, ir, ic])
        c = np.concatenate([dc, dr, ic, ir])
        v = np.concatenate([-np.ones(2 * len(dr)), np.ones(2 * len(ir))])
        dA = _csr(sp.coo_matrix((v, (r, c)), shape=(N, N)))
        R = np.unique(dA.nonzero()[0])
        s = len(R)
        DT = _csr(sp.csr_matrix((np.ones(s), R.astype(np.int32), np.arange(s + 1)), shape=(s, N)))
        batches.append(Batch("weights", _csr(dA[R]), DT))
        A = _csr(A + dA)
        # keep the edge list current for the next deletion draw
        cur = sp.triu(A, k=1).tocoo()
        elist_r, elist_c = cur.row.astype(np.int64), cur.col.astype(np.int64)
        if edges is not None:
            edges = set(zip(elist_r.tolist(), elist_c.tolist()))
    return Workload("C4-weights-rpi", k, U0, S0, V0, batches,
                    meta=dict(N=N, avg_deg=avg_deg, nnz=A.nnz, seed=seed, l=256, t=3))


# --------------------------------------------------------------------------- Fig-4 style
def synthetic_colappend(seed: int = 6, m: int = 2000, n: int = 2000, density: float = 1e-3, k: int = 16,
                        n_batches: int = 4) -> Workload:
    """PAPER.md:1014-1021 (Fig 4): random sparse matrix, init on the first 50 % of the
    columns, the rest appended as column batches."""
    A = random_sparse(m, n, density, seed)
    n0 = n // 2
    U0, S0, V0 = init_truncated_svd(A[:, :n0], k)
    step = (n - n0) // n_batches
    At = _csr(A.T)
    batches = [Batch("cols", _csr(At[n0 + b * step: n0 + (b + 1) * step])) for b in range(n_batches)]
    return Workload("F4-synthetic-colappend", k, U0, S0, V0, batches, meta=dict(m=m, n=n, seed=seed))


# --------------------------------------------------------------------------- C5
def scaleout_rowappend(seed: int = 5, m: int = 20_000_000, n: int = 2_000_000, k: int = 256, m_init=None,
                       batch: int = 100_000, n_batches: int = 20, deg_min: int = 5, deg_max: int = 200_000,
                       deg_exp: float = 2.0, zipf: float = 0.8, init_method: str = "randomized") -> Workload:
    """BASELINE.json configs[4] recipe as a host Workload with a host-computed
    initial SVD (reduced instances for the parity tests): the vectorised generator of
    synth.scaleout on the CPU (the full size is generated on the GPU by bench.py --config c5).
    m_init (if given) must equal m - n_batches * batch."""
    from .scaleout import scaleout_rowappend as _gen
    if m_init is not None and m_init != m - n_batches * batch:
        raise ValueError("m_init is m - n_batches * batch")
    so = _gen(seed=seed, m=m, n=n, k=k, batch=batch, n_batches=n_batches, deg_min=deg_min, deg_max=deg_max,
              deg_exp=deg_exp, zipf=zipf, device="cpu", chunk_rows=1 << 16)
    A0 = _csr(so.init.to_scipy())
    U0, S0, V0 = init_truncated_svd(A0, k, seed=seed + 100, method=init_method)
    batches = [Batch("rows", _csr(b.to_scipy())) for b in so.batches]
    return Workload("C5-scaleout-rowappend", k, U0, S0, V0, batches,
                    meta=dict(m=m, n=n, nnz=so.meta["nnz"], seed=seed, l=256, t=3))

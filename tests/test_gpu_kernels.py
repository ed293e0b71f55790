"""Kernel-level parity (-m gpu): each step of the CUDA path, called through the
step-level C-ABI (include/tsvd_kernels.h), against the oracle's plain definition of that
step (oracle/steps.py) or the closed form, on seeded inputs that span several tiles and
a ragged tail, including empty / duplicate / dependent update vectors."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import metrics, steps
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2401_09703_b200 as P
    return P


def dev(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


# (60001, 130, 96) / (70000, 256, 17): more than two waves of output tiles, ragged M / N / K —
# the persistent multi-tile mode (one cp.async pipeline across a CTA's tiles)
# (517, 130, 300), (518, 130, 301): even leading dimensions with ragged M / N / K — the 16-byte
# pair-staged path (zero-filled half pairs at the edges)
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (64, 64, 16), (130, 77, 45), (517, 64, 300), (64, 5000, 64),
                                   (60001, 130, 96), (70000, 256, 17), (517, 130, 300), (518, 130, 301)])
@pytest.mark.parametrize("tA,tB", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_dgemm(P, M, N, K, tA, tB):
    rng = np.random.default_rng(M * 7 + N + K)
    A = rng.standard_normal((K, M) if tA else (M, K))
    B = rng.standard_normal((N, K) if tB else (K, N))
    Cm = rng.standard_normal((M, N))
    ref = 0.7 * ((A.T if tA else A) @ (B.T if tB else B)) - 1.3 * Cm
    dA, dB, dC = dev(A), dev(B), dev(Cm)
    P.k_dgemm(tA, tB, M, N, K, 0.7, dA, A.shape[1], dB, B.shape[1], -1.3, dC, N)
    assert np.allclose(host(dC), ref, rtol=1e-13, atol=1e-12 * np.sqrt(K))


# (1000, 300): 5 x 5 tiles, split-K, warps below the diagonal of the diagonal tiles skipping
@pytest.mark.parametrize("K,n", [(33, 200), (1000, 300)])
def test_dgemm_upper(P, K, n):
    rng = np.random.default_rng(5 + K)
    X = rng.standard_normal((K, n))
    G = rng.standard_normal((n, n))
    dX, dG = dev(X), dev(G)
    P.k_dgemm(1, 0, n, n, K, -1.0, dX, n, dX, n, 1.0, dG, n, 1)
    out = host(dG)
    ref = G - X.T @ X
    iu = np.triu_indices(n)
    assert np.allclose(out[iu], ref[iu], atol=1e-12 * np.sqrt(K))
    il = np.tril_indices(n, -1)
    assert np.array_equal(out[il], G[il])       # lower triangle untouched


@pytest.mark.parametrize("k", [16, 32, 64, 128, 256, 24])
def test_gather_spmm(P, k):
    s, d = 1037, 3001
    E = synth.random_sparse(s, d, 0.004, seed=k, values="normal").tolil()
    E[5, :] = 0
    E[7, :40] = 1.0      # a heavier row
    E[9, 100:2100] = np.linspace(-1, 1, 2000)   # a hub row (> 256 nonzeros: CTA-per-row path)
    E = sp.csr_matrix(E)
    X = synth.random_orthonormal(d, k, seed=3)
    W_ref, _ = steps.lift(E, X, np.eye(k))
    dW = torch.empty((s, k), dtype=torch.float64, device="cuda")
    P.k_gather_spmm(P.Sparse.from_scipy(E, device="cuda"), dev(X), k, dW)
    assert np.allclose(host(dW), W_ref, rtol=1e-13, atol=1e-14)


def _heavy_rows(s, d, seed):
    """over 2^20 nonzeros with rows of 12k and 30k nonzeros (several 4096-long chunks each),
    plus many rows just above the long-row threshold: the chunked long-row path"""
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for i in range(s):
        n_i = 30_000 if i == 3 else 12_000 if i in (10, 11) else (40 if i % 7 == 0 else 300)
        c = rng.choice(d, size=n_i, replace=False)
        rows.append(np.full(n_i, i))
        cols.append(c)
    r, c = np.concatenate(rows), np.concatenate(cols)
    return sp.csr_matrix((rng.standard_normal(len(r)), (r, c)), shape=(s, d))


@pytest.mark.parametrize("k", [64, 256])
def test_gather_spmm_chunked_rows(P, k):
    E = _heavy_rows(4200, 60_000, seed=k)
    assert E.nnz >= 1 << 20
    X = synth.random_orthonormal(60_000, k, seed=4)
    W_ref, _ = steps.lift(E, X, np.eye(k))
    dW = torch.empty((E.shape[0], k), dtype=torch.float64, device="cuda")
    P.k_gather_spmm(P.Sparse.from_scipy(E, device="cuda"), dev(X), k, dW)
    assert np.allclose(host(dW), W_ref, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("k", [64, 256])
def test_scatter_add_chunked_columns(P, k):
    """The CSC side: hot columns of E^T (the transposed heavy rows) through the chunked path."""
    Et = _heavy_rows(4200, 50_000, seed=k + 1)
    E = sp.csr_matrix(Et.T)                 # 50000 update vectors, columns with 30k / 12k entries
    rng = np.random.default_rng(k)
    Z = rng.standard_normal((E.shape[0], k))
    X = rng.standard_normal((E.shape[1], k))
    ref = X + E.T @ Z
    dX = dev(X)
    P.k_scatter_add(P.Sparse.from_scipy(E, device="cuda"), dev(Z), k, dX)
    assert np.allclose(host(dX), ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("s,d,dens", [(1, 10, 0.5), (200, 500, 0.02), (1500, 4000, 0.003), (7000, 9000, 0.0004)])
def test_sparse_gram(P, s, d, dens):
    E = synth.random_sparse(s, d, dens, seed=s, values="normal")
    ref = steps.sparse_gram(E)
    dG = torch.empty((s, s), dtype=torch.float64, device="cuda")
    P.k_sparse_gram(P.Sparse.from_scipy(E, device="cuda"), dG)
    iu = np.triu_indices(s)   # the upper triangle is the result (include/tsvd_kernels.h)
    assert np.allclose(host(dG)[iu], ref[iu], rtol=1e-13, atol=1e-13)


def test_sparse_gram_heavy_rows_deterministic(P):
    """Power-user rows (thousands of nonzeros over moderately popular columns): their products
    are split over many row-block tasks; the result equals E E^T and is bitwise reproducible
    (each entry summed in row-nonzero order whatever the split)."""
    rng = np.random.default_rng(17)
    s, d = 2600, 6000
    deg = np.where(rng.random(s) < 0.02, rng.integers(2000, 5000, s), rng.integers(3, 60, s))
    rows, cols = [], []
    for i in range(s):
        c = np.unique(rng.integers(0, d, deg[i]))
        rows.append(np.full(len(c), i))
        cols.append(c)
    r, c = np.concatenate(rows), np.concatenate(cols)
    E = sp.csr_matrix((rng.standard_normal(len(r)), (r, c)), shape=(s, d))
    ref = steps.sparse_gram(E)
    dE = P.Sparse.from_scipy(E, device="cuda")
    G1 = torch.empty((s, s), dtype=torch.float64, device="cuda")
    G2 = torch.empty((s, s), dtype=torch.float64, device="cuda")
    P.k_sparse_gram(dE, G1)
    P.k_sparse_gram(dE, G2)
    iu = np.triu_indices(s)
    A, B = host(G1)[iu], host(G2)[iu]
    assert np.array_equal(A, B)
    assert np.allclose(A, ref[iu], rtol=1e-12, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("s,d", [(3500, 10_000), (900, 2000)])
def test_sparse_gram_hot_columns(P, s, d):
    """Zipf-popular columns (the configs[2] item popularity): the hot columns (above the
    threshold of least modelled cost) go through the dense SYRK, the rest through the sparse
    enumeration; the upper
    triangle (what the Cholesky and SYRK read) equals E E^T."""
    rng = np.random.default_rng(s)
    rows, cols = [], []
    p = 1.0 / np.arange(1, d + 1)
    p /= p.sum()
    for i in range(s):
        c = np.unique(rng.choice(d, size=int(rng.integers(5, 300)), p=p))
        rows.append(np.full(len(c), i))
        cols.append(c)
    r, c = np.concatenate(rows), np.concatenate(cols)
    E = sp.csr_matrix((rng.standard_normal(len(r)), (r, c)), shape=(s, d))
    assert np.diff(E.tocsc().indptr).max() > 256   # some hot columns
    ref = steps.sparse_gram(E)
    dG = torch.empty((s, s), dtype=torch.float64, device="cuda")
    P.k_sparse_gram(P.Sparse.from_scipy(E, device="cuda"), dG)
    G = host(dG)
    iu = np.triu_indices(s)
    assert np.allclose(G[iu], ref[iu], rtol=1e-12, atol=1e-12 * np.abs(ref).max())


_GRAM_CHILD = r"""
import sys, numpy as np, scipy.sparse as sp, torch
sys.path.insert(0, sys.argv[1])
import paper_2401_09703_b200 as P
from oracle import steps
rng = np.random.default_rng(5)
s, d = 1500, 4000
p = 1.0 / np.arange(1, d + 1); p /= p.sum()
rows, cols = [], []
for i in range(s):
    c = np.unique(rng.choice(d, size=int(rng.integers(5, 200)), p=p))
    rows.append(np.full(len(c), i)); cols.append(c)
r, c = np.concatenate(rows), np.concatenate(cols)
E = sp.csr_matrix((rng.standard_normal(len(r)), (r, c)), shape=(s, d))
ref = steps.sparse_gram(E)
G = torch.empty((s, s), dtype=torch.float64, device="cuda")
P.k_sparse_gram(P.Sparse.from_scipy(E, device="cuda"), G)
iu = np.triu_indices(s)
err = np.abs(G.cpu().numpy()[iu] - ref[iu]).max() / np.abs(ref).max()
print("ERR", err)
sys.exit(0 if err < 1e-13 else 1)
"""


@pytest.mark.parametrize("env", [{"TSVD_GRAM_ESC": "0"}, {"TSVD_GRAM_ESC": "0", "TSVD_GRAM_HOT": "64"},
                                 {"TSVD_GRAM_HOT": "-1"}, {"TSVD_GRAM_HOT": "16"}])
def test_sparse_gram_paths(P, env):
    """The K3 paths the threshold model does not pick on its own (the knobs are read once per
    process, so each runs in a child): the row-walk cold part with and without a dense part,
    expand-sort-reduce with no dense part, and a forced low threshold."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _GRAM_CHILD, root], env={**os.environ, **env},
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.parametrize("s", [5, 64, 65, 200, 333, 700, 1100])
def test_chol_deflate(P, s):
    rng = np.random.default_rng(s)
    k, d = 6, 2 * s + 50
    U = synth.random_orthonormal(d, k, seed=s)
    E = synth.random_sparse(s, d, min(0.5, 8.0 / d), seed=s + 1, values="normal").toarray()
    # rank deficiency: empty, duplicate, dependent and in-span vectors
    if s > 10:
        E[3] = 0
        E[4] = E[1]
        E[8] = E[0] - 2 * E[2]
        E[9] = (U @ rng.standard_normal(k))
    if s > 600:   # deflations inside later recursion blocks of the GPU factorisation
        E[300] = 0
        E[555] = E[20] + E[400]
        E[s - 1] = E[s - 2]
    ET = sp.csr_matrix(E)
    C0T = E @ U
    G = steps.svlcov_gram(ET, C0T)
    en = (E ** 2).sum(1)
    R_ref, keep_ref = steps.chol_deflate(G, en)
    dG = dev(G.copy())
    keep = torch.zeros(s, dtype=torch.int32, device="cuda")
    r = P.k_chol_deflate(dG, s, dev(en), 1e-12, keep)
    R = host(dG)
    assert np.array_equal(host(keep).astype(bool), keep_ref)
    assert r == keep_ref.sum()
    assert np.allclose(R, R_ref, rtol=1e-10, atol=1e-10 * np.sqrt(G.diagonal().max()))
    assert np.allclose(np.tril(R, -1), 0)


@pytest.mark.parametrize("s,k", [(10, 16), (64, 64), (130, 64), (257, 128)])
def test_trsm_upper(P, s, k):
    rng = np.random.default_rng(s + k)
    # well-conditioned upper factor (random triangular matrices are exponentially ill-conditioned)
    R = np.triu(rng.standard_normal((s, s)), 1) / np.sqrt(s) + np.diag(2.0 + rng.random(s))
    keep = np.ones(s, dtype=np.int32)
    keep[::7] = 0
    R[keep == 0] = 0.0
    X = rng.standard_normal((s, k))
    kk = keep.astype(bool)
    ref = np.zeros((s, k))
    ref[kk] = np.linalg.solve(R[np.ix_(kk, kk)], X[kk])
    dX = dev(X)
    P.k_trsm_upper(dev(R), s, dev(keep), dX, k)
    assert np.allclose(host(dX), ref, rtol=1e-11, atol=1e-11)


def _jacobi(P, K, kk):
    m, n = K.shape
    dK = dev(np.asfortranarray(K).T.copy().reshape(-1))  # column-major
    th = torch.empty(n, dtype=torch.float64, device="cuda")
    F = torch.empty(kk * m, dtype=torch.float64, device="cuda")
    G = torch.empty(kk * n, dtype=torch.float64, device="cuda")
    sw = P.k_jacobi_svd(dK, m, n, kk, th, F, G)
    return host(th), host(F).reshape(kk, m).T, host(G).reshape(kk, n).T, sw


@pytest.mark.parametrize("m,n,kk", [(8, 8, 3), (116, 116, 16), (200, 150, 64), (333, 333, 40), (700, 513, 64),
                                    (384, 384, 128), (512, 512, 256), (512, 300, 100), (160, 129, 64)])
def test_jacobi_svd(P, m, n, kk):
    rng = np.random.default_rng(m + n)
    K = rng.standard_normal((m, n)) * np.logspace(0, -6, n)[None, :]
    th, F, G, sw = _jacobi(P, K, kk)
    ref = np.linalg.svd(K, compute_uv=False)
    assert np.allclose(th, ref, rtol=1e-11, atol=1e-13 * ref[0])
    u, s, vt = np.linalg.svd(K, full_matrices=False)
    kq = metrics.gap_rank(ref, kk)
    assert metrics.sin_theta(F[:, :kq], u[:, :kq]) < 1e-10
    assert metrics.sin_theta(G[:, :kq], vt[:kq].T) < 1e-10
    # G = K^T F Θ^-1 (right_from_left): a left pair left at the stopping tolerance |f_i.f_j| <=
    # tol = 1e-14 enters g_j with weight θ_i / θ_j, so G's orthogonality scales with the spread
    # of the kk leading values (the subspace of G_kk is unaffected)
    assert metrics.orth_err(F) < 1e-12
    assert metrics.orth_err(G) < 1e-12 * max(1.0, 0.01 * th[0] / th[kk - 1])
    assert np.allclose(K @ G, F * th[:kk], atol=1e-11 * ref[0])


def test_jacobi_rank_deficient_and_completion(P):
    """Core with fewer than kk nonzero singular values: trailing θ = 0 and F padded
    orthonormally."""
    rng = np.random.default_rng(1)
    K = np.zeros((40, 20))
    K[:, :3] = rng.standard_normal((40, 3))
    th, F, G, sw = _jacobi(P, K, 8)
    ref = np.linalg.svd(K, compute_uv=False)
    assert np.allclose(th[:3], ref[:3], rtol=1e-12) and np.all(th[3:] < 1e-12 * th[0])
    assert metrics.orth_err(F) < 1e-12 and metrics.orth_err(G) < 1e-12


def test_jacobi_structured_core(P):
    """The Alg 9 core [Σ, 0; C0^T, R^T] with clustered singular values."""
    S = np.array([10, 9.99, 9.98, 5, 4, 3, 2, 1.0])
    rng = np.random.default_rng(3)
    s = 50
    C0T = rng.standard_normal((s, 8)) * 0.1
    R = np.triu(rng.standard_normal((s, s))) * 0.05
    K = np.block([[np.diag(S), np.zeros((8, s))], [C0T, R.T]])
    th, F, G, sw = _jacobi(P, K, 8)
    ref = np.linalg.svd(K, compute_uv=False)
    assert np.allclose(th, ref, rtol=1e-12, atol=1e-14 * ref[0])


@pytest.mark.parametrize("n", [160, 384, 512])
def test_jacobi_cluster_clustered(P, n):
    """K9 (the cluster-resident Jacobi, 128 < n <= 512) on a weight-update-like core: a
    dominant diagonal (the previous Σ, with a near tie) plus a small low-rank part and a
    cluster of tiny trailing values; exactly zero columns ride along."""
    rng = np.random.default_rng(n)
    k = n // 3
    S = np.concatenate([np.linspace(1000, 100, k), np.zeros(n - k)])
    S[1] = S[0] * (1 - 1e-9)
    L = rng.standard_normal((n, 8)) * 3.0
    K = np.diag(S) + L @ rng.standard_normal((8, n)) + 1e-6 * rng.standard_normal((n, n))
    K[:, -3:] = 0.0
    th, F, G, sw = _jacobi(P, K, k)
    ref = np.linalg.svd(K, compute_uv=False)
    assert np.allclose(th, ref, rtol=1e-11, atol=1e-13 * ref[0])
    u, s_, vt = np.linalg.svd(K, full_matrices=False)
    kq = metrics.gap_rank(ref, k)
    assert metrics.sin_theta(F[:, :kq], u[:, :kq]) < 1e-10
    assert metrics.orth_err(F) < 1e-12 and metrics.orth_err(G) < 1e-12


def _core(P, K, kk):
    m, n = K.shape
    dK = dev(np.asfortranarray(K).ravel(order="F"))
    th = torch.zeros(kk + 1, dtype=torch.float64, device="cuda")
    F = torch.empty(kk * m, dtype=torch.float64, device="cuda")
    G = torch.empty(kk * n, dtype=torch.float64, device="cuda")
    info = P.k_core_svd(dK, m, n, kk, th, F, G)
    return host(th), host(F).reshape(kk, m).T, host(G).reshape(kk, n).T, info


def _graph_core(N=12000, n_init=6000, batch=1200, k=32):
    """The Alg 9 core of one configs[1]-recipe row batch (reduced), via the oracle's plain
    step definitions (oracle/steps.py)."""
    w = synth.graph_nodeappend(N=N, n_init=n_init, batch=batch, n_batches=1, k=k)
    b = w.batches[0]
    _, C0T = steps.lift(b.E, w.V0, np.eye(k))
    G = steps.svlcov_gram(b.E, C0T)
    en = np.asarray(b.E.multiply(b.E).sum(axis=1)).ravel()
    R, keep = steps.chol_deflate(G, en)
    return steps.core_rows(w.S0, C0T, R, keep)


@pytest.mark.parametrize("case", ["graph", "decay", "tall", "weights", "weights512"])
def test_core_svd_paths(P, case):
    """A5 as the updates run it: Rayleigh-Ritz reduction (path 2) for large cores, Cholesky-
    QR2 preconditioning (path 1) for tall ones; SVD_kk against LAPACK, the energy ||K||_F^2."""
    rng = np.random.default_rng(5)
    if case == "graph":
        K, kk, path = _graph_core(), 32, 2
    elif case == "decay":
        m, n = 1500, 900
        U, _ = np.linalg.qr(rng.standard_normal((m, n)))
        V, _ = np.linalg.qr(rng.standard_normal((n, n)))
        K, kk, path = (U * np.logspace(2, -3, n)) @ V.T, 40, 2
    elif case == "weights":
        # configs[3]-like weight-update core (384 = k + l): diag(Σ, 0) plus a low-rank update and a
        # decaying tail — K9 in one cluster with the leading-set (tail-skip) convergence
        n, kk, path = 384, 128, 2
        S = np.concatenate([np.linspace(1000, 100, kk), np.zeros(n - kk)])
        T = rng.standard_normal((n, n)) * np.logspace(0, -3, n)[None, :] * 0.5
        K = np.diag(S) + rng.standard_normal((n, 6)) @ rng.standard_normal((6, n)) + T
    elif case == "weights512":
        n, kk, path = 512, 256, 0
        S = np.concatenate([np.linspace(1000, 300, kk), np.zeros(n - kk)])
        K = np.diag(S) + rng.standard_normal((n, n)) * np.logspace(0, -4, n)[None, :]
    else:
        K, kk, path = rng.standard_normal((3000, 150)) * np.logspace(0, -4, 150), 20, 1
    th, F, G, info = _core(P, K, kk)
    assert info["path"] == path, info
    u, ref, vt = np.linalg.svd(K, full_matrices=False)
    assert np.allclose(th[:kk], ref[:kk], rtol=1e-11, atol=1e-13 * ref[0]), (th[:5], ref[:5])
    # θ_{kk+1} (a statistic: the Rayleigh-Ritz path stops on the leading kk pairs, and the
    # (kk+1)-th Ritz value is accurate to second order in its residual)
    assert np.isclose(th[kk], ref[kk], rtol=1e-8, atol=1e-13 * ref[0]), (th[kk], ref[kk])
    kq = metrics.gap_rank(ref, kk)
    assert metrics.sin_theta(F[:, :kq], u[:, :kq]) < 1e-10
    assert metrics.sin_theta(G[:, :kq], vt[:kq].T) < 1e-10
    assert metrics.orth_err(F) < 1e-12 and metrics.orth_err(G) < 1e-12
    assert np.isclose(info["energy"], (ref ** 2).sum(), rtol=1e-12)


@pytest.mark.parametrize("k", [4, 16, 37, 64, 96, 97, 128, 160, 200, 256, 300, 384, 512])
def test_inverse_cond(P, k):
    rng = np.random.default_rng(k)
    M = rng.standard_normal((k, k)) + 2 * np.eye(k)
    Minv = torch.empty((k, k), dtype=torch.float64, device="cuda")
    cond = torch.empty(1, dtype=torch.float64, device="cuda")
    P.k_inverse(dev(M), k, Minv, cond)
    assert np.allclose(host(Minv) @ M, np.eye(k), atol=1e-10)
    assert np.isclose(host(cond)[0], steps.cond1(M), rtol=1e-9)


@pytest.mark.parametrize("k", [8, 37, 64, 100, 128, 256, 512])
def test_inverse_pivoting(P, k):
    """Zero diagonal (a shifted permutation plus small noise): every pivot needs a row swap."""
    rng = np.random.default_rng(7 + k)
    M = np.roll(np.eye(k), 1, axis=0) * (1.0 + rng.random(k))[:, None] + 1e-3 * rng.standard_normal((k, k))
    np.fill_diagonal(M, 0.0)
    Minv = torch.empty((k, k), dtype=torch.float64, device="cuda")
    cond = torch.empty(1, dtype=torch.float64, device="cuda")
    P.k_inverse(dev(M), k, Minv, cond)
    assert np.allclose(host(Minv) @ M, np.eye(k), atol=1e-9)
    assert np.isclose(host(cond)[0], steps.cond1(M), rtol=1e-9)


@pytest.mark.parametrize("k", [3, 100, 128, 256])
def test_inverse_singular(P, k):
    M = np.diag(np.arange(1.0, k + 1.0))
    M[k - 1, k - 1] = 0.0
    cond = torch.empty(1, dtype=torch.float64, device="cuda")
    P.k_inverse(dev(M), k, torch.empty((k, k), dtype=torch.float64, device="cuda"), cond)
    assert np.isinf(host(cond)[0])


@pytest.mark.parametrize("k", [16, 64, 128, 256])
def test_norm2_estimate(P, k):
    """The MII decision's cond_2 (reading R18): ||M||_2 of a matrix with known singular values
    (Q1 diag(s) Q2^T, s log-spaced over 4 decades, top gap 1.5x) to 1e-10; a lower estimate."""
    rng = np.random.default_rng(k)
    Q1 = np.linalg.qr(rng.standard_normal((k, k)))[0]
    Q2 = np.linalg.qr(rng.standard_normal((k, k)))[0]
    s = np.logspace(0, -4, k)
    s[0] = 1.5 * s[1]
    M = Q1 @ np.diag(s) @ Q2.T
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    P.k_norm2_est(dev(M), k, out)
    e = host(out)[0]
    assert e <= s[0] * (1 + 1e-14) and abs(e - s[0]) < 1e-10 * s[0], (e, s[0])


@pytest.mark.parametrize("k", [16, 64, 256, 24])
def test_scatter_add(P, k):
    s, d = 900, 2500
    E = synth.random_sparse(s, d, 0.003, seed=k + 1, values="normal").tolil()
    E[:, 11] = 1.0  # a hot column (long CSC segment)
    E = sp.csr_matrix(E)
    rng = np.random.default_rng(k)
    Z = rng.standard_normal((s, k))
    X = rng.standard_normal((d, k))
    ref = X + E.T @ Z
    dX = dev(X)
    P.k_scatter_add(P.Sparse.from_scipy(E, device="cuda"), dev(Z), k, dX)
    assert np.allclose(host(dX), ref, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("rows,k", [(1, 16), (1000, 16), (4097, 64), (333, 256), (50, 12), (70000, 64), (300001, 256)])
def test_materialize(P, rows, k):
    rng = np.random.default_rng(rows)
    X = rng.standard_normal((rows, k))
    M = rng.standard_normal((k, k))
    dX = dev(X)
    P.k_materialize(dX, rows, k, dev(M))
    assert np.allclose(host(dX), X @ M, rtol=1e-13, atol=1e-12)


@pytest.mark.parametrize("rows,l", [(300, 16), (500, 37), (3345, 96), (3000, 100), (3345, 128), (2000, 200),
                                    (2000, 201), (20000, 256), (5000, 384)])
def test_cholqr_dense(P, rows, l):
    """Cholesky-QR2 with deflation of a dense block (the fused one-CTA small Cholesky +
    inverse for l <= 128, the blocked path above): Q orthonormal on the kept columns,
    Q R = X, R upper with the LAPACK QR's |diagonal|; an exactly dependent column deflates."""
    rng = np.random.default_rng(rows + l)
    X = rng.standard_normal((rows, l)) * np.logspace(0, -3, l)
    X[:, 5] = X[:, 1] - 2 * X[:, 3]            # dependent: deflated
    dX, dR = dev(X.copy()), torch.zeros((l, l), dtype=torch.float64, device="cuda")
    P.k_cholqr(dX, rows, l, 2, 1e-14, dR)
    Q, R = host(dX), host(dR)
    live = np.linalg.norm(Q, axis=0) > 0.5
    assert live.sum() == l - 1 and not live[5]
    assert metrics.orth_err(Q[:, live]) < 1e-13
    assert np.allclose(Q @ R, X, atol=1e-12 * np.abs(X).max())
    assert np.allclose(np.tril(R, -1), 0)
    _, Rl = np.linalg.qr(np.delete(X, 5, axis=1))
    assert np.allclose(np.abs(np.diag(R))[live], np.abs(np.diag(Rl)), rtol=1e-9)


@pytest.mark.parametrize("rows,l", [(3000, 64), (20000, 256)])
def test_cholqr_one_pass_range(P, rows, l):
    """One Cholesky-QR pass (the RPI range passes): Q spans range(X) to rounding, Q R = X,
    and its orthogonality error is of order eps cond(X)^2."""
    rng = np.random.default_rng(rows - l)
    X = rng.standard_normal((rows, l)) * np.logspace(0, -2, l)
    dX, dR = dev(X.copy()), torch.zeros((l, l), dtype=torch.float64, device="cuda")
    P.k_cholqr(dX, rows, l, 1, 1e-14, dR)
    Q, R = host(dX), host(dR)
    assert np.allclose(Q @ R, X, atol=1e-12 * np.abs(X).max())
    assert metrics.orth_err(Q) < 1e-8
    assert metrics.sin_theta(Q, X) < 1e-10


@pytest.mark.parametrize("kind,nt,nkb", [(0, 1, 1), (0, 2, 1), (0, 5, 1), (0, 66, 1), (0, 130, 1),
                                         (1, 1, 1), (1, 3, 2), (1, 66, 1), (1, 40, 3)])
def test_dag_device_order_matches_host(P, kind, nt, nkb):
    """The device task generator of the tile-DAG kernels emits exactly the host order that
    tests/test_dag_order.py proves complete and deadlock-free."""
    assert P.dag_check(kind, nt, nkb) == 0

"""F1: the initial truncated SVD on the GPU, tsvd_init_sparse (-m gpu).

Randomized subspace iteration ("randomized numerical linear algebra"; the
initialisation of PAPER.md:486-488) through the C-ABI, checked against LAPACK:
  * an A of rank r <= p = k + oversample is recovered exactly (to rounding): σ within 1e-10,
    sin θ of U_k / V_k below 1e-8 (the north_star tolerances) — including k = 256, whose
    p = 288 runs the gathers in 256 + 32 column panels and the projected SVD in K9;
  * a full-rank A: orthonormal factors, σ close to LAPACK's with power steps;
  * the initialised context then runs an update against the oracle."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import metrics, zha_simon
import synth
from tests import helpers as H

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2401_09703_b200 as P
    return P


def _low_rank_sparse(m, n, r, dens, seed):
    """sum of r outer products of sparse vectors: rank r, sparse, distinct decaying weights"""
    rng = np.random.default_rng(seed)
    Us = sp.random(m, r, density=dens, random_state=seed, format="csc")
    Vs = sp.random(n, r, density=dens, random_state=seed + 1, format="csc")
    w = np.logspace(1, -1, r) * (1 + 0.1 * rng.random(r))
    return sp.csr_matrix(Us @ sp.diags(w) @ Vs.T)


def _run(P, A, k, oversample, power_iters):
    m, n = A.shape
    t = P.TSVD(k, m_capacity=m, n_capacity=n)
    t.init_sparse(P.Sparse.from_scipy(A, device="cuda"), oversample=oversample, power_iters=power_iters, seed=7)
    return t


@pytest.mark.parametrize("m,n,k,r,over", [(3000, 2000, 16, 24, 16), (1500, 1200, 64, 80, 32), (2000, 1600, 256, 270, 32)])
def test_exact_for_low_rank(P, m, n, k, r, over):
    A = _low_rank_sparse(m, n, r, 0.08, seed=m + k)
    t = _run(P, A, k, over, 1)
    U, S, V = t.get_U(), t.get_S(), t.get_V()
    u, s, vt = np.linalg.svd(A.toarray(), full_matrices=False)
    assert metrics.sigma_relerr(S, s[:k]) < 1e-10, (S[:4], s[:4])
    kk = metrics.gap_rank(s, k)
    assert metrics.sin_theta(U[:, :kk], u[:, :kk]) < 1e-8
    assert metrics.sin_theta(V[:, :kk], vt[:kk].T) < 1e-8
    # (V comes from the Jacobi's left vectors through R^T U Θ^-1: its orthogonality scales with
    # the spread θ_1 / θ_k, 100 here; tsvd_init's own bar is 1e-10)
    assert metrics.orth_err(U) < 1e-12 and metrics.orth_err(V) < 1e-11


def test_full_rank_power_steps(P):
    """Full rank: a decaying rank-40 part plus sparse noise of 1 % of its smallest weight."""
    A = sp.csr_matrix(_low_rank_sparse(4000, 3000, 40, 0.05, seed=3) + 0.01 * synth.random_sparse(4000, 3000, 0.01, seed=4))
    k = 32
    t = _run(P, A, k, 32, 3)
    U, S, V = t.get_U(), t.get_S(), t.get_V()
    s = np.linalg.svd(A.toarray(), compute_uv=False)
    assert metrics.orth_err(U) < 1e-12 and metrics.orth_err(V) < 1e-11
    assert np.all(np.diff(S) <= 0) and S[-1] > 0
    assert np.all(S <= s[:k] * (1 + 1e-12))            # Rayleigh-Ritz values never exceed
    assert np.max(np.abs(S - s[:k]) / s[:k]) < 1e-6    # randomized approximation with 3 power steps


def test_init_then_update_matches_oracle(P):
    """The GPU-initialised state is a valid start: one exact row update against the oracle run
    from LAPACK's truncated SVD of the same A (its own input, nothing read back from the GPU;
    for this exactly low-rank A with distinct singular values both starts are the same
    factorisation up to column signs, to which the update is indifferent)."""
    A = _low_rank_sparse(1200, 900, 20, 0.1, seed=11)
    k = 16
    t = _run(P, A, k, 16, 1)
    u, s, vt = np.linalg.svd(A.toarray(), full_matrices=False)
    U0, S0, V0 = u[:, :k].copy(), s[:k].copy(), vt[:k].T.copy()
    Er = synth.random_sparse(50, 900, 0.05, seed=12, values="normal")
    H.gpu_apply(P, t, synth.Batch("rows", Er))
    Uo, So, Vo, th = zha_simon.add_rows(U0, S0, V0, Er)
    ok, d = H.compare(*H.gpu_factors(t), Uo, So, Vo, th, k)
    assert ok, d


def test_shape_errors(P):
    A = synth.random_sparse(40, 30, 0.2, seed=1)
    t = P.TSVD(16, m_capacity=40, n_capacity=30)
    with pytest.raises(P.TsvdError) as ei:
        t.init_sparse(P.Sparse.from_scipy(A, device="cuda"), oversample=32)
    assert ei.value.status == 1

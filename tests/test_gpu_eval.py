"""F2 on the GPU (-m gpu): tsvd_score_pairs / tsvd_residual_fro on the maintained Ã against
the oracle's dense U Σ V^T after the same stream (scores are basis independent)."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import zha_simon
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


def _stream(P):
    w = synth.tiny_rowappend(n_batches=3)
    t = H.gpu_state(P, w)
    U, S, V = w.U0, w.S0, w.V0
    for b in w.batches:
        H.gpu_apply(P, t, b)
        U, S, V, _ = zha_simon.apply_batch(U, S, V, b)
    return w, t, U, S, V


def test_score_pairs_match_oracle(P):
    w, t, U, S, V = _stream(P)
    rng = np.random.default_rng(1)
    m, n = U.shape[0], V.shape[0]
    r = rng.integers(0, m, 5000)
    c = rng.integers(0, n, 5000)
    ref = np.einsum("pk,k,pk->p", U[r], S, V[c])
    got = t.score_pairs(r, c)
    assert np.abs(got - ref).max() <= 1e-9 * S[0]
    # device arrays in and out
    dr, dc = torch.from_numpy(r).cuda(), torch.from_numpy(c).cuda()
    out = torch.empty(5000, dtype=torch.float64, device="cuda")
    t.score_pairs(dr, dc, out)
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-9 * S[0]
    with pytest.raises(P.TsvdError) as ei:
        t.score_pairs([m], [0])
    assert ei.value.status == 6


def test_residual_fro_matches_dense(P):
    w, t, U, S, V = _stream(P)
    m = U.shape[0]
    A = synth.random_sparse(2000, 1000, 10_000 / 2e6, 1)[:m]   # the C1 matrix's first m rows
    A = sp.csr_matrix(A)
    res, inner, a2 = t.residual_fro(P.Sparse.from_scipy(A, device="cuda"))
    At = (U * S) @ V.T
    assert np.isclose(a2, (A.multiply(A)).sum(), rtol=1e-12)
    assert np.isclose(inner, (A.multiply(At)).sum(), rtol=1e-9)
    assert np.isclose(res, np.linalg.norm(A.toarray() - At), rtol=1e-7)

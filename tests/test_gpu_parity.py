"""Update-level parity (-m gpu): the CUDA path through the C-ABI vs the CPU oracle on
identical seeded inputs and identical init factors.  Bar (BASELINE.json north_star):
σ within 1e-10 relative, sin θ_max of U_k and V_k below 1e-8 (gap-guarded)."""
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


def _stream_parity(P, w, opts=None, n_batches=None, check_every=1):
    t = H.gpu_state(P, w)
    ref = H.run_oracle(w, n_batches)
    worst = dict(sigma=0.0, angle_u=0.0, angle_v=0.0)
    for i, b in enumerate(w.batches[:n_batches]):
        H.gpu_apply(P, t, b, opts)
        if (i + 1) % check_every and i + 1 != len(ref):
            continue
        Ug, Sg, Vg = H.gpu_factors(t)
        Uo, So, Vo, th = ref[i]
        assert Ug.shape == Uo.shape and Vg.shape == Vo.shape
        ok, d = H.compare(Ug, Sg, Vg, Uo, So, Vo, th, w.k)
        for key in worst:
            worst[key] = max(worst[key], d[key])
        assert ok, (i, d, t.stats())
        assert metrics.orth_err(Ug) < 1e-9 and metrics.orth_err(Vg) < 1e-9
    return t, worst


def test_c1_tiny_rowappend_full(P):
    """BASELINE.json configs[0] at full size: 10 batches of 100 appended rows, k = 16."""
    w = synth.tiny_rowappend()
    t, worst = _stream_parity(P, w)
    st = t.stats()
    assert st["launches"] > 0
    print("C1 worst", worst, st)


@pytest.mark.parametrize("m,n,k,s,dens", [(60, 50, 5, 4, 0.15), (40, 70, 8, 12, 0.2), (90, 80, 16, 40, 0.05)])
@pytest.mark.parametrize("kind", ["rows", "cols", "weights"])
def test_small_random(P, m, n, k, s, dens, kind):
    A = synth.random_sparse(m, n, dens, seed=m * n + s, values="normal")
    U0, S0, V0 = synth.init_truncated_svd(A, k)
    rng_seed = 100 + s
    if kind == "rows":
        b = synth.Batch("rows", synth.random_sparse(s, n, dens, rng_seed, values="normal"))
    elif kind == "cols":
        b = synth.Batch("cols", synth.random_sparse(s, m, dens, rng_seed, values="normal"))
    else:
        b = synth.Batch("weights", synth.random_sparse(s, n, dens, rng_seed, values="normal"),
                        synth.random_sparse(s, m, dens, rng_seed + 1, values="normal"))
    w = synth.Workload("small", k, U0, S0, V0, [b, b] if kind != "weights" else [b])
    _stream_parity(P, w)


def test_rank_deficient_batch(P):
    """Empty, duplicate, dependent and in-span update vectors."""
    m, n, k = 80, 60, 6
    A = synth.random_sparse(m, n, 0.1, seed=7, values="normal")
    U0, S0, V0 = synth.init_truncated_svd(A, k)
    E = synth.random_sparse(10, n, 0.15, seed=8, values="normal").toarray()
    E[2] = 0
    E[5] = E[1]
    E[7] = E[0] + E[3]
    E[9] = V0[:, 0] * 3.0          # inside span(V_k)
    w = synth.Workload("defl", k, U0, S0, V0, [synth.Batch("rows", sp.csr_matrix(E))])
    t, _ = _stream_parity(P, w)
    Z = E - (E @ V0) @ V0.T
    assert t.stats()["rank"][1] == np.linalg.matrix_rank(Z, tol=1e-8)


def test_graph_nodeappend_reduced(P):
    """configs[1] recipe at reduced scale (4k nodes, 200-node batches, rows then columns):
    power-law graph, many empty / duplicate rows, MII resets active."""
    w = synth.graph_nodeappend(N=4000, n_init=2000, batch=200, n_batches=5, k=32)
    _stream_parity(P, w)


def test_ratings_rowappend_reduced(P):
    """configs[2] recipe at reduced scale."""
    w = synth.ratings_rowappend(users=3000, items=800, nnz=120_000, k=32, u_init=1500, batch=300, n_batches=3)
    _stream_parity(P, w)


def test_spec_examples(P):
    """SPEC.md:248 (append e3 to diag(3,2) keeps σ = [3,2]) and SPEC.md:266 (rank-1
    cancellation gives σ_k = 0) through the GPU path."""
    t = P.TSVD(2, 3, 3)
    U = np.eye(3)[:, :2].copy(); V = np.eye(2); S = np.array([3.0, 2.0])
    t.init(U, S, V)
    t.update_cols(P.Sparse.from_scipy(sp.csr_matrix(np.array([[0, 0, 1.0]]))))
    assert np.allclose(t.get_S(), [3, 2], atol=1e-14)
    t3 = P.TSVD(3, 3, 3)
    d = np.array([5.0, 3.0, 2.0])
    t3.init(np.eye(3), d, np.eye(3))
    t3.update_weights(P.Sparse.from_scipy(sp.csr_matrix(np.array([[0, 0, -2.0]]))),
                      P.Sparse.from_scipy(sp.csr_matrix(np.array([[0, 0, 1.0]]))))
    assert np.allclose(t3.get_S(), [5, 3, 0], atol=1e-13)
    Ug = t3.get_U()
    assert metrics.orth_err(Ug) < 1e-12   # orthonormal completion of the zero triplet


def test_zero_update_and_noop(P):
    t = P.TSVD(2, 5, 5)
    t.init(np.eye(3)[:, :2].copy(), np.array([4.0, 2.0]), np.eye(2))
    t.update_rows(P.Sparse.from_scipy(sp.csr_matrix((1, 2))))
    assert np.allclose(t.get_S(), [4, 2]) and t.dims()[0] == 4
    assert np.allclose(t.get_U()[-1], 0, atol=1e-15)
    t.update_rows(P.Sparse.from_scipy(sp.csr_matrix((0, 2))))     # s = 0: no-op
    assert t.dims()[0] == 4


def test_query_and_materialize(P):
    w = synth.tiny_rowappend(n_batches=3)
    t = H.gpu_state(P, w)
    for b in w.batches:
        H.gpu_apply(P, t, b)
    U = t.get_U()
    V = t.get_V()
    for i in (0, 5, U.shape[0] - 1):
        assert np.allclose(t.query_row(0, i), U[i], rtol=1e-12, atol=1e-15)
    assert np.allclose(t.query_row(1, 7), V[7], rtol=1e-12, atol=1e-15)
    t.materialize()
    assert np.allclose(t.get_U(), U, atol=1e-13) and np.allclose(t.get_V(), V, atol=1e-13)
    with pytest.raises(P.TsvdError):
        t.query_row(0, U.shape[0])


def test_deferred_resets_of_the_append_side(P):
    """MII resets forced at every update (threshold 1 + 1e-9, reading R18): the append side's
    resets are deferred (pending row blocks with their own multiplier, R18).  Row
    queries inside pending blocks, score_pairs and get_U (which materialises them) agree, and
    the stream matches the oracle; a later column update lifts U (flush) and still matches."""
    w = synth.tiny_rowappend(n_batches=4)
    t = H.gpu_state(P, w)
    opts = P.make_opts(reset_cond=1.0 + 1e-9)
    for b in w.batches:
        H.gpu_apply(P, t, b, opts)
    assert t.stats()["total_resets"] >= 4
    m = t.dims()[0]
    rows = (0, 999, 1000, 1150, 1299, m - 1)
    q = [t.query_row(0, i) for i in rows]          # before anything materialises
    sc = t.score_pairs(np.array(rows, dtype=np.int64), np.array([3, 5, 7, 11, 13, 17], dtype=np.int64))
    U, S, V = H.gpu_factors(t)
    for i, qi in zip(rows, q):
        assert np.allclose(qi, U[i], rtol=1e-12, atol=1e-14)
    ref = (U[list(rows)] * S) @ V[[3, 5, 7, 11, 13, 17]].T
    assert np.allclose(sc, np.diag(ref), rtol=1e-10, atol=1e-13)
    Uo, So, Vo, th = H.run_oracle(w)[-1]
    ok, d = H.compare(U, S, V, Uo, So, Vo, th, w.k)
    assert ok, d
    # a column update after the deferred row resets: U is the lift side now
    Ec = synth.random_sparse(20, m, 0.01, seed=9)
    t.update_cols(P.Sparse.from_scipy(Ec, device="cuda"), opts)
    U2, S2, V2 = H.gpu_factors(t)
    Uo2, So2, Vo2, th2 = zha_simon.add_columns(Uo, So, Vo, Ec)
    ok, d = H.compare(U2, S2, V2, Uo2, So2, Vo2, th2, w.k)
    assert ok, d


def test_invalid_input_leaves_state_unchanged(P):
    w = synth.tiny_rowappend(n_batches=1)
    t = H.gpu_state(P, w)
    U0 = t.get_U()
    bad = P.Sparse(1, w.n0, np.array([0, 2], np.int64), np.array([5, 5000], np.int32), np.array([1.0, 2.0]))
    with pytest.raises(P.TsvdError) as ei:
        t.update_rows(bad)
    assert ei.value.status == 7
    unsorted = P.Sparse(1, w.n0, np.array([0, 2], np.int64), np.array([9, 3], np.int32), np.array([1.0, 2.0]))
    with pytest.raises(P.TsvdError):
        t.update_rows(unsorted)
    dup = P.Sparse(2, w.n0, np.array([0, 2, 4], np.int64), np.array([3, 7, 2, 2], np.int32), np.ones(4))
    with pytest.raises(P.TsvdError) as ei:           # a repeated column inside the second row
        t.update_rows(dup)
    assert ei.value.status == 7
    nan = P.Sparse(1, w.n0, np.array([0, 1], np.int64), np.array([3], np.int32), np.array([np.nan]))
    with pytest.raises(P.TsvdError) as ei:
        t.update_rows(nan)
    assert ei.value.status == 4
    with pytest.raises(P.TsvdError) as ei:
        t.update_cols(P.Sparse.from_scipy(sp.csr_matrix((2, 7))))
    assert ei.value.status == 1
    assert np.array_equal(t.get_U(), U0) and t.dims()[0] == w.m0
    # a column descent at a row start is legal
    ok = P.Sparse(2, w.n0, np.array([0, 2, 4], np.int64), np.array([3, 7, 2, 5], np.int32), np.ones(4))
    t.update_rows(ok)
    assert t.dims()[0] == w.m0 + 2


def test_host_inputs_e2e(P):
    """Host (numpy) inputs are staged by the library: same result as device inputs."""
    w = synth.tiny_rowappend(n_batches=2)
    t1 = H.gpu_state(P, w)
    t2 = P.TSVD(w.k, 1200, 1000)
    t2.init(w.U0, w.S0, w.V0)
    for b in w.batches:
        H.gpu_apply(P, t1, b)
        t2.update_rows(P.Sparse.from_scipy(b.E))
    assert np.allclose(t1.get_U(), t2.get_U(), atol=1e-14)


def test_init_validation(P):
    t = P.TSVD(2, 4, 4)
    with pytest.raises(P.TsvdError) as ei:
        t.init(np.ones((4, 2)), np.array([2.0, 1.0]), np.eye(4)[:, :2].copy())
    assert ei.value.status == 2
    with pytest.raises(P.TsvdError) as ei:
        t.init(np.eye(4)[:, :2].copy(), np.array([1.0, 2.0]), np.eye(4)[:, :2].copy())
    assert ei.value.status == 3


def test_empty_update_vectors_are_dropped(P):
    """Empty update vectors (21-26 % of a configs[1] row batch) are dropped
    before the Gram / core (their rows of the new factor are zero); weight pairs with an
    empty d_i or e_i contribute d_i e_i^T = 0 and are dropped too."""
    m, n, k, s = 80, 60, 6, 20
    A = synth.random_sparse(m, n, 0.1, seed=11, values="normal")
    U0, S0, V0 = synth.init_truncated_svd(A, k)
    E = synth.random_sparse(s, n, 0.15, seed=12, values="normal").toarray()
    E[[0, 5, 6, 19]] = 0
    D = synth.random_sparse(s, m + s, 0.15, seed=13, values="normal").toarray()
    D[[2, 5]] = 0
    Ew = synth.random_sparse(s, n + s, 0.15, seed=14, values="normal").toarray()
    Dw = synth.random_sparse(s, m + s, 0.15, seed=15, values="normal").toarray()
    Ew[[0, 6]] = 0
    Dw[[2, 5, 19]] = 0
    bs = [synth.Batch("rows", sp.csr_matrix(E)), synth.Batch("cols", sp.csr_matrix(D)),
          synth.Batch("weights", sp.csr_matrix(Ew), sp.csr_matrix(Dw))]
    w = synth.Workload("empty", k, U0, S0, V0, bs)
    t, _ = _stream_parity(P, w)
    assert t.stats()["s_eff"] == s - 5          # pairs 0, 2, 5, 6, 19 have an empty side
    t2 = H.gpu_state(P, w)
    H.gpu_apply(P, t2, w.batches[0])
    assert t2.stats()["s_eff"] == s - 4
    assert np.abs(t2.get_U()[m + np.array([0, 5, 6, 19])]).max() < 1e-15


def test_duplicate_update_vectors_are_merged(P):
    """Identical update vectors (about 10 % of a configs[1] batch's nonempty ones) are merged into
    one vector scaled by sqrt(multiplicity) before the Gram / core: the result is
    the oracle's (which keeps every copy), and the copies' rows of the new factor are equal."""
    m, n, k, s = 90, 70, 6, 24
    A = synth.random_sparse(m, n, 0.1, seed=21, values="normal")
    U0, S0, V0 = synth.init_truncated_svd(A, k)
    E = synth.random_sparse(s, n, 0.15, seed=22, values="normal").toarray()
    E[3] = E[1]
    E[7] = E[1]          # a group of three
    E[10] = E[4]         # a pair
    E[[12, 13]] = 0      # two empty ones
    E[20] = 0
    E[20, 5] = 1.0
    E[21] = E[20]        # a pair of one-nonzero rows (the common duplicate in graph batches)
    D = synth.random_sparse(s, m + s, 0.15, seed=23, values="normal").toarray()
    D[9] = D[2]
    bs = [synth.Batch("rows", sp.csr_matrix(E)), synth.Batch("cols", sp.csr_matrix(D))]
    w = synth.Workload("dups", k, U0, S0, V0, bs)
    _stream_parity(P, w)
    t = H.gpu_state(P, w)
    H.gpu_apply(P, t, w.batches[0])
    assert t.stats()["s_eff"] == s - 2 - 4          # 2 empty rows, 4 merged copies
    U = t.get_U()
    for a, b in [(1, 3), (1, 7), (4, 10), (20, 21)]:
        assert np.abs(U[m + a] - U[m + b]).max() <= 1e-14 * max(1.0, np.abs(U[m + a]).max())


def test_graph_nodeappend_intermediate_rr_path(P):
    """configs[1] recipe at intermediate scale — N = 30k, k = 64, 5 batches of 1500 nodes (rows
    then columns) — large enough that the exact cores exceed 512 columns (the Rayleigh-Ritz
    core reduction of the full-size path), the Gram Cholesky spans several 64-row tiles of the
    tile DAG, duplicates are merged and MII resets fire; every half-update element-wise
    against the oracle (VERDICT r1 'prove parity where the numbers are taken')."""
    w = synth.graph_nodeappend(N=30_000, n_init=15_000, batch=1_500, n_batches=5, k=64)
    t = H.gpu_state(P, w)
    ref = H.run_oracle(w)
    paths, cores, worst = set(), [], 0.0
    for i, b in enumerate(w.batches):
        H.gpu_apply(P, t, b)
        st = t.stats()
        paths.add(st["core_path"])
        cores.append((st["core_rows"], st["core_cols"]))
        Ug, Sg, Vg = H.gpu_factors(t)
        Uo, So, Vo, th = ref[i]
        ok, d = H.compare(Ug, Sg, Vg, Uo, So, Vo, th, w.k)
        worst = max(worst, d["sigma"], d["angle_u"], d["angle_v"])
        assert ok, (i, b.kind, d, st)
    st = t.stats()
    assert 2 in paths, (paths, cores)                 # the Rayleigh-Ritz reduction ran
    assert max(c for _, c in cores) >= 512, cores     # cores as wide as the full-size path's
    assert st["total_resets"] > 0, st                 # MII resets fired (reading R18)
    print("C2-intermediate worst", worst, "cores", cores, "resets", st["total_resets"])


def _near_dependent_rows(eps, n=200, k=10, s=30, m=300, seed=0):
    """A rows update whose vectors 0..5 lie within relative distance eps of span(V_k) and whose
    vectors 10..13 lie within eps of other update vectors (dense rows)."""
    rng = np.random.default_rng(seed)
    A = synth.random_sparse(m, n, 0.1, seed=seed + 1, values="normal")
    U0, S0, V0 = synth.init_truncated_svd(A, k)
    E = synth.random_sparse(s, n, 0.2, seed=seed + 2, values="normal").toarray()
    for i in range(6):
        x = V0 @ rng.standard_normal(k)
        d = rng.standard_normal(n)
        d -= V0 @ (V0.T @ d)
        E[i] = x + eps * np.linalg.norm(x) * d / np.linalg.norm(d)
    for i, j in zip(range(10, 14), range(20, 24)):
        d = rng.standard_normal(n)
        E[i] = E[j] + eps * np.linalg.norm(E[j]) * d / np.linalg.norm(d)
    return synth.Workload("near-dep", k, U0, S0, V0, [synth.Batch("rows", sp.csr_matrix(E))])


def test_near_dependent_update_vectors_kept(P):
    """Update vectors whose component outside span(V_k, the earlier vectors) is 1e-5 of their
    norm: the Gram's Schur diagonal (1e-10 of ||e_i||^2) is
    above the deflation threshold, the direction is kept, and the result matches the oracle's
    Householder QR to the parity bar."""
    w = _near_dependent_rows(1e-5)
    t, _ = _stream_parity(P, w)
    assert t.stats()["rank"][1] == 30


def _deflated_projection(E, V, tau=1e-12):
    """What reading R8 computes for a rows update: in pivot order, an update vector whose
    squared residual outside span(V, earlier kept vectors) is <= tau ||e_i||^2 is replaced by
    its projection onto that span (its residual is dropped).  Plain numpy Gram-Schmidt."""
    E = np.array(E, dtype=np.float64)
    Q = [V[:, j] for j in range(V.shape[1])]
    out = E.copy()
    for i in range(E.shape[0]):
        e = E[i]
        r = e.copy()
        for _ in range(2):
            for q in Q:
                r -= q * (q @ r)
        if r @ r <= tau * (e @ e):
            out[i] = e - r
        else:
            Q.append(r / np.linalg.norm(r))
    return out


def test_near_dependent_update_vectors_deflated(P):
    """Relative residual 1e-7: below what a Gram can resolve (its rounding noise is ~1e-12 of
    ||e_i||^2 against a Schur diagonal of 1e-14), so reading R8 deflates the direction — the
    SV-LCOV tuple algebra of the paper shares the floor (alpha = sqrt(b.b - c.c), Alg 2 line 5,
    PAPER.md:260).  The update then equals the exact update of E with those residuals dropped
    (oracle on the projected block, parity bar), and differs from the exact update of E by the
    dropped part only (1e-7 relative)."""
    w = _near_dependent_rows(1e-7)
    b = w.batches[0]
    t = H.gpu_state(P, w)
    H.gpu_apply(P, t, b)
    assert t.stats()["rank"][1] == 20              # the 10 near-dependent vectors deflated
    Ug, Sg, Vg = H.gpu_factors(t)
    Ep = sp.csr_matrix(_deflated_projection(b.E.toarray(), w.V0))
    Uo, So, Vo, th = zha_simon.add_rows(w.U0, w.S0, w.V0, Ep)
    ok, d = H.compare(Ug, Sg, Vg, Uo, So, Vo, th, w.k)
    assert ok, d
    Uo, So, Vo, th = zha_simon.add_rows(w.U0, w.S0, w.V0, b.E)
    assert metrics.sigma_relerr(Sg, So) < 1e-8

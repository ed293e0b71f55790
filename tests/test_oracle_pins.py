"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

None of these re-run the oracle's own formula: each checks it against brute force
(Def 2 by a full dense SVD of the explicitly updated matrix), exactness, an energy
identity, a closed form, a hand-derived worked example (tests/golden/), or a different
algorithm the paper says gives the same result (Alg 1 vs Alg 2 vs Householder vs
Cholesky; Eq (1) vs Eq (2); a variant at l = s vs the exact update).
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import metrics, steps, svlcov, variants, zha_simon
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


# ----------------------------------------------------------------------------- helpers
def _state(m, n, k, density, seed, full_rank_init=False):
    """A random sparse A with its exact SVD_k as the maintained state."""
    A = synth.random_sparse(m, n, density, seed, values="normal").toarray()
    u, s, vt = np.linalg.svd(A, full_matrices=False)
    return A, u[:, :k], s[:k], vt[:k].T


def _brute(Abar, k):
    u, s, vt = np.linalg.svd(Abar, full_matrices=False)
    return u[:, :k], s[:k], vt[:k].T, s


def _check_against_brute(Un, Sn, Vn, th, Abar, k, tol_s=1e-12, tol_ang=1e-10):
    Ub, Sb, Vb, sall = _brute(Abar, k)
    assert metrics.sigma_relerr(Sn, Sb) <= tol_s
    kk = metrics.gap_rank(sall, k)
    if kk:
        assert metrics.sin_theta(Un[:, :kk], Ub[:, :kk]) <= tol_ang
        assert metrics.sin_theta(Vn[:, :kk], Vb[:, :kk]) <= tol_ang
    # full core spectrum = the nonzero spectrum of the updated matrix (rank <= k+s)
    nz = sall[sall > 1e-10 * sall[0]]
    assert np.allclose(th[:nz.size], nz, rtol=1e-11, atol=1e-12 * sall[0])
    assert np.all(th[nz.size:] <= 1e-9 * sall[0])
    assert metrics.orth_err(Un) < 1e-13 and metrics.orth_err(Vn) < 1e-13
    assert np.all(np.diff(Sn) <= 1e-15 * Sn[0]) and np.all(Sn >= 0)


SHAPES = [(40, 30, 5, 4, 0.15), (30, 50, 6, 8, 0.2), (25, 20, 8, 12, 0.3), (60, 60, 3, 1, 0.05)]


# ----------------------------------------------------------------------------- metrics
@pytest.mark.parametrize("theta", [1e-13, 1e-9, 1e-4, 0.3, 1.2])
def test_sin_theta_closed_form(theta):
    """sin of the angle between e1 and (cos t) e1 + (sin t) e2 is sin t (closed form),
    also far below the 1.5e-8 floor of sqrt(1 - cos^2)."""
    X = np.zeros((5, 1)); X[0, 0] = 1
    Y = np.zeros((5, 1)); Y[0, 0] = np.cos(theta); Y[1, 0] = np.sin(theta)
    assert abs(metrics.sin_theta(X, Y) - np.sin(theta)) <= 1e-15 + 1e-12 * np.sin(theta)


def test_sigma_relerr_closed_form():
    assert metrics.sigma_relerr([2.0, 1.0 + 1e-11], [2.0, 1.0]) == pytest.approx(1e-11, rel=1e-4)
    # |Δσ_i| <= max(1e-10 σ_i, 1e-13 σ_1) passes the 1e-10 bar
    assert metrics.sigma_relerr([1.0, 0.0], [1.0, 5e-14]) == pytest.approx(5e-11, rel=1e-9)   # 5e-14 <= 1e-13
    assert metrics.sigma_relerr([1.0, 0.0], [1.0, 2e-13]) == pytest.approx(2e-10, rel=1e-9)   # 2e-13 > 1e-13
    # σ_i = 1e-4 σ_1: a 1e-6 relative error (1e-10 σ_1 absolute) fails, 1e-10 relative passes
    assert metrics.sigma_relerr([1.0, 1e-4 * (1 + 1e-6)], [1.0, 1e-4]) == pytest.approx(1e-7, rel=1e-6)
    assert metrics.sigma_relerr([1.0, 1e-2 * (1 + 1e-11)], [1.0, 1e-2]) == pytest.approx(1e-11, rel=1e-4)
    assert metrics.gap_rank([3, 2, 2, 1], 2) == 1 and metrics.gap_rank([3, 2, 1], 2) == 2


# ----------------------------------------------------------------------------- brute force (Def 2)
@pytest.mark.parametrize("m,n,k,s,dens", SHAPES)
def test_add_rows_brute_force(m, n, k, s, dens):
    """Theorem 1 Add rows with Def 2: result = SVD_k([Ã; E_r])."""
    A, U, S, V = _state(m, n, k, dens, seed=m + n + s)
    Er = synth.random_sparse(s, n, dens, seed=7 * s + 1, values="normal")
    Un, Sn, Vn, th = zha_simon.add_rows(U, S, V, Er)
    Abar = np.vstack([zha_simon.reconstruct(U, S, V), Er.toarray()])
    _check_against_brute(Un, Sn, Vn, th, Abar, k)


@pytest.mark.parametrize("m,n,k,s,dens", SHAPES)
def test_add_columns_brute_force(m, n, k, s, dens):
    """Theorem 1 Add columns: SVD_k([Ã, E_c])."""
    A, U, S, V = _state(m, n, k, dens, seed=3 * m + n + s)
    EcT = synth.random_sparse(s, m, dens, seed=11 * s + 2, values="normal")
    Un, Sn, Vn, th = zha_simon.add_columns(U, S, V, EcT)
    Abar = np.hstack([zha_simon.reconstruct(U, S, V), EcT.toarray().T])
    _check_against_brute(Un, Sn, Vn, th, Abar, k)


@pytest.mark.parametrize("m,n,k,s,dens", SHAPES)
def test_update_weights_brute_force(m, n, k, s, dens):
    """Theorem 1 Update weights: SVD_k(Ã + D E_m^T)."""
    A, U, S, V = _state(m, n, k, dens, seed=5 * m + n + s)
    DT = synth.random_sparse(s, m, dens, seed=13 * s + 3, values="normal")
    EmT = synth.random_sparse(s, n, dens, seed=17 * s + 4, values="normal")
    Un, Sn, Vn, th = zha_simon.update_weights(U, S, V, DT, EmT)
    Abar = zha_simon.reconstruct(U, S, V) + DT.toarray().T @ EmT.toarray()
    Ub, Sb, Vb, sall = _brute(Abar, k)
    assert metrics.sigma_relerr(Sn, Sb) <= 1e-12
    kk = metrics.gap_rank(sall, k)
    if kk:
        assert metrics.sin_theta(Un[:, :kk], Ub[:, :kk]) <= 1e-10
        assert metrics.sin_theta(Vn[:, :kk], Vb[:, :kk]) <= 1e-10
    assert metrics.orth_err(Un) < 1e-13 and metrics.orth_err(Vn) < 1e-13


def test_rank_deficient_updates_brute_force():
    """Empty and duplicate update vectors (the normal case on graphs):
    Householder R gets a ~0 diagonal, the result stays Def 2's."""
    A, U, S, V = _state(50, 40, 6, 0.2, seed=99)
    Er = synth.random_sparse(6, 40, 0.2, seed=5, values="normal").toarray()
    Er[2] = 0.0
    Er[4] = Er[1]
    Er[5] = 2.0 * Er[0] - Er[3]
    Er = sp.csr_matrix(Er)
    Un, Sn, Vn, th = zha_simon.add_rows(U, S, V, Er)
    Abar = np.vstack([zha_simon.reconstruct(U, S, V), Er.toarray()])
    _check_against_brute(Un, Sn, Vn, th, Abar, 6)


# ----------------------------------------------------------------------------- exactness
def test_exactness_low_rank():
    """BASELINE.json north_star: if rank(A) <= k and the init is A's exact SVD, the update
    is the TRUE truncated SVD of Ā, the full core spectrum is Ā's nonzero spectrum
    (rank <= k+s) and the untruncated factors reconstruct Ā (Eq (1) is an exact
    factorisation)."""
    rng = np.random.default_rng(3)
    m, n, k, s = 60, 45, 5, 3
    A = rng.standard_normal((m, k)) @ rng.standard_normal((k, n))
    u, sv, vt = np.linalg.svd(A, full_matrices=False)
    U, S, V = u[:, :k], sv[:k], vt[:k].T
    Er = sp.csr_matrix(rng.standard_normal((s, n)) * (rng.random((s, n)) < 0.3))
    Abar = np.vstack([A, Er.toarray()])
    for kk in (k, k + 2):
        # pad the state with zero singular triplets to ask for more than rank(A)
        if kk > k:
            Up = np.hstack([U, np.linalg.qr(np.hstack([U, rng.standard_normal((m, kk - k))]))[0][:, k:]])
            Vp = np.hstack([V, np.linalg.qr(np.hstack([V, rng.standard_normal((n, kk - k))]))[0][:, k:]])
            Sp = np.concatenate([S, np.zeros(kk - k)])
        else:
            Up, Sp, Vp = U, S, V
        Un, Sn, Vn, th = zha_simon.add_rows(Up, Sp, Vp, Er)
        true = np.linalg.svd(Abar, compute_uv=False)
        assert np.allclose(Sn, true[:kk], rtol=1e-12, atol=1e-12 * true[0])
        assert np.allclose(th[:k + s], true[:k + s], rtol=1e-12)
    # untruncated reconstruction: rebuild with all k+s triplets
    C0 = V.T @ Er.toarray().T
    Z = Er.toarray().T - V @ C0
    Q, R = np.linalg.qr(Z)
    K = np.block([[np.diag(S), np.zeros((k, Q.shape[1]))], [C0.T, R.T]])
    F, t, Gt = np.linalg.svd(K)
    Ufull = np.block([[U, np.zeros((m, s))], [np.zeros((s, k)), np.eye(s)]]) @ F
    Vfull = np.hstack([V, Q]) @ Gt.T
    assert np.allclose((Ufull * t) @ Vfull.T, Abar, atol=1e-12 * np.abs(Abar).max())


# ----------------------------------------------------------------------------- energy
@pytest.mark.parametrize("kind", ["rows", "cols"])
def test_energy_identity(kind):
    """Σ_all θ² = ||Σ||² + ||E||_F² : the core is an orthogonal transform of [Ã; E]
    (Eq (1) factorisation), and the Eckart–Young residual
    ||Ā - U Θ V^T||_F² = Σ_{i>k} θ_i²."""
    A, U, S, V = _state(45, 35, 6, 0.2, seed=21)
    dim = 35 if kind == "rows" else 45
    E = synth.random_sparse(7, dim, 0.25, seed=8, values="normal")
    f = zha_simon.add_rows if kind == "rows" else zha_simon.add_columns
    Un, Sn, Vn, th = f(U, S, V, E)
    assert np.isclose((th ** 2).sum(), (S ** 2).sum() + (E.data ** 2).sum(), rtol=1e-13)
    At = zha_simon.reconstruct(U, S, V)
    Abar = np.vstack([At, E.toarray()]) if kind == "rows" else np.hstack([At, E.toarray().T])
    res = np.linalg.norm(Abar - zha_simon.reconstruct(Un, Sn, Vn)) ** 2
    assert np.isclose(res, (th[6:] ** 2).sum(), rtol=1e-10, atol=1e-24)


# ----------------------------------------------------------------------------- Eq (1) vs Eq (2)
def test_add_rows_equals_weight_update_on_padded_state():
    """[Ã; E_r] = [Ã; 0] + [0; I] E_r: Eq (1) on the transpose and Eq (2) must agree
    (two different factorisations of the same Def 2 target)."""
    A, U, S, V = _state(30, 25, 5, 0.2, seed=4)
    Er = synth.random_sparse(4, 25, 0.3, seed=6, values="normal")
    Un, Sn, Vn, _ = zha_simon.add_rows(U, S, V, Er)
    Up = np.vstack([U, np.zeros((4, 5))])
    DT = sp.csr_matrix(np.hstack([np.zeros((4, 30)), np.eye(4)]))
    Uw, Sw, Vw, _ = zha_simon.update_weights(Up, S, V, DT, Er)
    assert metrics.sigma_relerr(Sn, Sw) < 1e-13
    assert metrics.sin_theta(Un, Uw) < 1e-11 and metrics.sin_theta(Vn, Vw) < 1e-11


# ----------------------------------------------------------------------------- worked examples
def test_golden_svlcov_qr_disjoint():
    g = GOLD["svlcov_qr_disjoint"]
    U = np.array(g["U_cols"], float).T
    E = np.array(g["E_cols"], float).T
    B, C, R, keep = svlcov.alg2_svlcov_qr(E, U)
    assert np.array_equal(R, np.array(g["R"], float)) and keep.all()
    Rc, kc = steps.chol_deflate(steps.svlcov_gram(sp.csr_matrix(E.T), (E.T @ U)), (E ** 2).sum(0))
    assert np.allclose(Rc, np.array(g["R"], float), atol=0)


def test_golden_lift_examples():
    g = GOLD["lift_examples"]
    X = np.array(g["X"], float)
    for c in g["cases"]:
        b = np.zeros(3); b[c["b_index"]] = c["b_value"]
        _, cc = svlcov.lift(b[:, None], X)
        assert np.array_equal(cc[:, 0], np.array(c["c"], float))
        W, C0T = steps.lift(sp.csr_matrix(b[None, :]), X, np.eye(2))
        assert np.array_equal(C0T[0], np.array(c["c"], float))


def test_golden_append_e3():
    g = GOLD["append_e3_to_diag32"]
    A = np.array(g["A"], float)
    u, s, vt = np.linalg.svd(A, full_matrices=False)
    EcT = sp.csr_matrix(np.array([g["Ec_col"]], float))
    Un, Sn, Vn, th = zha_simon.add_columns(u, s, vt.T, EcT)
    assert np.allclose(Sn, g["sigma"], atol=1e-15)
    assert np.allclose(sorted(th, reverse=True), [3, 2, 1], atol=1e-15)


def test_golden_rank1_cancel():
    g = GOLD["rank1_cancel"]
    d = np.array(g["A_diag"], float)
    U = np.eye(3); V = np.eye(3); k = g["k"]; i = g["cancel_index"]
    DT = sp.csr_matrix((-d[i] * U[:, i])[None, :])
    EmT = sp.csr_matrix(V[:, i][None, :])
    Un, Sn, Vn, th = zha_simon.update_weights(U, d, V, DT, EmT)
    assert np.allclose(Sn, g["sigma"], atol=1e-14)


@pytest.mark.parametrize("kind", ["rows", "cols"])
def test_golden_zero_update(kind):
    g = GOLD["zero_update"]
    d = np.array(g["A_diag"], float)
    U = np.eye(3)[:, :2]; V = np.eye(2)
    E = sp.csr_matrix((1, 2 if kind == "rows" else 3))
    f = zha_simon.add_rows if kind == "rows" else zha_simon.add_columns
    Un, Sn, Vn, th = f(U, d, V, E)
    assert np.allclose(Sn, g["sigma"], atol=1e-15)
    newrow = Un[-1] if kind == "rows" else Vn[-1]
    assert np.allclose(newrow, 0, atol=1e-15)


# ----------------------------------------------------------------------------- SV-LCOV
def test_lemma3_isometry():
    """Lemma 3: <(b1,c1),(b2,c2)> = ((I-UU^T)b1) . ((I-UU^T)b2)."""
    rng = np.random.default_rng(0)
    for trial in range(200):
        m, k = rng.integers(5, 60), rng.integers(1, 5)
        U = synth.random_orthonormal(m, k, seed=trial)
        b = synth.random_sparse(m, 2, 0.3, seed=1000 + trial, values="normal").toarray()
        B, C = svlcov.lift(b, U)
        z = b - U @ (U.T @ b)
        lhs = svlcov.dot(B[:, 0], C[:, 0], B[:, 1], C[:, 1])
        assert abs(lhs - z[:, 0] @ z[:, 1]) <= 1e-12 * (1 + np.abs(b).sum() ** 2)
        assert np.allclose(svlcov.materialize(B[:, 0], C[:, 0], U), z[:, 0], atol=1e-14)


def test_alg2_equals_alg1_and_householder():
    """Alg 2 (tuples) = Alg 1 (dense MGS) = Householder R with rows sign-normalised
    (same QR of a full-rank matrix)."""
    for seed in range(20):
        m, k, s = 40, 4, 6
        U = synth.random_orthonormal(m, k, seed)
        E = synth.random_sparse(m, s, 0.3, 50 + seed, values="normal").toarray()
        if np.linalg.matrix_rank(E - U @ (U.T @ E)) < s:
            continue
        _, _, R2, keep = svlcov.alg2_svlcov_qr(E, U)
        Q1, R1 = svlcov.alg1_mgs(E, U)
        _, Rh = np.linalg.qr(E - U @ (U.T @ E))
        Rh = Rh * np.sign(np.diag(Rh))[:, None]
        assert keep.all()
        assert np.allclose(R2, R1, atol=1e-12) and np.allclose(R2, Rh, atol=1e-12)
        B, C, _, _ = svlcov.alg2_svlcov_qr(E, U)
        Q2 = B - U @ C
        assert np.allclose(Q2, Q1, atol=1e-11)
        assert metrics.orth_err(np.hstack([U, Q2])) < 1e-12


def test_chol_deflate_equals_alg2_with_deflation():
    """Cholesky of the SV-LCOV Gram with deflation (R8) reproduces Alg 2's R,
    including empty / duplicate / dependent update vectors."""
    for seed in range(15):
        m, k, s = 50, 5, 8
        U = synth.random_orthonormal(m, k, seed)
        E = synth.random_sparse(m, s, 0.25, 80 + seed, values="normal").toarray()
        E[:, 2] = 0.0
        E[:, 5] = E[:, 1]
        E[:, 7] = E[:, 0] - 3 * E[:, 3]
        E[:, 6] = U @ np.arange(1.0, k + 1)        # inside span(U): projects to 0
        ET = sp.csr_matrix(E.T)
        C0T = E.T @ U
        R, keep = steps.chol_deflate(steps.svlcov_gram(ET, C0T), (E ** 2).sum(0))
        _, _, R2, keep2 = svlcov.alg2_svlcov_qr(E, U)
        assert np.array_equal(keep, keep2)
        assert keep.sum() == np.linalg.matrix_rank(E - U @ (U.T @ E), tol=1e-8)
        assert np.allclose(R, R2, atol=1e-10)
        Z = E - U @ (U.T @ E)
        assert np.allclose(R.T @ R, Z.T @ Z, atol=1e-11)


def test_chol_deflate_full_rank_is_cholesky():
    rng = np.random.default_rng(1)
    X = rng.standard_normal((30, 9))
    G = X.T @ X
    R, keep = steps.chol_deflate(G, np.ones(9))
    assert keep.all() and np.allclose(R, np.linalg.cholesky(G).T, atol=1e-13)


def test_sparse_gram_brute_force():
    E = synth.random_sparse(7, 20, 0.3, 3, values="normal")
    G = steps.sparse_gram(E)
    Ed = E.toarray()
    for i in range(7):
        for j in range(7):
            assert abs(G[i, j] - sum(Ed[i, t] * Ed[j, t] for t in range(20))) < 1e-14


def test_method_chain_matches_brute_force():
    """The method's own chain in plain form — lift, SV-LCOV Gram, Cholesky with deflation,
    Alg 9 core — has the spectrum of [Ã; E_r] (Def 2), with duplicates and empty rows."""
    A, U, S, V = _state(40, 35, 5, 0.2, seed=31)
    Er = synth.random_sparse(9, 35, 0.2, seed=32, values="normal").toarray()
    Er[3] = 0; Er[6] = Er[2]
    Er = sp.csr_matrix(Er)
    W, C0T = steps.lift(Er, V, np.eye(5))
    R, keep = steps.chol_deflate(steps.svlcov_gram(Er, C0T), np.asarray(Er.multiply(Er).sum(1)).ravel())
    K = steps.core_rows(S, C0T, R, keep)
    th = np.linalg.svd(K, compute_uv=False)
    sall = np.linalg.svd(np.vstack([zha_simon.reconstruct(U, S, V), Er.toarray()]), compute_uv=False)
    assert np.allclose(th, sall[:th.size], rtol=1e-11, atol=1e-12 * sall[0])


def test_core_weights_matches_brute_force():
    A, U, S, V = _state(30, 28, 4, 0.2, seed=41)
    DT = synth.random_sparse(3, 30, 0.2, 42, values="normal")
    EmT = synth.random_sparse(3, 28, 0.2, 43, values="normal")
    _, PD = steps.lift(DT, U, np.eye(4))
    _, PE = steps.lift(EmT, V, np.eye(4))
    RD, kD = steps.chol_deflate(steps.svlcov_gram(DT, PD), np.asarray(DT.multiply(DT).sum(1)).ravel())
    RE, kE = steps.chol_deflate(steps.svlcov_gram(EmT, PE), np.asarray(EmT.multiply(EmT).sum(1)).ravel())
    K = steps.core_weights(S, PD, RD, kD, PE, RE, kE)
    th = np.linalg.svd(K, compute_uv=False)
    sall = np.linalg.svd(zha_simon.reconstruct(U, S, V) + DT.toarray().T @ EmT.toarray(), compute_uv=False)
    assert np.allclose(th, sall[:th.size], rtol=1e-11, atol=1e-12 * sall[0])


def test_cond1_closed_form():
    assert steps.cond1(np.diag([4.0, 2.0, 0.5])) == pytest.approx(8.0)


# ----------------------------------------------------------------------------- variants
def _Z(U, ET):
    return ET.toarray().T - U @ (U.T @ ET.toarray().T)


@pytest.mark.parametrize("mode", ["rpi", "gkl"])
def test_variant_full_width_equals_exact(mode):
    """With l = s = rank(Z) the approximate augmented space is the exact one, so the
    variants equal the exact update (P:426 'same output' + P:423)."""
    A, U, S, V = _state(40, 36, 4, 0.25, seed=51)
    s = 5
    Er = synth.random_sparse(s, 36, 0.3, 52, values="normal")
    EcT = synth.random_sparse(s, 40, 0.3, 53, values="normal")
    sk = synth.gaussian_sketch(54, s, s) if mode == "rpi" else synth.unit_vector(54, s)
    for f_ex, f_ap, E in ((zha_simon.add_rows, variants.add_rows, Er),
                          (zha_simon.add_columns, variants.add_columns, EcT)):
        Ue, Se, Ve, the = f_ex(U, S, V, E)
        Ua, Sa, Va, tha = f_ap(U, S, V, E, mode, sk, l=s, t=2)
        assert metrics.sigma_relerr(Sa, Se) < 1e-10
        kk = metrics.gap_rank(the, 4)
        assert metrics.sin_theta(Ua[:, :kk], Ue[:, :kk]) < 1e-9
        assert metrics.sin_theta(Va[:, :kk], Ve[:, :kk]) < 1e-9
    DT = synth.random_sparse(s, 40, 0.3, 55, values="normal")
    skD = synth.gaussian_sketch(56, s, s) if mode == "rpi" else synth.unit_vector(56, s)
    Ue, Se, Ve, the = zha_simon.update_weights(U, S, V, DT, Er)
    Ua, Sa, Va, tha = variants.update_weights(U, S, V, DT, Er, mode, skD, sk, l=s, t=2)
    assert metrics.sigma_relerr(Sa, Se) < 1e-10


@pytest.mark.parametrize("mode", ["rpi", "gkl"])
def test_variant_QtZ_equals_Pt(mode):
    """Q is orthonormal and Q^T Z = P^T (H read as l x (l+1))."""
    m, k, s, l = 80, 5, 30, 10
    U = synth.random_orthonormal(m, k, 61)
    ET = synth.random_sparse(s, m, 0.15, 62, values="normal")
    op = variants.AugmentedOp(U, ET)
    if mode == "rpi":
        Q, P = variants.rpi_dense(op, synth.gaussian_sketch(63, s, l), 3)
    else:
        Q, P = variants.gkl_dense(op, synth.unit_vector(63, s), l)
    Z = _Z(U, ET)
    assert metrics.orth_err(Q) < 1e-12
    assert np.abs(U.T @ Q).max() < 1e-12
    assert np.allclose(Q.T @ Z, P.T, atol=1e-12 * np.abs(Z).max())


def test_rpi_converges_to_dominant_subspace():
    """RPI with many iterations captures the dominant l-dimensional left subspace of Z
    (SPEC.md:187 example, DERIVED) — closed form via the dense SVD of Z."""
    m, k, s, l = 60, 3, 20, 4
    U = synth.random_orthonormal(m, k, 71)
    rng = np.random.default_rng(72)
    ET = sp.csr_matrix(rng.standard_normal((s, m)) * (rng.random((s, m)) < 0.5))
    op = variants.AugmentedOp(U, ET)
    Q, P = variants.rpi_dense(op, synth.gaussian_sketch(73, s, l), 200)
    uz, sz, _ = np.linalg.svd(_Z(U, ET), full_matrices=False)
    assert (sz[l - 1] - sz[l]) / sz[0] > 1e-3
    assert metrics.sin_theta(Q, uz[:, :l]) < 1e-6


def test_synth_determinism():
    a = synth.tiny_rowappend()
    b = synth.tiny_rowappend()
    assert np.array_equal(a.U0, b.U0) and all((x.E != y.E).nnz == 0 for x, y in zip(a.batches, b.batches))

"""Parity of the approximate-augmented-space variants (-m gpu): RPI (Alg 8)
and GKL (Alg 6) with the App D.3 updates, CUDA path
through the C-ABI vs the dense oracle (oracle/variants.py: Alg 7 / Alg 5 on the densified
operator Z) on identical seeded inputs and identical start blocks."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import metrics, variants
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


MODES = {"rpi": 2, "gkl": 1}


def _sketch(mode, seed, s, l):
    return synth.gaussian_sketch(seed, s, l) if mode == "rpi" else synth.unit_vector(seed, s)


def test_k12_matches_spec(P):
    """K12 on the device equals the numpy implementation of the same spec."""
    s, l = 1000, 37
    for side in (0, 1):
        out = torch.empty(s, l, dtype=torch.float64, device="cuda")
        P.k_gaussian(12345, side, s, l, out)
        ref = synth.counter_gaussian(12345, side, s, l)
        assert np.allclose(out.cpu().numpy(), ref, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("mode", ["rpi", "gkl"])
@pytest.mark.parametrize("s,l", [(40, 8), (120, 37), (300, 64)])
def test_basis_properties_and_oracle(P, mode, s, l):
    """Q = B' - X C' is orthonormal, Q^T Z = P^T (PAPER.md:835 / 900), and Q P^T (basis
    independent: the projection of Z onto range(Q)) equals the dense oracle's."""
    d, k = 400, 12
    X = synth.random_orthonormal(d, k, seed=s)
    ET = synth.random_sparse(s, d, 0.03, seed=s + 1, values="normal")
    sk = _sketch(mode, 7 + s, s, l)
    t = 3
    opts = P.make_opts(mode=MODES[mode], l=l, t=t, sketch=torch.from_numpy(np.ascontiguousarray(sk)).cuda())
    BJ = torch.zeros(d, l, dtype=torch.float64, device="cuda")
    Cp = torch.zeros(k, l, dtype=torch.float64, device="cuda")
    Pm = torch.zeros(s, l, dtype=torch.float64, device="cuda")
    P.k_approx_basis(P.Sparse.from_scipy(ET, device="cuda"), torch.from_numpy(X).cuda(), k, opts, 1, BJ, Cp, Pm)
    B, Cc, Pg = BJ.cpu().numpy(), Cp.cpu().numpy(), Pm.cpu().numpy()
    Q = B - X @ Cc
    Z = ET.toarray().T - X @ (X.T @ ET.toarray().T)
    live = np.linalg.norm(Q, axis=0) > 0.5
    assert metrics.orth_err(Q[:, live]) < 1e-11
    assert np.allclose(Q.T @ Z, Pg.T, atol=1e-11 * max(1.0, np.abs(Z).max()))
    Zop = variants.AugmentedOp(X, ET)
    Qo, Po = (variants.rpi_dense(Zop, sk, t) if mode == "rpi" else variants.gkl_dense(Zop, sk, l))
    assert np.allclose(Q @ Pg.T, Qo @ Po.T, atol=1e-9 * np.abs(Qo @ Po.T).max())


def _variant_stream(P, w, mode, l, t, use_seed=False):
    """Run w through the CUDA path and the dense-variant oracle with the same start blocks."""
    tg = H.gpu_state(P, w)
    U, S, V = w.U0.copy(), w.S0.copy(), w.V0.copy()
    worst = 0.0
    for bi, b in enumerate(w.batches):
        s = b.s
        seed = 1000 + bi
        if b.kind == "weights":
            if use_seed:
                skD = synth.counter_gaussian(seed, 0, s, l if mode == "rpi" else 1)
                skE = synth.counter_gaussian(seed, 1, s, l if mode == "rpi" else 1)
            else:
                skD, skE = _sketch(mode, seed, s, l), _sketch(mode, seed + 50, s, l)
            if mode == "gkl":
                skD, skE = skD.ravel(), skE.ravel()
            sk = np.concatenate([skD.ravel(), skE.ravel()])
            U, S, V, th = variants.update_weights(U, S, V, b.D, b.E, mode, skD, skE, l=l, t=t)
        else:
            side = 1 if b.kind == "rows" else 0
            if use_seed:
                sk = synth.counter_gaussian(seed, side, s, l if mode == "rpi" else 1)
                if mode == "gkl":
                    sk = sk.ravel()
            else:
                sk = _sketch(mode, seed, s, l)
            fn = variants.add_rows if b.kind == "rows" else variants.add_columns
            U, S, V, th = fn(U, S, V, b.E, mode, sk, l=l, t=t)
        if use_seed:
            opts = P.make_opts(mode=MODES[mode], l=l, t=t, seed=seed)
        else:
            opts = P.make_opts(mode=MODES[mode], l=l, t=t, sketch=np.ascontiguousarray(sk, dtype=np.float64))
        H.gpu_apply(P, tg, b, opts)
        Ug, Sg, Vg = H.gpu_factors(tg)
        ok, d = H.compare(Ug, Sg, Vg, U, S, V, th, w.k)
        assert ok, (bi, b.kind, d, tg.stats())
        assert metrics.orth_err(Ug) < 1e-9 and metrics.orth_err(Vg) < 1e-9
        worst = max(worst, d["sigma"], d["angle_u"], d["angle_v"])
    return worst


@pytest.mark.parametrize("mode", ["rpi", "gkl"])
@pytest.mark.parametrize("kind", ["rows", "cols", "weights"])
def test_variant_updates_small(P, mode, kind):
    m, n, k, s, l = 90, 70, 8, 30, 10
    A = synth.random_sparse(m, n, 0.08, seed=m + s, values="normal")
    U0, S0, V0 = synth.init_truncated_svd(A, k)
    if kind == "rows":
        bs = [synth.Batch("rows", synth.random_sparse(s, n, 0.1, 5 + i, values="normal")) for i in range(2)]
    elif kind == "cols":
        bs = [synth.Batch("cols", synth.random_sparse(s, m, 0.1, 5 + i, values="normal")) for i in range(2)]
    else:
        bs = [synth.Batch("weights", synth.random_sparse(s, n, 0.1, 5, values="normal"),
                          synth.random_sparse(s, m, 0.1, 6, values="normal"))]
    w = synth.Workload("v", k, U0, S0, V0, bs)
    _variant_stream(P, w, mode, l, 3)


@pytest.mark.parametrize("mode", ["rpi", "gkl"])
def test_variant_counter_generator_path(P, mode):
    """sketch = NULL: the library draws the start block with K12 from the seed; the oracle
    uses the numpy implementation of the same spec."""
    w = synth.tiny_rowappend(n_batches=2)
    _variant_stream(P, w, mode, 20, 3, use_seed=True)


def test_rpi_weights_reduced_c4(P):
    """configs[3] recipe at reduced scale: Chung-Lu weight updates, D one-hot, RPI."""
    w = synth.weights_rpi(N=3000, avg_deg=20, k=16, changes=600, n_batches=2)
    _variant_stream(P, w, "rpi", 48, 3)


def test_rpi_full_width_equals_exact(P):
    """l >= s: the RPI range is the whole augmented space, so the update is the exact one
    (PAPER.md:426 'same as'); GPU RPI vs oracle exact."""
    from oracle import zha_simon
    w = synth.tiny_rowappend(n_batches=1)
    b = w.batches[0]
    tg = H.gpu_state(P, w)
    H.gpu_apply(P, tg, b, P.make_opts(mode=2, l=b.s, t=2, seed=3))
    U, S, V, th = zha_simon.add_rows(w.U0, w.S0, w.V0, b.E)
    ok, d = H.compare(*H.gpu_factors(tg), U, S, V, th, w.k)
    assert ok, d


def test_rpi_rows_reduced_c5(P):
    """configs[4] recipe at reduced scale (power-law row degrees, Zipf columns, RPI row
    append), against the dense RPI oracle with the same start blocks."""
    w = synth.scaleout_rowappend(m=6000, n=3000, k=32, batch=600, n_batches=2, deg_max=2000)
    _variant_stream(P, w, "rpi", 64, 3)


def test_rpi_rows_c5_real_l_and_k(P):
    """configs[4] at its real l = 256 and k = 256 on a reduced matrix (24k x 6k, batches of 1500
    rows): the same kernels as the full size run — the (k+s) x (k+l) = 1756 x 512 tall core through
    Cholesky-QR2 and the cluster-resident Jacobi K9 on 512 columns, the 256-wide RPI gathers,
    l = 256 Cholesky-QR passes — against the dense RPI oracle with the same start blocks."""
    w = synth.scaleout_rowappend(m=24_000, n=6_000, k=256, batch=1_500, n_batches=2, deg_max=6_000)
    tg = H.gpu_state(P, w)
    U, S, V = w.U0.copy(), w.S0.copy(), w.V0.copy()
    for bi, b in enumerate(w.batches):
        sk = synth.counter_gaussian(1000 + bi, 1, b.s, 256)
        U, S, V, th = variants.add_rows(U, S, V, b.E, "rpi", sk, l=256, t=3)
        H.gpu_apply(P, tg, b, P.make_opts(mode=P.RPI, l=256, t=3, seed=1000 + bi))
        st = tg.stats()
        assert (st["core_rows"], st["core_cols"]) == (256 + b.s, 512) and st["core_path"] == 1, st
        ok, d = H.compare(*H.gpu_factors(tg), U, S, V, th, w.k)
        assert ok, (bi, d, st)


def test_rpi_rows_reduced_c5_sharded(P):
    """The same stream on 4 virtual row shards (the scale-out layout of configs[4])."""
    from tests.test_gpu_shard import _stream
    w = synth.scaleout_rowappend(m=6000, n=3000, k=32, batch=600, n_batches=2, deg_max=2000)
    _stream(P, w, dict(world=4, virtual=True, block=256), mode="rpi", l=64, t_it=3)

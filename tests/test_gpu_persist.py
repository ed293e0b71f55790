"""F4 on the GPU (-m gpu): tsvd_save / tsvd_load and the CLI.  A saved and re-loaded state
writes the same bytes again ("save→load→save byte-identical"), including after MII
resets deferred on an append-only side; a stream interrupted by save/load continues to the same
factors as the uninterrupted one; corrupt / foreign files are rejected without touching the
context; the CLI's init + update + query match the library called directly and the oracle."""
import json
import os

import numpy as np
import pytest
import scipy.io
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


def _stream(P, n_batches, reset_cond=1e4):
    w = synth.tiny_rowappend(n_batches=n_batches)
    t = H.gpu_state(P, w)
    opts = P.make_opts(reset_cond=reset_cond)
    return w, t, opts


def test_save_load_save_byte_identical(P, tmp_path):
    # reset threshold 1.0: every update resets (U' resets of the append side stay deferred)
    w, t, opts = _stream(P, 4, reset_cond=1.0)
    for b in w.batches:
        H.gpu_apply(P, t, b, opts)
    assert t.stats()["total_resets"] > 0
    a, b2 = tmp_path / "a.tsvd", tmp_path / "b.tsvd"
    U1, S1, V1 = t.get_U(), t.get_S(), t.get_V()
    t.save(str(a))
    assert not os.path.exists(str(a) + ".tmp")
    m, n, k = t.dims()
    assert P.state_info(str(a)) == (k, m, n)
    assert os.path.getsize(a) == 64 + 8 * (m * k + n * k + 2 * k * k + k)
    u = P.TSVD.from_file(str(a))
    u.save(str(b2))
    assert a.read_bytes() == b2.read_bytes()
    assert np.array_equal(u.get_U(), U1) and np.array_equal(u.get_S(), S1) and np.array_equal(u.get_V(), V1)


def test_interrupted_stream_continues(P, tmp_path):
    w, t, opts = _stream(P, 6)
    ref = H.gpu_state(P, w)
    for b in w.batches:
        H.gpu_apply(P, ref, b, opts)
    for b in w.batches[:3]:
        H.gpu_apply(P, t, b, opts)
    p = tmp_path / "mid.tsvd"
    t.save(str(p))
    m, n = w.final_dims()
    u = P.TSVD.from_file(str(p), m_capacity=m, n_capacity=n)
    for b in w.batches[3:]:
        H.gpu_apply(P, u, b, opts)
    assert np.allclose(u.get_S(), ref.get_S(), rtol=1e-13, atol=0)
    assert np.allclose(u.get_U(), ref.get_U(), atol=1e-12) and np.allclose(u.get_V(), ref.get_V(), atol=1e-12)


@pytest.mark.parametrize("damage", ["payload", "truncate", "trailing", "version", "k"])
def test_load_rejects_and_leaves_context(P, tmp_path, damage):
    from paper_2401_09703_b200.tsvd import STATUS, TsvdError
    w, t, opts = _stream(P, 1)
    H.gpu_apply(P, t, w.batches[0], opts)
    p = tmp_path / "s.tsvd"
    t.save(str(p))
    raw = bytearray(p.read_bytes())
    want = "E_IO"
    if damage == "payload":
        raw[200] ^= 0x40
    elif damage == "truncate":
        raw = raw[:-8]
    elif damage == "trailing":
        raw += b"\0"
    elif damage == "version":  # version 2 with a valid header checksum
        import struct
        raw[8:12] = struct.pack("<I", 2)
        h = 1469598103934665603
        for x in bytes(raw[:48]):
            h = ((h ^ x) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        raw[48:56] = struct.pack("<Q", h)
        want = "E_STATE_VERSION"
    p.write_bytes(bytes(raw))
    other = H.gpu_state(P, w) if damage != "k" else P.TSVD(w.k + 1, m_capacity=2000, n_capacity=1000)
    if damage == "k":
        p.write_bytes(bytes(raw))
        want = "E_SHAPE"
    before = other.get_S().copy() if damage != "k" else None
    with pytest.raises(TsvdError) as ei:
        other.load(str(p))
    assert STATUS[ei.value.status] == want
    if before is not None:
        assert np.array_equal(other.get_S(), before)


def _run_cli(args):
    from paper_2401_09703_b200 import cli
    import contextlib
    import io
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(args)
    return rc, [json.loads(x) for x in buf.getvalue().splitlines() if x.strip()]


def test_cli_init_update_query(P, tmp_path):
    """a 200 x 200 fixture: init on the first 100 rows (the GPU randomized SVD), two row batches
    of 50 through the CLI; the state matches the library driven directly from the same initial
    state, and the oracle (dense Zha-Simon from the CLI's own initial factors)"""
    A = synth.random_sparse(200, 200, 0.05, seed=11)
    mtx = tmp_path / "A.mtx"
    scipy.io.mmwrite(str(mtx), A)
    st = str(tmp_path / "s.tsvd")
    rc, out = _run_cli(["init", "--matrix", str(mtx), "--k", "8", "--fraction", "0.5", "--state", st, "--verify"])
    assert rc == 0 and out[0]["m"] == 100 and out[0]["orth_err"] <= 1e-10, out
    t0 = P.TSVD.from_file(st)
    U, S, V = t0.get_U(), t0.get_S(), t0.get_V()
    for b in range(2):
        E = A[100 + 50 * b: 150 + 50 * b]
        bp = tmp_path / f"b{b}.mtx"
        scipy.io.mmwrite(str(bp), E, comment="tsvd-batch rows")
        rc, out = _run_cli(["update", "--state", st, "--E", str(bp), "--verify"])
        assert rc == 0 and out[0]["kind"] == "rows" and out[0]["orth_err"] <= 1e-10, out
        t0.update_rows(P.Sparse.from_scipy(E.tocsr()))
        U, S, V, th = zha_simon.add_rows(U, S, V, E)
    t1 = P.TSVD.from_file(st)
    assert t1.dims() == (200, 200, 8)
    assert np.array_equal(t1.get_S(), t0.get_S())
    ok, info = H.compare(t1.get_U(), t1.get_S(), t1.get_V(), U, S, V, th, 8)
    assert ok, info
    rc, out = _run_cli(["query", "--state", st, "--side", "u", "--index", "150"])
    assert rc == 0 and np.allclose(out[0]["row"], t1.get_U()[150], atol=1e-14, rtol=0)
    rc, out = _run_cli(["info", "--state", st])
    assert rc == 0 and (out[0]["k"], out[0]["m"], out[0]["n"]) == (8, 200, 200)


def test_cli_cols_and_weights(P, tmp_path):
    """column and weight batches through the CLI (MatrixMarket m x s new columns; D m x s, E n x s)
    against the library driven directly and the dense Zha-Simon oracle"""
    A = synth.random_sparse(160, 120, 0.08, seed=21)
    mtx = tmp_path / "A.mtx"
    scipy.io.mmwrite(str(mtx), A)
    st = str(tmp_path / "s.tsvd")
    rc, out = _run_cli(["init", "--matrix", str(mtx), "--k", "6", "--fraction", "1.0", "--state", st])
    assert rc == 0, out
    t0 = P.TSVD.from_file(st, n_capacity=200)
    U, S, V = t0.get_U(), t0.get_S(), t0.get_V()
    Ec = synth.random_sparse(160, 30, 0.1, seed=22)            # 30 new columns (m x s)
    p = tmp_path / "c.mtx"
    scipy.io.mmwrite(str(p), Ec, comment="tsvd-batch cols")
    rc, out = _run_cli(["update", "--state", st, "--E", str(p), "--verify"])
    assert rc == 0 and out[0]["kind"] == "cols" and out[0]["n"] == 150, out
    EcT = sp.csr_matrix(Ec.T)
    t0.update_cols(P.Sparse.from_scipy(EcT))
    U, S, V, th = zha_simon.add_columns(U, S, V, EcT)
    D = synth.random_sparse(160, 4, 0.2, seed=23)               # A + D E^T, s = 4
    E = synth.random_sparse(150, 4, 0.2, seed=24)
    pd, pe = tmp_path / "D.mtx", tmp_path / "E.mtx"
    scipy.io.mmwrite(str(pd), D)
    scipy.io.mmwrite(str(pe), E)
    rc, out = _run_cli(["update", "--state", st, "--kind", "weights", "--D", str(pd), "--E", str(pe), "--verify"])
    assert rc == 0 and out[0]["kind"] == "weights", out
    DT, ET = sp.csr_matrix(D.T), sp.csr_matrix(E.T)
    t0.update_weights(P.Sparse.from_scipy(DT), P.Sparse.from_scipy(ET))
    U, S, V, th = zha_simon.update_weights(U, S, V, DT, ET)
    t1 = P.TSVD.from_file(st)
    assert t1.dims() == (160, 150, 6)
    assert np.array_equal(t1.get_S(), t0.get_S())
    ok, info = H.compare(t1.get_U(), t1.get_S(), t1.get_V(), U, S, V, th, 6)
    assert ok, info

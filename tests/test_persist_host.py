"""F4 host side (-m "not gpu"): the state-file header that tsvd_state_info parses (written here
byte by byte from include/tsvd.h "State persistence", so the documented layout is what the
library reads), its error statuses, and the CLI's dataset loaders and usage errors."""
import os
import struct

import numpy as np
import pytest
import scipy.io
import scipy.sparse as sp


@pytest.fixture(scope="module")
def P():
    import paper_2401_09703_b200 as P
    return P


def _fnv1a(b: bytes) -> int:
    h = 1469598103934665603
    for x in b:
        h ^= x
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def _header(version=1, k=4, m=10, n=7, resets=3, payload=0, magic=b"TSVDSTAT", corrupt=False):
    h = bytearray(64)
    h[0:8] = magic
    h[8:48] = struct.pack("<IiqqqQ", version, k, m, n, resets, payload)
    hs = _fnv1a(bytes(h[:48])) ^ (1 if corrupt else 0)
    h[48:56] = struct.pack("<Q", hs)
    return bytes(h)


def test_state_info_reads_documented_header(P, tmp_path):
    p = tmp_path / "s.tsvd"
    p.write_bytes(_header(k=4, m=10, n=7))
    assert P.state_info(str(p)) == (4, 10, 7)


@pytest.mark.parametrize("case,status", [("magic", "E_IO"), ("hsum", "E_IO"), ("version", "E_STATE_VERSION"),
                                         ("dims", "E_IO"), ("short", "E_IO"), ("missing", "E_IO")])
def test_state_info_errors(P, tmp_path, case, status):
    from paper_2401_09703_b200.tsvd import TsvdError, STATUS
    p = tmp_path / "s.tsvd"
    if case == "magic":
        p.write_bytes(_header(magic=b"TSVDSTAX"))
    elif case == "hsum":
        p.write_bytes(_header(corrupt=True))
    elif case == "version":
        p.write_bytes(_header(version=2))
    elif case == "dims":
        p.write_bytes(_header(k=8, m=4))
    elif case == "short":
        p.write_bytes(_header()[:40])
    with pytest.raises(TsvdError) as ei:
        P.state_info(str(p))
    assert STATUS[ei.value.status] == status


def test_load_edges_symmetric(tmp_path):
    from paper_2401_09703_b200 import cli
    p = tmp_path / "g.tsv"
    p.write_text("# comment\n0\t1\n1\t2\n2\t0\n")
    A = cli.load_edges(str(p)).toarray()
    assert A.shape == (3, 3)
    assert np.array_equal(A, A.T) and np.array_equal(A, 1.0 - np.eye(3))


def test_load_edges_duplicates_keep_max_and_line_numbers(tmp_path):
    from paper_2401_09703_b200 import cli
    p = tmp_path / "g.tsv"
    p.write_text("0 1 2.0\n1 0 5.0\n0 1 3.0\n")
    A = cli.load_edges(str(p), undirected=False).toarray()
    assert A[0, 1] == 3.0 and A[1, 0] == 5.0
    q = tmp_path / "bad.tsv"
    q.write_text("0 1\nx y\n")
    with pytest.raises(ValueError, match=":2:"):
        cli.load_edges(str(q))


def test_load_ratings(tmp_path):
    from paper_2401_09703_b200 import cli
    p = tmp_path / "r.csv"
    p.write_text("userId,movieId,rating\n17,99,4.5\n")
    A = cli.load_ratings(str(p))
    assert A.shape == (1, 1) and A[0, 0] == 4.5
    p.write_text("5,7,1.0\n6,7,2.0\n5,8,3.0\n5,7,0.5\n")
    A = cli.load_ratings(str(p)).toarray()
    assert np.array_equal(A, [[1.0, 3.0], [2.0, 0.0]])


def test_batch_kind_line_and_mtx_roundtrip(tmp_path):
    from paper_2401_09703_b200 import cli
    A = sp.random(5, 9, density=0.3, random_state=1, format="csr")
    p = tmp_path / "b.mtx"
    scipy.io.mmwrite(str(p), A, comment="tsvd-batch rows")
    B, kind = cli.read_batch_mtx(str(p))
    assert kind == "rows" and (abs(B - A)).max() == 0


def test_cli_usage_errors_exit_2(tmp_path):
    from paper_2401_09703_b200 import cli
    with pytest.raises(SystemExit) as e:
        cli.main(["init", "--matrix", "a.mtx", "--edges", "b.tsv", "--k", "4", "--state", "s"])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["update", "--state", "s"])  # --E missing
    assert e.value.code == 2
    p = tmp_path / "b.mtx"
    scipy.io.mmwrite(str(p), sp.eye(3, format="csr"))
    assert cli.main(["update", "--state", str(tmp_path / "s"), "--E", str(p)]) == 2  # no kind
    assert cli.main(["update", "--state", str(tmp_path / "s"), "--E", str(p), "--kind", "rows",
                     "--D", str(p)]) == 2  # D without weights

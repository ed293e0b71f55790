"""Row-sharded path on one GPU (-m gpu).

Virtual mode holds all W shards of U' and V' in one context (partials summed on the
device), so the partitioned computation — the column split of E, per-shard CSC / gather /
scatter, the sums of W = E X', the RPI Gram and E^T B' over shards, appended rows dealt
block-cyclically, the assembly in get_U / query_row — is checked on a single B200 against
the oracle.  NCCL mode is exercised with a 1-rank communicator (the same code path, the
collective an identity): the multi-rank collective itself cannot run on one GPU."""
import numpy as np
import pytest

from oracle import metrics, variants, zha_simon
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


def _state(P, w, shard):
    m, n = w.final_dims()
    t = P.TSVD(w.k, m_capacity=m, n_capacity=n, shard=shard)
    t.init(torch.from_numpy(w.U0).cuda(), torch.from_numpy(w.S0).cuda(), torch.from_numpy(w.V0).cuda())
    return t


def _stream(P, w, shard, mode="exact", l=12, t_it=3):
    tg = _state(P, w, shard)
    U, S, V = w.U0.copy(), w.S0.copy(), w.V0.copy()
    for bi, b in enumerate(w.batches):
        if mode == "exact":
            U, S, V, th = zha_simon.apply_batch(U, S, V, b)
            opts = None
        else:
            s = b.s
            if b.kind == "weights":
                skD, skE = synth.gaussian_sketch(50 + bi, s, l), synth.gaussian_sketch(90 + bi, s, l)
                U, S, V, th = variants.update_weights(U, S, V, b.D, b.E, "rpi", skD, skE, l=l, t=t_it)
                sk = np.concatenate([skD.ravel(), skE.ravel()])
            else:
                sk = synth.gaussian_sketch(50 + bi, s, l)
                fn = variants.add_rows if b.kind == "rows" else variants.add_columns
                U, S, V, th = fn(U, S, V, b.E, "rpi", sk, l=l, t=t_it)
            opts = P.make_opts(mode=P.RPI, l=l, t=t_it, sketch=np.ascontiguousarray(sk))
        H.gpu_apply(P, tg, b, opts)
        Ug, Sg, Vg = H.gpu_factors(tg)
        ok, d = H.compare(Ug, Sg, Vg, U, S, V, th, w.k)
        assert ok, (bi, b.kind, d, tg.stats())
        assert metrics.orth_err(Ug) < 1e-9 and metrics.orth_err(Vg) < 1e-9
    return tg


def _small(kind, m=90, n=70, k=8, s=25):
    A = synth.random_sparse(m, n, 0.08, seed=m + s, values="normal")
    U0, S0, V0 = synth.init_truncated_svd(A, k)
    if kind == "rows":
        bs = [synth.Batch("rows", synth.random_sparse(s, n, 0.1, 5 + i, values="normal")) for i in range(3)]
    elif kind == "cols":
        bs = [synth.Batch("cols", synth.random_sparse(s, m, 0.1, 5 + i, values="normal")) for i in range(3)]
    else:
        bs = [synth.Batch("weights", synth.random_sparse(s, n, 0.1, 5 + i, values="normal"),
                          synth.random_sparse(s, m, 0.1, 6 + i, values="normal")) for i in range(2)]
    return synth.Workload("shard-small", k, U0, S0, V0, bs)


@pytest.mark.parametrize("mode", ["exact", "rpi"])
@pytest.mark.parametrize("kind", ["rows", "cols", "weights"])
def test_virtual_shards_vs_oracle(P, mode, kind):
    _stream(P, _small(kind), dict(world=3, virtual=True, block=7), mode=mode)


def test_virtual_shards_graph_stream(P):
    """configs[1] recipe (reduced), rows then columns, 4 shards of 64-row blocks: the sharded
    and unsharded GPU results agree and both match the oracle (MII resets included)."""
    w = synth.graph_nodeappend(N=4000, n_init=2000, batch=200, n_batches=3, k=16)
    ts = _stream(P, w, dict(world=4, virtual=True, block=64))
    t1 = H.gpu_state(P, w)
    for b in w.batches:
        H.gpu_apply(P, t1, b)
    assert np.allclose(ts.get_S(), t1.get_S(), rtol=1e-12)
    assert metrics.sin_theta(ts.get_U(), t1.get_U()) < 1e-10


def test_virtual_shards_query_materialize(P):
    w = _small("rows")
    t = _state(P, w, dict(world=3, virtual=True, block=5))
    for b in w.batches:
        H.gpu_apply(P, t, b)
    U, V = t.get_U(), t.get_V()
    for i in (0, 4, 5, 17, U.shape[0] - 1):
        assert np.allclose(t.query_row(0, i), U[i], atol=1e-14)
    assert np.allclose(t.query_row(1, 11), V[11], atol=1e-14)
    t.materialize()
    assert np.allclose(t.get_U(), U, atol=1e-13) and np.allclose(t.get_V(), V, atol=1e-13)


def test_sharded_gkl_is_unsupported(P):
    w = _small("rows")
    t = _state(P, w, dict(world=2, virtual=True, block=8))
    with pytest.raises(P.TsvdError) as ei:
        t.update_rows(P.Sparse.from_scipy(w.batches[0].E), P.make_opts(mode=P.GKL, l=5, seed=1))
    assert ei.value.status == 11


def test_nccl_one_rank_communicator(P):
    """NCCL mode end to end on one GPU: the library dlopens NCCL, builds the communicator from
    a ncclUniqueId and runs every reduction through ncclAllReduce (1 rank)."""
    import socket
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        for mode in ("exact", "rpi"):
            uid = P.nccl_unique_id()          # one ncclUniqueId per communicator
            assert len(uid) == 128
            _stream(P, _small("rows"), dict(world=1, rank=0, nccl_id=uid), mode=mode)
    finally:
        dist.destroy_process_group()


def test_virtual_shards_get_shard_and_local_query(P):
    """tsvd_get_U/V_shard return each shard's rows with their global ids (together: the whole
    factor, each row once); tsvd_query_row_local answers for rows this context holds."""
    w = _small("cols")
    W, B = 3, 5
    t = _state(P, w, dict(world=W, virtual=True, block=B))
    for b in w.batches:
        H.gpu_apply(P, t, b)
    for side, X in ((0, t.get_U()), (1, t.get_V())):
        seen = np.zeros(X.shape[0], int)
        for g in range(W):
            rows, ids = t.get_shard(side, g)
            assert rows.shape == (len(ids), w.k)
            assert all(P.shard_owner(int(i), W, B)[0] == g for i in ids)
            assert np.allclose(rows, X[ids], atol=1e-14)
            seen[ids] += 1
        assert (seen == 1).all()
        for i in (0, 3, X.shape[0] - 1):
            assert np.allclose(t.query_row_local(side, i), X[i], atol=1e-14)


def test_unsharded_get_shard_is_whole_factor(P):
    w = _small("rows")
    t = H.gpu_state(P, w)
    for b in w.batches:
        H.gpu_apply(P, t, b)
    rows, ids = t.get_shard(0, 0)
    assert (ids == np.arange(rows.shape[0])).all()
    assert np.allclose(rows, t.get_U(), atol=1e-14)


def test_virtual_shards_c4_reduced_matches_unsharded(P):
    """configs[3] recipe (reduced) with the library's K12 start blocks: 2 virtual row shards of
    U', V' agree with the unsharded context to rounding (the partial sums over the shards are
    added in a fixed order, so the two differ only in summation order)."""
    w = synth.weights_rpi(N=20_000, avg_deg=20, k=32, changes=4_000, n_batches=2)
    t1 = H.gpu_state(P, w)
    t2 = _state(P, w, dict(world=2, virtual=True, block=512))
    for bi, b in enumerate(w.batches):
        o = P.make_opts(mode=P.RPI, l=64, t=3, seed=1000 + bi)
        H.gpu_apply(P, t1, b, o)
        H.gpu_apply(P, t2, b, o)
    S1, S2 = t1.get_S(), t2.get_S()
    assert metrics.sigma_relerr(S2, S1) < 1e-12
    assert metrics.sin_theta(t2.get_U(), t1.get_U()) < 1e-10
    assert metrics.sin_theta(t2.get_V(), t1.get_V()) < 1e-10

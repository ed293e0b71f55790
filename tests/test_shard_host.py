"""Host logic of the row-sharded path (-m "not gpu"), multi-process over gloo (world_size
2, 127.0.0.1): the block-cyclic deal is a bijection, the library's host CSR split keeps
exactly the owned columns with local indices, and the sum over ranks of the partial lifts
W_g = E_g X'_g (and the RPI Gram partial B'_g^T B'_g) equals the unsharded product — the
reduction the library performs with ncclAllReduce."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import paper_2401_09703_b200 as P
    import synth
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        d, k, s, block = 1000, 8, 40, 16
        X = synth.random_orthonormal(d, k, seed=1)
        E = synth.random_sparse(s, d, 0.02, seed=2, values="normal")
        Es = P.Sparse.from_scipy(E)
        rp, ci, v = P.shard_split_host(Es, world, block, rank)
        # local rows of X owned by this rank, in local order
        own = [i for i in range(d) if P.shard_owner(i, world, block)[0] == rank]
        loc = [P.shard_owner(i, world, block)[1] for i in own]
        assert loc == list(range(len(own)))                # local index = rank among owned rows
        Xl = X[own]
        import scipy.sparse as sp
        Eg = sp.csr_matrix((v, ci, rp), shape=(s, len(own)))
        Wg = torch.from_numpy(np.asarray(Eg @ Xl))
        dist.all_reduce(Wg)
        ok_w = np.allclose(Wg.numpy(), E @ X, atol=1e-13)
        # RPI Gram partial: B'_g = E_g^T P on the local rows, sum_g B'_g^T B'_g = (E^T P)^T (E^T P)
        Pm = np.random.default_rng(3).standard_normal((s, 5))
        Bg = np.asarray(Eg.T @ Pm)
        Gg = torch.from_numpy(Bg.T @ Bg)
        dist.all_reduce(Gg)
        B = np.asarray(E.T @ Pm)
        ok_g = np.allclose(Gg.numpy(), B.T @ B, atol=1e-12)
        cnt = torch.tensor([len(own)], dtype=torch.int64)
        dist.all_reduce(cnt)
        q.put((rank, ok_w, ok_g, int(cnt.item()) == d, Eg.nnz))
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover
        q.put((rank, repr(ex)))


def test_two_rank_gloo_partition_and_reduce():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert len(r) == 5, r
        _, ok_w, ok_g, ok_cnt, _ = r
        assert ok_w and ok_g and ok_cnt, r
    import synth
    E = synth.random_sparse(40, 1000, 0.02, seed=2, values="normal")
    assert sum(r[4] for r in res) == E.nnz            # every nonzero goes to exactly one rank


def test_owner_bijection_single_process():
    import paper_2401_09703_b200 as P
    for world, block in [(1, 1024), (3, 5), (8, 64)]:
        seen = {}
        for i in range(1000):
            g, li = P.shard_owner(i, world, block)
            assert 0 <= g < world
            assert (g, li) not in seen
            seen[(g, li)] = i
        for g in range(world):
            locs = sorted(li for (gg, li) in seen if gg == g)
            assert locs == list(range(len(locs)))


@pytest.mark.parametrize("rows,world,block", [(1, 2, 4), (37, 3, 5), (1000, 8, 64), (4096, 4, 1024), (10, 8, 1)])
def test_allgather_layout_host(rows, world, block):
    """The NCCL-mode get_U layout (shard.cu unshuffle_kernel): every shard contributes a block
    of maxl rows (shard 0 owns the most rows of the block-cyclic deal), its local row j at
    offset j; global row i is read from block owner(i) at local(i) — a bijection onto the
    concatenated blocks' used rows, and local(i) < maxl for every i."""
    from paper_2401_09703_b200 import tsvd as T
    owners = [T.shard_owner(i, world, block) for i in range(rows)]
    counts = [sum(1 for g, _ in owners if g == r) for r in range(world)]
    maxl = counts[0]
    assert maxl == max(counts)
    slots = {(g, l) for g, l in owners}
    assert len(slots) == rows and all(l < maxl for _, l in slots)
    for r in range(world):
        assert sorted(l for g, l in owners if g == r) == list(range(counts[r]))

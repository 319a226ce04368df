"""Multi-GPU C^2 by hash function (N2, paper_2010_11497_b200/dist.py) on CPU ranks: world_size 2
and 3 over gloo, the CPU oracle standing in for the per-rank GPU steps (Steps 1-2 + Alg. 3 over
the rank's functions) and for the per-block merge.  The exchange/assembly logic under test is
the product's; the result must equal the single-process t-function oracle build bytewise
(Alg. 3 is the top-k of the union, A16, so sharding by function is exact)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(name):
    if name == "c1":
        C = synth.config("c1")
        offs, items = synth.generate("c1")
        return offs, items, C.k, C.t, C.b, C.N, C.hash_seed
    rng = np.random.default_rng(17)
    offs, items = synth.random_instance(rng, 301, 150, 2, 30)
    return offs, items, 9, 3, 16, 40, 5  # odd n (uneven user blocks), t = 3 (uneven function split)


def _oracle_local(offs, items, *, k, t, b, N, seed, f0, t_g, sim_mode):
    from paper_2010_11497_b200 import dist as c2d
    n = len(offs) - 1
    if t_g == 0:
        return c2d.pad_lists(n, k, "cpu")
    m = int(items.max()) + 1
    htab = oracle.hash_table(seed, f0 + t_g, b, m)[f0:f0 + t_g]  # functions f0.. of the stream (A2)
    cl = oracle.cluster(offs, items, htab, N)
    nbr, inter, uni, _ = oracle.merge(oracle.local_knn(offs, items, cl, k))
    return c2d.pack_lists(torch.from_numpy(nbr), torch.from_numpy(inter.astype(np.int32)),
                          torch.from_numpy(uni.astype(np.int32)))


def _oracle_merge(lists):
    G, nb, k, _ = lists.shape
    cand = np.ascontiguousarray(lists.numpy()).view(oracle.CAND).reshape(G, nb, k)
    nbr, inter, uni, sim = oracle.merge(cand)
    return (torch.from_numpy(nbr), torch.from_numpy(inter.astype(np.int32)), torch.from_numpy(uni.astype(np.int32)),
            torch.from_numpy(sim))


def _worker(rank, world, port, case, out):
    import torch.distributed as dist
    from paper_2010_11497_b200 import dist as c2d
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        offs, items, k, t, b, N, seed = _case(case)
        o = torch.from_numpy(offs) if rank == 0 else torch.zeros(1, dtype=torch.int32)
        i = torch.from_numpy(items) if rank == 0 else torch.zeros(1, dtype=torch.int32)
        o, i = c2d.broadcast_csr(o, i)
        nbr, inter, uni, _ = c2d.build_sharded(
            o, i, k=k, t=t, b=b, N=N, seed=seed,
            local_fn=lambda oo, ii, **kw: _oracle_local(oo.numpy(), ii.numpy(), **kw), merge_fn=_oracle_merge)
        out.put((rank, nbr.numpy(), inter.numpy(), uni.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "c1"), (2, "rand"), (3, "rand")])
def test_sharded_by_function_equals_single_build(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    offs, items, k, t, b, N, seed = _case(case)
    ref = oracle.build_graph(offs, items, k=k, t=t, b=b, N=N, seed=seed)
    for rank, nbr, inter, uni in res:
        assert np.array_equal(nbr, ref["nbr"]), rank
        assert np.array_equal(inter, ref["inter"].astype(np.int32)) and np.array_equal(uni, ref["uni"].astype(np.int32))


def test_function_and_user_splits_cover_everything():
    from paper_2010_11497_b200 import dist as c2d
    for t in (1, 3, 8, 13):
        for G in (1, 2, 3, 4, 8):
            fs = [c2d.function_range(t, G, g) for g in range(G)]
            assert fs[0][0] == 0 and fs[-1][1] == t and all(a[1] == b[0] for a, b in zip(fs, fs[1:]))
            us = [c2d.user_block(1001, G, j) for j in range(G)]
            assert us[0][0] == 0 and us[-1][1] == 1001 and all(a[1] == b[0] for a, b in zip(us, us[1:]))

"""bench.py's multi-process (N > 1) host logic on CPU: world_size 2 over gloo (no GPU).

The data path does not shard: every rank builds the graph of its own dataset (data seed +
1000 * rank), so the only cross-rank step is the reduction of the
timing and the work: job time = max over ranks, job pairs = sum over ranks."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import bench
import synth


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ms, pairs = bench.reduce_over_ranks(10.0 + 5.0 * rank, 100 * (rank + 1), "cpu")
        e2e, _ = bench.reduce_over_ranks(20.0 - rank, 0, "cpu")
        out.put((rank, ms, pairs, e2e))
    finally:
        dist.destroy_process_group()


def test_reduce_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ms, pairs, e2e in res:
        assert ms == 15.0          # max over ranks
        assert pairs == 300.0      # sum over ranks
        assert e2e == 20.0


def test_reduce_single_process_is_identity():
    assert bench.reduce_over_ranks(12.5, 7, "cpu") == (12.5, 7.0)


def test_ranks_get_independent_datasets():
    c0, c1 = bench.cfg_for_rank("c1", 0), bench.cfg_for_rank("c1", 1)
    assert c0.data_seed != c1.data_seed and c0.n == c1.n
    o0, i0 = synth.generate(c0, cache=False)
    o1, i1 = synth.generate(c1, cache=False)
    assert len(o0) == len(o1) and not (np.array_equal(o0, o1) and np.array_equal(i0, i1))

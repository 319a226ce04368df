"""bench.py's multi-process (N > 1) host logic on CPU: world_size 2 over gloo (no GPU).

Strong scaling by hash function (N2): every rank works on the same dataset with its own t/G
functions (the exchange itself is tested in tests/test_dist.py); the timing reduction is job
time = max over ranks, job pairs = sum over ranks (each rank counts its functions' pairs)."""
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


def test_gpus_flag_must_match_world_size(monkeypatch):
    import subprocess
    import sys
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(bench.__file__), "bench.py"), "--gpus", "2",
                        "--steps", "1"], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0 and "torchrun" in r.stderr

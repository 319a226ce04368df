"""Sharding by hash function (N2) on ONE GPU: the G per-shard builds (C2_OPT_FUNC_OFFSET) merged
with c2_merge must equal the single t-function c2_build bytewise (Alg. 3 = top-k of the union,
A16).  The multi-process exchange itself is covered on CPU ranks (tests/test_dist.py)."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2010_11497_b200 as c2  # noqa: E402
from paper_2010_11497_b200 import dist as c2d  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = c2.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("cfg,G", [("c2", 2), ("c3", 4), ("c4", 8), ("c4", 3)])
def test_shards_merge_to_single_build(ctx, cfg, G):
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    o, i = torch.from_numpy(offs).cuda(), torch.from_numpy(items).cuda()
    ref = [x.cpu().numpy() for x in c2.build(o, i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)[:3]]
    parts = []
    for g in range(G):
        f0, f1 = c2d.function_range(C.t, G, g)
        parts.append(c2d.gpu_local(o, i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, f0=f0, t_g=f1 - f0,
                                   sim_mode=0, ctx=ctx))
    nbr, inter, uni, _ = c2.merge(torch.stack(parts).contiguous(), ctx=ctx)
    assert np.array_equal(nbr.cpu().numpy(), ref[0])
    assert np.array_equal(inter.cpu().numpy(), ref[1]) and np.array_equal(uni.cpu().numpy(), ref[2])


def test_build_sharded_over_nccl_single_rank(ctx):
    """The real exchange path (NCCL all-to-all + all-gather of CUDA tensors, c2_merge of the
    received lists) in a one-rank NCCL group: equals the single-process build bytewise."""
    import os
    import socket
    import torch.distributed as dist
    if not dist.is_nccl_available():
        pytest.skip("no NCCL")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        C = synth.config("c3")
        offs, items = synth.generate("c3")
        o, i = torch.from_numpy(offs).cuda(), torch.from_numpy(items).cuda()
        ref = [x.cpu().numpy() for x in c2.build(o, i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)[:3]]
        o2, i2 = c2d.broadcast_csr(o, i)
        nbr, inter, uni, _ = c2d.build_sharded(o2, i2, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)
        torch.cuda.synchronize()
        assert np.array_equal(nbr.cpu().numpy(), ref[0])
        assert np.array_equal(inter.cpu().numpy(), ref[1].astype(np.int32))
        assert np.array_equal(uni.cpu().numpy(), ref[2].astype(np.int32))
    finally:
        dist.destroy_process_group()

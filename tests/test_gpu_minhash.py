"""C^2/MinHash variant on the GPU vs the CPU oracle (``-m gpu``).

Clustering with C2_OPT_CLUSTERING = C2_CLUSTER_MINHASH: one cluster per min-hash item, no
splitting (clusters > N chunked, A9).  Cluster arrays and the whole build (local brute force +
Alg. 3 merge on those clusters) are compared bytewise with the oracle.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2010_11497_b200 as c2  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def npy(t):
    return t.cpu().numpy()


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = c2.Context(0)
    c.set_option(c2.OPT_CLUSTERING, c2.CLUSTER_MINHASH)
    yield c
    c.close()


def check_clusters(ctx, offs, items, t, N, seed):
    g = c2.fastrandomhash(dev(offs), dev(items), t, 64, N, seed, ctx=ctx)
    o = oracle.cluster_minhash(offs, items, seed, t, N)
    assert np.asarray(g["n_clusters"]).tolist() == o["n_clusters"].tolist()
    for key in ("offsets", "members", "cluster_of"):
        assert np.array_equal(npy(g[key]), o[key]), key
    st = ctx.stats()
    assert st["pairs"] == o["stats"]["pairs"] and st["split_nodes"] == 0
    assert st["chunked_residuals"] == o["stats"]["chunked_residuals"]


def check_build(ctx, offs, items, t, N, k, seed, mode=0):
    nbr, inter, uni, sim = c2.build(dev(offs), dev(items), k=k, t=t, b=64, N=N, seed=seed, sim_mode=mode, ctx=ctx)
    o = oracle.build_graph(offs, items, k=k, t=t, b=64, N=N, seed=seed, sim_mode=mode, clustering="minhash")
    assert np.array_equal(npy(nbr), o["nbr"])
    assert np.array_equal(npy(inter), o["inter"]) and np.array_equal(npy(uni), o["uni"])
    assert np.array_equal(npy(sim).view(np.uint32), o["sim"].view(np.uint32))


@pytest.mark.parametrize("seed", range(12))
def test_minhash_random(ctx, seed):
    rng = np.random.default_rng(300 + seed)
    n, m = int(rng.integers(1, 500)), int(rng.integers(2, 400))
    offs, items = synth.random_instance(rng, n, m, 1, min(40, m), zipf=float(rng.uniform(0.5, 1.3)))
    t, N, k = int(rng.integers(1, 9)), int(rng.choice([2, 7, 60, 10**6])), int(rng.integers(1, 40))
    check_clusters(ctx, offs, items, t, N, seed)
    check_build(ctx, offs, items, t, N, k, seed, mode=seed % 2)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_minhash_configs_unbounded(ctx, cfg):
    """The paper's variant: t x m clusters, no splitting (N >= n)."""
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    check_clusters(ctx, offs, items, C.t, C.n, C.hash_seed)
    check_build(ctx, offs, items, C.t, C.n, C.k, C.hash_seed)


def test_minhash_c4_clusters_chunked(ctx):
    C = synth.config("c4")
    offs, items = synth.generate("c4")
    check_clusters(ctx, offs, items, C.t, C.N, C.hash_seed)

"""Alg. 2's hybrid local solver (N4): Hyrec for clusters with |C| >= 5k^2,
GPU (C2_OPT_LOCAL_SOLVER = C2_SOLVER_HYBRID) vs the oracle (solver=1), bytewise (``-m gpu``)."""
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
    c.set_option(c2.OPT_LOCAL_SOLVER, c2.SOLVER_HYBRID)
    yield c
    c.close()


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("mode", [0, 1])
def test_hyrec_local_knn(ctx, seed, mode):
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(350, 900))
    offs, items = synth.random_instance(rng, n, 300, 2, 40, zipf=0.9)
    t, b, k = int(rng.integers(1, 4)), int(rng.choice([1, 2, 4])), int(rng.integers(3, 9))
    m = int(items.max()) + 1
    cl = oracle.cluster(offs, items, oracle.hash_table(seed, t, b, m), 10**6)
    gcl = {key: dev(cl[key]) for key in ("offsets", "members", "cluster_of")}
    gcl["n_clusters"] = cl["n_clusters"].tolist()
    g = npy(c2.local_knn(dev(offs), dev(items), gcl, k, mode, seed, ctx=ctx)).view(oracle.CAND).reshape(t, n, k)
    gtab = oracle.gf_table(seed, m) if mode else None
    st = {}
    o = oracle.local_knn(offs, items, cl, k, mode, gtab, solver=1, seed=seed, stats=st)
    assert st["hyrec_iters"] > 0  # the Hyrec branch ran
    assert np.array_equal(g, o)


@pytest.mark.parametrize("seed", range(4))
def test_hyrec_build_fused(ctx, seed):
    rng = np.random.default_rng(950 + seed)
    offs, items = synth.random_instance(rng, 700, 250, 2, 30, zipf=1.0)
    t, b, k, N = 3, 2, 6, 10**6  # clusters of ~350 >= 5 k^2 = 180 -> Hyrec; smaller ones brute force
    nbr, inter, uni, sim = c2.build(dev(offs), dev(items), k=k, t=t, b=b, N=N, seed=seed, ctx=ctx)
    o = oracle.build_graph(offs, items, k=k, t=t, b=b, N=N, seed=seed, solver=1)
    assert o["hyrec_iters"] > 0
    assert np.array_equal(npy(nbr), o["nbr"])
    assert np.array_equal(npy(inter), o["inter"]) and np.array_equal(npy(uni), o["uni"])


def test_hyrec_minhash_c3(ctx):
    """The paper's setting for Hyrec: unsplit (MinHash) clusters, the large ones solved greedily."""
    C = synth.config("c3")
    offs, items = synth.generate("c3")
    ctx.set_option(c2.OPT_CLUSTERING, c2.CLUSTER_MINHASH)
    try:
        nbr, inter, uni, _ = c2.build(dev(offs), dev(items), k=10, t=4, b=64, N=C.n, seed=3, ctx=ctx)
    finally:
        ctx.set_option(c2.OPT_CLUSTERING, c2.CLUSTER_FRH)
    o = oracle.build_graph(offs, items, k=10, t=4, b=64, N=C.n, seed=3, clustering="minhash", solver=1)
    assert o["hyrec_iters"] > 0
    assert np.array_equal(npy(nbr), o["nbr"])
    assert np.array_equal(npy(inter), o["inter"]) and np.array_equal(npy(uni), o["uni"])

"""Full-size parity of the GPU path against the CPU oracle, ALL users, every BASELINE config
(``-m gpu``).

The expected values are SHA-256 digests of the oracle's own outputs, written by
``tools/make_golden.py`` (which calls only ``oracle/`` and ``synth/``) into
``tests/golden/oracle_digests.json``: Alg. 1 + recursive split -> Alg. 2 brute
force -> Alg. 3 merge.  A digest match is a bytewise match of the
whole array (1,000,000 x 30 entries at c5).  On a mismatch the test recomputes a sample of
users with the oracle so the failure names the first users that differ.

The paper's three-call boundary (c2_fastrandomhash -> c2_local_knn -> c2_merge) is checked
at c4 and c5 too, on the cluster arrays, the t per-function candidate lists and the merged
graph.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2010_11497_b200 as c2  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def golden(cfg, mode):
    with open(os.path.join(GOLD, "oracle_digests.json")) as f:
        return json.load(f)[f"{cfg}/{mode}"]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def npy(t):
    return t.cpu().numpy()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = c2.Context(0)
    yield c
    c.close()


def diagnose(offs, items, rec, nbr, inter, uni, clusters_np):
    """Oracle on the first differing-looking users (sampled) to name them in the failure."""
    n = len(offs) - 1
    users = np.random.default_rng(1).choice(n, min(n, 2000), replace=False).astype(np.int32)
    o = oracle.knn_union_users(offs, items, clusters_np, rec["k"], users, rec["sim_mode"],
                               oracle.gf_table(rec["seed"], int(items.max()) + 1) if rec["sim_mode"] else None)
    bad = [int(users[i]) for i in range(len(users))
           if not (np.array_equal(nbr[users[i]], o[0][i]) and np.array_equal(inter[users[i]], o[1][i])
                   and np.array_equal(uni[users[i]], o[2][i]))]
    return bad[:10]


def gpu_clusters_np(cl):
    return dict(offsets=npy(cl["offsets"]), members=npy(cl["members"]), cluster_of=npy(cl["cluster_of"]),
                n_clusters=np.asarray(cl["n_clusters"], np.int32))


@pytest.mark.parametrize("cfg,mode", [("c1", 0), ("c2", 0), ("c3", 0), ("c4", 0), ("c4", 1), ("c5", 0)])
def test_build_all_users_bytewise(ctx, cfg, mode):
    rec = golden(cfg, mode)
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    assert sha(offs, items) == rec["csr_sha256"], "generator output differs from the one the digests belong to"
    d_o, d_i = dev(offs), dev(items)
    nbr, inter, uni, sim = c2.build(d_o, d_i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, sim_mode=mode, ctx=ctx)
    g = [npy(x) for x in (nbr, inter, uni, sim)]
    assert ctx.stats()["pairs"] == rec["pairs"]
    ok = (sha(g[0]) == rec["nbr_sha256"] and sha(g[1]) == rec["inter_sha256"] and sha(g[2]) == rec["uni_sha256"])
    if not ok:
        cl = gpu_clusters_np(c2.fastrandomhash(d_o, d_i, C.t, C.b, C.N, C.hash_seed, ctx=ctx))
        pytest.fail(f"{cfg}/{mode}: GPU graph differs from the oracle's; differing sampled users "
                    f"{diagnose(offs, items, rec, g[0], g[1], g[2], cl)}")
    assert sha(g[3]) == rec["sim_sha256"]
    # properties at any size: no self neighbour, no duplicate ids
    nb = g[0]
    assert not (nb == np.arange(len(offs) - 1)[:, None]).any()
    s = np.sort(nb, axis=1)
    assert not ((s[:, 1:] == s[:, :-1]) & (s[:, 1:] >= 0)).any()


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_three_call_boundary_bytewise(ctx, cfg):
    """c2_fastrandomhash -> c2_local_knn -> c2_merge (the paper's Steps 1-3 as separate calls)
    against the oracle's cluster arrays, per-function candidate lists and merged graph."""
    rec = golden(cfg, 0)
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    d_o, d_i = dev(offs), dev(items)
    cl = c2.fastrandomhash(d_o, d_i, C.t, C.b, C.N, C.hash_seed, ctx=ctx)
    cnp = gpu_clusters_np(cl)
    assert sha(cnp["n_clusters"], cnp["offsets"], cnp["members"], cnp["cluster_of"]) == rec["clusters_sha256"]
    del cnp
    cand = c2.local_knn(d_o, d_i, cl, C.k, 0, C.hash_seed, ctx=ctx)
    assert sha(npy(cand)) == rec["cand_sha256"]
    nbr, inter, uni, sim = c2.merge(cand, ctx=ctx)
    del cand
    assert sha(npy(nbr)) == rec["nbr_sha256"]
    assert sha(npy(inter)) == rec["inter_sha256"] and sha(npy(uni)) == rec["uni_sha256"]
    assert sha(npy(sim)) == rec["sim_sha256"]


def test_a7_fold_hand_built(ctx):
    """The hand-worked A7 instance (tests/golden/a7_fold.json): lone users stay in
    the residual of the node being split; a lone grandchild folds into its own parent."""
    with open(os.path.join(GOLD, "a7_fold.json")) as f:
        g = json.load(f)
    rows = g["profiles"]
    offs = np.zeros(len(rows) + 1, np.int32)
    offs[1:] = np.cumsum([len(r) for r in rows])
    items = np.asarray([x for r in rows for x in r], np.int32)
    htab = dev(np.asarray([g["h"]], np.uint16))
    for depth in (8, 1):
        ctx.set_option(c2.OPT_SKETCH_DEPTH, depth)
        try:
            cl = c2.fastrandomhash_table(dev(offs), dev(items), 1, g["b"], g["N"], htab, ctx=ctx)
        finally:
            ctx.set_option(c2.OPT_SKETCH_DEPTH, 8)
        o, m = npy(cl["offsets"])[0], npy(cl["members"])[0]
        got = [m[o[c]:o[c + 1]].tolist() for c in range(cl["n_clusters"][0])]
        assert got == g["expected_clusters"], depth
        st = ctx.stats()
        assert st["split_nodes"] == g["expected_split_nodes"]
        assert st["folded_singletons"] == g["expected_folded_singletons"]


def test_local_knn_rejects_null_cluster_of(ctx):
    offs = dev(np.asarray([0, 2, 4], np.int32))
    items = dev(np.asarray([1, 3, 2, 5], np.int32))
    cl = c2.fastrandomhash(offs, items, 1, 4, 10, 0, ctx=ctx)
    cl["cluster_of"] = None
    with pytest.raises(c2.C2Error) as e:
        c2.local_knn(offs, items, cl, 3, ctx=ctx)
    assert e.value.code == c2.C2_EINVAL


def test_table_values_must_be_below_b(ctx):
    offs = dev(np.asarray([0, 2, 4], np.int32))
    items = dev(np.asarray([0, 1, 1, 2], np.int32))
    htab = dev(np.asarray([[0, 3, 1]], np.uint16))  # 3 >= b = 2
    with pytest.raises(c2.C2Error) as e:
        c2.fastrandomhash_table(offs, items, 1, 2, 10, htab, ctx=ctx)
    assert e.value.code == c2.C2_EINVAL


def test_item_ids_past_window_limit(ctx):
    """Item ids far above the shared-memory window range (here up to 2^31 - 2): Step 2
    compacts the ids it streams (an order-preserving renaming leaves every intersection
    unchanged); the hash still sees the original ids."""
    rng = np.random.default_rng(9)
    offs, items = synth.random_instance(rng, 600, 300, 2, 40, zipf=0.8)
    ids = np.sort(rng.choice(2**31 - 1, size=300, replace=False)).astype(np.int64)
    big = ids[items].astype(np.int32)
    for t, b, N, k in ((3, 8, 100, 12), (2, 1, 600, 20)):
        nbr, inter, uni, _ = c2.build(dev(offs), dev(big), k=k, t=t, b=b, N=N, seed=4, ctx=ctx)
        # the oracle's hash of every ORIGINAL id, tabulated by compact id (item_hash = A1's rule)
        a, c = oracle.hash_params(4, t)
        htab = np.asarray([[oracle.item_hash(int(a[f]), int(c[f]), int(x), b) for x in ids] for f in range(t)],
                          np.uint16)
        o = oracle.build_graph(offs, items, k=k, t=t, b=b, N=N, seed=4, htab=htab)
        assert np.array_equal(npy(nbr), o["nbr"])
        assert np.array_equal(npy(inter), o["inter"]) and np.array_equal(npy(uni), o["uni"])


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_repeated_builds_match_digests(ctx, cfg):
    """Determinism at full speed (no per-launch synchronisation): three back-to-back builds on one
    stream, each compared with the oracle's digests -- a race in the tile kernel's shared-memory
    reuse or the in-place running lists would show up as a run-to-run difference."""
    rec = golden(cfg, 0)
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    d_o, d_i = dev(offs), dev(items)
    outs = [c2.build(d_o, d_i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx) for _ in range(3)]
    for nbr, inter, uni, sim in outs:
        assert sha(npy(nbr)) == rec["nbr_sha256"]
        assert sha(npy(inter)) == rec["inter_sha256"] and sha(npy(uni)) == rec["uni_sha256"]


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_build_host_all_users_bytewise(ctx, cfg):
    """c2_build_host (host buffers, chunked upload overlapped with validation and sketch) equals the
    oracle on every user."""
    rec = golden(cfg, 0)
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    nbr, inter, uni, sim = c2.build_host(offs, items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)
    assert sha(nbr) == rec["nbr_sha256"] and sha(inter) == rec["inter_sha256"] and sha(uni) == rec["uni_sha256"]
    assert sha(sim) == rec["sim_sha256"]

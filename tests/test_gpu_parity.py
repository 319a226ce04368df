"""GPU (B200) vs CPU-oracle parity, through the C ABI (``-m gpu``).

All comparisons are bit-exact: every stage of the C^2 path is integer, and the only float
output (sim = inter/uni, IEEE round-to-nearest f32 division on both sides) is compared
bytewise too.  Inputs are the seeded synthetic configs c1-c5 (synth/) plus seeded random
tiny instances and edge cases.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2010_11497_b200 as c2  # noqa: E402


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.cuda()


def npy(t):
    return t.cpu().numpy()


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = c2.Context(0)
    c.set_option(c2.OPT_SYNC_CHECK, 1)
    yield c
    c.close()


def mval(items):
    return int(items.max()) + 1


def random_case(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 400))
    m = int(rng.integers(2, 300))
    offs, items = synth.random_instance(rng, n, m, 1, min(int(rng.integers(1, 60)), m), zipf=float(rng.uniform(0.5, 1.5)))
    t = int(rng.integers(1, 9))
    b = int(rng.choice([1, 2, 3, 7, 16, 64, 1000, 32768]))
    N = int(rng.integers(2, 80))
    k = int(rng.integers(1, 65))
    return offs, items, t, b, N, k, 7 + seed


def gpu_clusters(cl):
    return dict(offsets=npy(cl["offsets"]), members=npy(cl["members"]), cluster_of=npy(cl["cluster_of"]),
                n_clusters=np.asarray(cl["n_clusters"], np.int32))


def assert_clusters_equal(g, o):
    assert np.array_equal(g["n_clusters"], o["n_clusters"])
    assert np.array_equal(g["offsets"], o["offsets"])
    assert np.array_equal(g["members"], o["members"])
    assert np.array_equal(g["cluster_of"], o["cluster_of"])


def cand_np(cand):
    t, n, k, _ = cand.shape
    return npy(cand).view(oracle.CAND).reshape(t, n, k)


# ------------------------------------------------------------------ step 1
@pytest.mark.parametrize("seed", range(16))
def test_sketch_random(ctx, seed):
    offs, items, t, b, N, k, hs = random_case(seed)
    g = npy(c2.sketch(dev(offs), dev(items), t, b, hs, 8, ctx=ctx))
    o = oracle.sketch(offs, items, oracle.hash_table(hs, t, b, mval(items)), 8)
    assert np.array_equal(g, o)
    g3 = npy(c2.sketch(dev(offs), dev(items), t, b, hs, 3, ctx=ctx))
    assert np.array_equal(g3, o[:, :, :3])


@pytest.mark.parametrize("t,b,lo,hi", [(13, 4096, 1, 12), (17, 32768, 1, 40), (9, 1000, 100, 3000), (8, 2, 1, 50),
                                        (3, 64, 2000, 5000)])
def test_sketch_windows(ctx, t, b, lo, hi):
    """k_sketch_w edge cases: several function groups (t > 8), short lists at large b (the value
    window slides up several times), long lists (many item chunks per lane), tiny b."""
    rng = np.random.default_rng(t * 100 + b)
    n, m = 300, 20000
    offs, items = synth.random_instance(rng, n, m, lo, hi, zipf=0.8)
    o = oracle.sketch(offs, items, oracle.hash_table(77, t, b, mval(items)), 8)
    for D in (8, 5):
        g = npy(c2.sketch(dev(offs), dev(items), t, b, 77, D, ctx=ctx))
        assert np.array_equal(g, o[:, :, :D])


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4"])
def test_sketch_configs(ctx, cfg):
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    g = npy(c2.sketch(dev(offs), dev(items), C.t, C.b, C.hash_seed, 8, ctx=ctx))
    o = oracle.sketch(offs, items, oracle.hash_table(C.hash_seed, C.t, C.b, mval(items)), 8)
    assert np.array_equal(g, o)


def test_frh_paper_worked_example(ctx):
    import json, os
    gdir = os.path.join(os.path.dirname(__file__), "golden")
    g = json.load(open(os.path.join(gdir, "frh_worked_example.json")))
    htab = np.asarray([[x - 1 for x in g["h1_paper_1based"]], [x - 1 for x in g["h2_paper_1based"]]], np.uint16)
    offs = np.asarray([0, 3, 6], np.int32)
    items = np.asarray(g["profiles"]["u"] + g["profiles"]["v"], np.int32)
    cl = gpu_clusters(c2.fastrandomhash_table(dev(offs), dev(items), 2, 3, 10, dev(htab), ctx=ctx))
    # H1 separates u (cluster 2) and v (cluster 1); H2 co-locates them
    assert cl["n_clusters"].tolist() == [2, 1]
    assert cl["cluster_of"][0][0] != cl["cluster_of"][0][1]
    assert cl["cluster_of"][1][0] == cl["cluster_of"][1][1]


def test_frh_fig3(ctx):
    import json, os
    gdir = os.path.join(os.path.dirname(__file__), "golden")
    g = json.load(open(os.path.join(gdir, "fig3_split.json")))
    rows = []
    for count, its in g["groups"]:
        rows += [its] * count
    offs = np.zeros(len(rows) + 1, np.int32)
    offs[1:] = np.cumsum([len(r) for r in rows])
    items = np.asarray([x for r in rows for x in r], np.int32)
    htab = np.asarray([[x - 1 for x in g["h_paper_1based"]]], np.uint16)
    for depth in (8, 1):
        ctx.set_option(c2.OPT_SKETCH_DEPTH, depth)
        cl = gpu_clusters(c2.fastrandomhash_table(dev(offs), dev(items), 1, g["b"], g["N"], dev(htab), ctx=ctx))
        sizes = sorted(np.diff(cl["offsets"][0][: cl["n_clusters"][0] + 1]).tolist())
        assert sizes == sorted(g["expected_final_sizes_paper"])
    ctx.set_option(c2.OPT_SKETCH_DEPTH, 8)


@pytest.mark.parametrize("seed", range(24))
def test_fastrandomhash_random(ctx, seed):
    offs, items, t, b, N, k, hs = random_case(seed)
    g = gpu_clusters(c2.fastrandomhash(dev(offs), dev(items), t, b, N, hs, ctx=ctx))
    o = oracle.cluster(offs, items, oracle.hash_table(hs, t, b, mval(items)), N)
    assert_clusters_equal(g, o)
    st = ctx.stats()
    for key in ("pairs", "clusters", "max_cluster_size", "split_nodes", "max_depth", "folded_singletons",
                "chunked_residuals"):
        assert st[key] == o["stats"][{"clusters": "clusters"}.get(key, key)], key


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_sketch_depth_fallback(ctx, depth):
    # A29: results must not depend on the sketch depth (deeper levels recompute from the CSR)
    C = synth.config("c1")
    offs, items = synth.generate("c1")
    o = oracle.cluster(offs, items, oracle.hash_table(C.hash_seed, C.t, C.b, mval(items)), 60)
    assert o["stats"]["max_depth"] >= 2
    ctx.set_option(c2.OPT_SKETCH_DEPTH, depth)
    try:
        g = gpu_clusters(c2.fastrandomhash(dev(offs), dev(items), C.t, C.b, 60, C.hash_seed, ctx=ctx))
    finally:
        ctx.set_option(c2.OPT_SKETCH_DEPTH, 8)
    assert_clusters_equal(g, o)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4"])
def test_fastrandomhash_configs(ctx, cfg):
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    g = gpu_clusters(c2.fastrandomhash(dev(offs), dev(items), C.t, C.b, C.N, C.hash_seed, ctx=ctx))
    o = oracle.cluster(offs, items, oracle.hash_table(C.hash_seed, C.t, C.b, mval(items)), C.N)
    assert_clusters_equal(g, o)
    assert ctx.stats()["pairs"] == o["stats"]["pairs"]


def test_chunk_guard_b1(ctx):
    rng = np.random.default_rng(5)
    offs, items = synth.random_instance(rng, 3001, 50, 1, 10)
    g = gpu_clusters(c2.fastrandomhash(dev(offs), dev(items), 2, 1, 100, 3, ctx=ctx))
    assert g["n_clusters"].tolist() == [31, 31]
    o = oracle.cluster(offs, items, oracle.hash_table(3, 2, 1, mval(items)), 100)
    assert_clusters_equal(g, o)
    assert ctx.stats()["chunked_residuals"] == 2


# ------------------------------------------------------------------ step 2
@pytest.mark.parametrize("seed", range(24))
@pytest.mark.parametrize("mode", [0, 1])
def test_local_knn_random(ctx, seed, mode):
    offs, items, t, b, N, k, hs = random_case(seed)
    o_cl = oracle.cluster(offs, items, oracle.hash_table(hs, t, b, mval(items)), N)
    cl = {key: dev(o_cl[key]) for key in ("offsets", "members", "cluster_of")}
    cl["n_clusters"] = o_cl["n_clusters"].tolist()
    g = cand_np(c2.local_knn(dev(offs), dev(items), cl, k, mode, hs, ctx=ctx))
    gtab = oracle.gf_table(hs, mval(items)) if mode else None
    o = oracle.local_knn(offs, items, o_cl, k, mode, gtab)
    assert np.array_equal(g, o)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_local_knn_configs(ctx, cfg):
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    o_cl = oracle.cluster(offs, items, oracle.hash_table(C.hash_seed, C.t, C.b, mval(items)), C.N)
    cl = {key: dev(o_cl[key]) for key in ("offsets", "members", "cluster_of")}
    cl["n_clusters"] = o_cl["n_clusters"].tolist()
    g = cand_np(c2.local_knn(dev(offs), dev(items), cl, C.k, 0, C.hash_seed, ctx=ctx))
    o = oracle.local_knn(offs, items, o_cl, C.k)
    assert np.array_equal(g, o)


# ------------------------------------------------------------------ step 3
@pytest.mark.parametrize("seed", range(10))
def test_merge_random_lists(ctx, seed):
    rng = np.random.default_rng(seed)
    t, n, k = int(rng.integers(1, 20)), int(rng.integers(1, 500)), int(rng.integers(1, 65))
    cand = np.zeros((t, n, k), oracle.CAND)
    # per user a fixed (inter, uni) per candidate id, so repeated ids carry identical values
    for u in range(n):
        pool = rng.choice(2 * k + 5, size=min(2 * k + 5, 3 * k), replace=False)
        vals = {int(v): (int(rng.integers(0, 50)), int(rng.integers(50, 120))) for v in pool}
        for f in range(t):
            L = int(rng.integers(0, k + 1))
            ids = rng.choice(pool, size=min(L, len(pool)), replace=False)
            es = sorted(((vals[int(v)][0], vals[int(v)][1], int(v)) for v in ids),
                        key=lambda e: (-e[0] / e[1], e[2]))
            # exact order via cross products
            import functools
            es.sort(key=functools.cmp_to_key(lambda a, b: (b[0] * a[1] - a[0] * b[1]) or (a[2] - b[2])))
            for j, (i, U, v) in enumerate(es):
                cand[f, u, j] = (v, i, U)
            for j in range(len(es), k):
                cand[f, u, j] = (-1, 0, 0)
    gc = torch.from_numpy(cand.view(np.int32).reshape(t, n, k, 2).copy()).cuda()
    nbr, inter, uni, sim = c2.merge(gc, ctx=ctx)
    o = oracle.merge(cand)
    assert np.array_equal(npy(nbr), o[0]) and np.array_equal(npy(inter), o[1]) and np.array_equal(npy(uni), o[2])
    assert np.array_equal(npy(sim).view(np.uint32), o[3].view(np.uint32))


# ------------------------------------------------------------------ whole path
def check_build(ctx, offs, items, t, b, N, k, hs, mode=0):
    nbr, inter, uni, sim = c2.build(dev(offs), dev(items), k=k, t=t, b=b, N=N, seed=hs, sim_mode=mode, ctx=ctx)
    o = oracle.build_graph(offs, items, k=k, t=t, b=b, N=N, seed=hs, sim_mode=mode)
    assert np.array_equal(npy(nbr), o["nbr"])
    assert np.array_equal(npy(inter), o["inter"])
    assert np.array_equal(npy(uni), o["uni"])
    assert np.array_equal(npy(sim).view(np.uint32), o["sim"].view(np.uint32))
    return o


@pytest.mark.parametrize("seed", range(24))
def test_build_random(ctx, seed):
    offs, items, t, b, N, k, hs = random_case(seed)
    check_build(ctx, offs, items, t, b, N, k, hs, mode=seed % 2)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4"])
def test_build_configs(ctx, cfg):
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    check_build(ctx, offs, items, C.t, C.b, C.N, C.k, C.hash_seed)


@pytest.mark.parametrize("tensor", [0, 1])
def test_build_c4_goldfinger(ctx, tensor):
    """c4 in GoldFinger mode, big clusters on the bit-sliced list kernel or the tensor cores."""
    C = synth.config("c4")
    offs, items = synth.generate("c4")
    ctx.set_option(c2.OPT_GF_TENSOR, tensor)
    try:
        check_build(ctx, offs, items, C.t, C.b, C.N, C.k, C.hash_seed, mode=1)
    finally:
        ctx.set_option(c2.OPT_GF_TENSOR, 0)


def test_build_b1_exact_knn(ctx):
    # b = 1 and N >= n: the output equals exact KNN (BJ.north_star invariant)
    rng = np.random.default_rng(3)
    offs, items = synth.random_instance(rng, 700, 120, 1, 40)
    nbr, inter, uni, _ = c2.build(dev(offs), dev(items), k=17, t=3, b=1, N=700, seed=1, ctx=ctx)
    e = oracle.exact_knn(offs, items, 17)
    assert np.array_equal(npy(nbr), e[0]) and np.array_equal(npy(inter), e[1]) and np.array_equal(npy(uni), e[2])


@pytest.mark.parametrize("case", ["single_user", "two_users", "identical_profiles", "one_item_each", "k64",
                                  "t64", "long_rows", "b32768_N2", "big_cluster_ties"])
def test_build_edge_cases(ctx, case):
    rng = np.random.default_rng(hash(case) % 2**32)
    t, b, N, k = 3, 16, 50, 10
    if case == "single_user":
        offs, items = np.asarray([0, 3], np.int32), np.asarray([1, 5, 9], np.int32)
    elif case == "two_users":
        offs, items = np.asarray([0, 2, 3], np.int32), np.asarray([1, 5, 5], np.int32)
    elif case == "identical_profiles":
        n = 300
        offs = np.arange(0, 4 * n + 1, 4, dtype=np.int32)
        items = np.tile(np.asarray([2, 3, 7, 11], np.int32), n)
        N = 100
    elif case == "one_item_each":
        n = 500
        offs = np.arange(n + 1, dtype=np.int32)
        items = rng.integers(0, 20, n).astype(np.int32)
    elif case == "k64":
        offs, items = synth.random_instance(rng, 400, 60, 1, 20)
        k, N = 64, 200
    elif case == "t64":
        offs, items = synth.random_instance(rng, 200, 60, 1, 20)
        t = 64
    elif case == "long_rows":
        offs, items = synth.random_instance(rng, 150, 40000, 2000, 5000, zipf=0.6)
        b, N = 4, 60
    elif case == "b32768_N2":
        offs, items = synth.random_instance(rng, 300, 100, 1, 30)
        b, N = 32768, 2
    elif case == "big_cluster_ties":
        offs, items = synth.random_instance(rng, 2500, 30, 1, 4, zipf=0.3)
        b, N, k = 1, 2500, 30
    check_build(ctx, offs, items, t, b, N, k, 11)


def test_c5_sampled(ctx):
    """Full-size c5 in bench's launch configuration: clusters compared in full against the
    oracle; final neighbourhoods compared on 300 sampled users against the oracle's
    union-of-cluster-mates formulation (equal to Alg. 2 + Alg. 3)."""
    C = synth.config("c5")
    offs, items = synth.generate("c5")
    n = C.n
    d_offs, d_items = dev(offs), dev(items)
    g_cl = gpu_clusters(c2.fastrandomhash(d_offs, d_items, C.t, C.b, C.N, C.hash_seed, ctx=ctx))
    o_cl = oracle.cluster(offs, items, oracle.hash_table(C.hash_seed, C.t, C.b, mval(items)), C.N)
    assert_clusters_equal(g_cl, o_cl)
    nbr, inter, uni, sim = c2.build(d_offs, d_items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)
    users = np.random.default_rng(0).choice(n, 300, replace=False).astype(np.int32)
    o = oracle.knn_union_users(offs, items, o_cl, C.k, users)
    assert np.array_equal(npy(nbr)[users], o[0])
    assert np.array_equal(npy(inter)[users], o[1]) and np.array_equal(npy(uni)[users], o[2])
    # properties at any size: sorted best-first, no self, no duplicates
    nb = npy(nbr)
    assert not (nb == np.arange(n)[:, None]).any()
    s = np.sort(nb, axis=1)
    assert not ((s[:, 1:] == s[:, :-1]) & (s[:, 1:] >= 0)).any()


def test_build_host_matches_device(ctx):
    C = synth.config("c2")
    offs, items = synth.generate("c2")
    a = c2.build(dev(offs), dev(items), k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)
    h = c2.build_host(offs, items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)
    for x, y in zip(a, h):
        assert np.array_equal(npy(x), y)


def test_determinism(ctx):
    C = synth.config("c3")
    offs, items = synth.generate("c3")
    r1 = [npy(x) for x in c2.build(dev(offs), dev(items), k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)]
    r2 = [npy(x) for x in c2.build(dev(offs), dev(items), k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)]
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)


def test_errors(ctx):
    offs = dev(np.asarray([0, 2, 4], np.int32))
    bad = dev(np.asarray([3, 1, 2, 5], np.int32))  # row 0 unsorted
    with pytest.raises(c2.C2Error) as e:
        c2.build(offs, bad, k=3, t=2, b=4, N=10, seed=0, ctx=ctx)
    assert e.value.code == c2.C2_EDATA
    good = dev(np.asarray([1, 3, 2, 5], np.int32))
    for kw in (dict(k=0), dict(k=65), dict(t=0), dict(t=65), dict(b=0), dict(b=40000), dict(N=1)):
        args = dict(k=3, t=2, b=4, N=10, seed=0)
        args.update(kw)
        with pytest.raises(c2.C2Error) as e:
            c2.build(offs, good, ctx=ctx, **args)
        assert e.value.code == c2.C2_EINVAL
    empty_row = dev(np.asarray([0, 0, 2], np.int32))
    with pytest.raises(c2.C2Error) as e:
        c2.build(empty_row, dev(np.asarray([1, 2], np.int32)), k=3, t=2, b=4, N=10, seed=0, ctx=ctx)
    assert e.value.code == c2.C2_EDATA


# ------------------------------------------------------------------ Step 2 without relabeling
@pytest.fixture(scope="module")
def ctx_win():
    """A ctx whose Step 2 streams global item windows instead of cluster-local ids
    (C2_OPT_RELABEL = 0): the second operand layout must give the same bits."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = c2.Context(0)
    c.set_option(c2.OPT_SYNC_CHECK, 1)
    c.set_option(c2.OPT_RELABEL, 0)
    yield c
    c.close()


@pytest.mark.parametrize("seed", range(8))
def test_build_random_windows(ctx_win, seed):
    offs, items, t, b, N, k, hs = random_case(seed)
    check_build(ctx_win, offs, items, t, b, N, k, hs, mode=seed % 2)


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_build_configs_windows(ctx_win, cfg):
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    check_build(ctx_win, offs, items, C.t, C.b, C.N, C.k, C.hash_seed)


def test_ctx_reuse_across_sizes():
    """One context serving problems of different sizes in turn (workspaces grow between calls)
    must give the same bits as a fresh context."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = c2.Context(0)
    try:
        for cfg in ["c1", "c2", "c1", "c3", "c2"]:
            C = synth.config(cfg)
            offs, items = synth.generate(cfg)
            nbr, inter, uni, _ = c2.build(dev(offs), dev(items), k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=c)
            o = oracle.build_graph(offs, items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed)
            assert np.array_equal(npy(nbr), o["nbr"]), cfg
            assert np.array_equal(npy(inter), o["inter"]) and np.array_equal(npy(uni), o["uni"]), cfg
    finally:
        c.close()


@pytest.mark.parametrize("cfg", ["c1", "c3", "c4"])
def test_pair_evaluations_equal_2P(ctx, cfg):
    """Work accounting: the local kernel evaluates every ordered pair of
    cluster-mates exactly once per row, i.e. 2P with P = sum over clusters of s(s-1)/2 computed
    from the returned cluster arrays (C2_OPT_KSTATS counter 70)."""
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    ks = torch.zeros(80, dtype=torch.int64, device="cuda")
    ctx.set_option(c2.OPT_KSTATS, ks.data_ptr())
    try:
        c2.build(dev(offs), dev(items), k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)
        torch.cuda.synchronize()
    finally:
        ctx.set_option(c2.OPT_KSTATS, 0)
    o = oracle.cluster(offs, items, oracle.hash_table(C.hash_seed, C.t, C.b, mval(items)), C.N)
    P = 0
    for f in range(C.t):
        sz = np.diff(o["offsets"][f][: int(o["n_clusters"][f]) + 1]).astype(np.int64)
        P += int((sz * (sz - 1) // 2).sum())
    assert int(ks[70]) == 2 * P
    assert ctx.stats()["pairs"] == P


@pytest.mark.parametrize("qmax", [0, 1, 3, 4096])
@pytest.mark.parametrize("cfg", ["c2", "c3", "c4"])
def test_build_survivor_slots(ctx, cfg, qmax):
    """Light-row path (C2_OPT_SURVIVORS): rows with a full running list are screened in the local
    kernel's epilogue and merged by k_surv_merge.  0 = every row merged in-tile; 1 and 3 slots make
    most light rows overflow into the in-tile fallback; all give the oracle's graph bytewise."""
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    ctx.set_option(c2.OPT_SURVIVORS, qmax)
    try:
        check_build(ctx, offs, items, C.t, C.b, C.N, C.k, C.hash_seed)
    finally:
        ctx.set_option(c2.OPT_SURVIVORS, 2048)


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("qmax", [1, 2])
def test_build_random_survivor_slots(ctx, seed, qmax):
    offs, items, t, b, N, k, hs = random_case(100 + seed)
    ctx.set_option(c2.OPT_SURVIVORS, qmax)
    try:
        check_build(ctx, offs, items, max(t, 3), b, N, k, hs, mode=seed % 2)
    finally:
        ctx.set_option(c2.OPT_SURVIVORS, 2048)


@pytest.mark.parametrize("tensor", [1, 0])
@pytest.mark.parametrize("n,N,k,lo,hi", [(3000, 700, 30, 20, 300), (1500, 1500, 64, 5, 120), (600, 150, 7, 1, 40)])
def test_goldfinger_tensor_cores(ctx, tensor, n, N, k, lo, hi):
    """GoldFinger mode: big clusters' intersections as 0/1 fingerprint contractions on the tensor
    cores (k_gf_mma: 128 x 128 blocks, clusters spanning several row and member blocks) or the
    bit-sliced list kernel -- both bytewise equal to the oracle (c2_build and c2_local_knn)."""
    rng = np.random.default_rng(n + N + k)
    offs, items = synth.random_instance(rng, n, 5000, lo, hi, zipf=0.9)
    ctx.set_option(c2.OPT_GF_TENSOR, tensor)
    try:
        check_build(ctx, offs, items, 3, 2, N, k, 11, mode=1)
        o_cl = oracle.cluster(offs, items, oracle.hash_table(11, 3, 2, mval(items)), N)
        cl = {key: dev(o_cl[key]) for key in ("offsets", "members", "cluster_of")}
        cl["n_clusters"] = o_cl["n_clusters"].tolist()
        g = cand_np(c2.local_knn(dev(offs), dev(items), cl, k, 1, 11, ctx=ctx))
        o = oracle.local_knn(offs, items, o_cl, k, 1, oracle.gf_table(11, mval(items)))
        assert np.array_equal(g, o)
    finally:
        ctx.set_option(c2.OPT_GF_TENSOR, 0)


@pytest.mark.parametrize("k,n,N", [(50, 2600, 2600), (64, 3000, 1800), (33, 2300, 2300)])
def test_build_big_clusters_large_k(ctx, k, n, N):
    """Clusters past 2048 members (count matrix in global scratch) and k > 32 (two-register
    running lists, 128-entry queues, round 1 on 64-candidate tops) against the oracle."""
    rng = np.random.default_rng(k * 7 + n)
    offs, items = synth.random_instance(rng, n, 400, 3, 60, zipf=0.8)
    check_build(ctx, offs, items, 2, 1, N, k, 5)


# ------------------------------------------------------------------ N1: device-side split loop
@pytest.mark.parametrize("split_dev", [0, 1])
@pytest.mark.parametrize("case", ["random", "c1", "c3", "c4", "depth", "deep"])
def test_split_device_loop(ctx, split_dev, case):
    """The cooperative split kernel (C2_OPT_SPLIT_DEVICE=1) and the host-driven level loop (0)
    both reproduce the oracle's clusters and statistics."""
    ctx.set_option(c2.OPT_SPLIT_DEVICE, split_dev)
    try:
        if case == "random":
            runs = []
            for s in range(12):
                offs, items, t, b, N, _, hs = random_case(s)
                runs.append((offs, items, t, b, N, hs, 8))
        elif case == "deep":
            # splits far past the sketch depth (b small against long profiles, N tiny): the
            # device loop refills each active user's sketch row every D levels
            rng = np.random.default_rng(77)
            offs, items = synth.random_instance(rng, 700, 500, 30, 150, zipf=0.8)
            runs = [(offs, items, 2, b, 6, 11, d) for b in (16, 64) for d in (8, 3)]
        elif case == "depth":
            C = synth.config("c1")
            offs, items = synth.generate("c1")
            runs = [(offs, items, C.t, C.b, 60, C.hash_seed, d) for d in (1, 2, 8)]
        else:
            C = synth.config(case)
            offs, items = synth.generate(case)
            runs = [(offs, items, C.t, C.b, N, C.hash_seed, 8) for N in (C.N, max(C.N // 4, 2))]
        for offs, items, t, b, N, hs, depth in runs:
            ctx.set_option(c2.OPT_SKETCH_DEPTH, depth)
            g = gpu_clusters(c2.fastrandomhash(dev(offs), dev(items), t, b, N, hs, ctx=ctx))
            o = oracle.cluster(offs, items, oracle.hash_table(hs, t, b, mval(items)), N)
            assert_clusters_equal(g, o)
            st = ctx.stats()
            for key in ("pairs", "split_nodes", "max_depth", "folded_singletons", "chunked_residuals"):
                assert st[key] == o["stats"][key], key
    finally:
        ctx.set_option(c2.OPT_SPLIT_DEVICE, 1)
        ctx.set_option(c2.OPT_SKETCH_DEPTH, 8)


def test_split_device_loop_fewer_syncs():
    """N1: with the device-side loop Step 1 synchronises with the host a fixed number of times,
    independent of the split depth (c4 splits 3 levels deep)."""
    C = synth.config("c4")
    offs, items = synth.generate("c4")
    d_o, d_i = dev(offs), dev(items)
    syncs = {}
    for sd in (0, 1):
        c = c2.Context(0)
        c.set_option(c2.OPT_SPLIT_DEVICE, sd)
        c2.fastrandomhash(d_o, d_i, C.t, C.b, C.N, C.hash_seed, ctx=c)
        syncs[sd] = c.stats()["host_syncs"]
        assert c.stats()["max_depth"] >= 2
        c.close()
    assert syncs[1] < syncs[0]
    assert syncs[1] <= 3, syncs


# ------------------------------------------------------------------ c2_build_host: chunked upload
@pytest.mark.parametrize("n", [1, 2, 5, 9, 40])
@pytest.mark.parametrize("clustering", [0, 1])
def test_build_host_small_and_minhash(ctx, n, clustering):
    """The host entry point uploads the CSR in up to 8 user chunks, validating and sketching each
    as it arrives; fewer users than chunks, and the MinHash clustering (no sketch), still give the
    device entry point's result."""
    rng = np.random.default_rng(900 + n)
    offs, items = synth.random_instance(rng, n, 60, 1, 25)
    ctx.set_option(c2.OPT_CLUSTERING, clustering)
    try:
        a = c2.build(dev(offs), dev(items), k=7, t=3, b=16, N=4, seed=5, ctx=ctx)
        h = c2.build_host(offs, items, k=7, t=3, b=16, N=4, seed=5, ctx=ctx)
    finally:
        ctx.set_option(c2.OPT_CLUSTERING, 0)
    for x, y in zip(a, h):
        assert np.array_equal(npy(x), y)


@pytest.mark.parametrize("where", ["first", "middle", "last"])
def test_build_host_reports_bad_row(ctx, where):
    """A rule violation in any upload chunk is reported as C2_EDATA with that row's index, and the
    context stays usable (the next call's sketch is recomputed)."""
    C = synth.config("c1")
    offs, items = synth.generate("c1")
    n = len(offs) - 1
    row = {"first": 0, "middle": n // 2, "last": n - 1}[where]
    bad = items.copy()
    p0, p1 = offs[row], offs[row + 1]
    bad[p0:p1] = bad[p0:p1][::-1]  # unsorted row (profiles have >= 5 items)
    with pytest.raises(c2.C2Error) as ei:
        c2.build_host(offs, bad, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)
    assert f"row {row}" in str(ei.value)
    a = c2.build(dev(offs), dev(items), k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)
    o = oracle.build_graph(offs, items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed)
    assert np.array_equal(npy(a[0]), o["nbr"])

"""Pins of the CPU oracle against things other than itself (``-m "not gpu"``).

Each test names the paper passage / closed form / independent computation that
fixes the expected value.  See DESIGN.md "Oracle pins".
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def csr(rows):
    offs = np.zeros(len(rows) + 1, np.int32)
    offs[1:] = np.cumsum([len(r) for r in rows])
    items = np.asarray([x for r in rows for x in sorted(r)], np.int32)
    return offs, items


def partition_sets(cl, f):
    n = cl["members"].shape[1]
    off = cl["offsets"][f]
    return {frozenset(cl["members"][f][off[c]:off[c + 1]].tolist()) for c in range(cl["n_clusters"][f])}


# ----------------------------------------------------------------- hashing (A1/A2)
def test_splitmix64_reference_vectors():
    g = gold("splitmix64.json")
    for seed, outs in g["vectors"].items():
        exp = [int(x, 0) for x in outs]
        assert oracle.splitmix64(int(seed), len(exp)) == exp


def test_hash_params_draw_order():
    # A2: (a_0, c_0, a_1, c_1, ...) are consecutive draws of SplitMix64(seed)
    s = oracle.splitmix64(42, 8)
    a, c = oracle.hash_params(42, 4)
    assert a.tolist() == s[0::2] and c.tolist() == s[1::2]


def test_item_hash_special_cases():
    rng = np.random.default_rng(0)
    for _ in range(200):
        a, c, x = (int(v) for v in rng.integers(0, 2**63, 3))
        z = (a * x + c) % 2**64
        assert oracle.item_hash(a, c, x, 1) == 0                       # b = 1 -> single bucket
        assert oracle.item_hash(a, c, x, 4096) == z >> 52               # b = 2^12 -> top 12 bits
        assert oracle.item_hash(a, c, x, 2**15) == z >> 49
        b = int(rng.integers(2, 32769))
        assert 0 <= oracle.item_hash(a, c, x, b) < b


def test_hash_uniformity_chi_square():
    # S:193 style chi-square.  Consecutive ids 0..m-1 form an arithmetic progression under
    # multiply-add, so their buckets are *more* even than random (A1): one-sided test.
    m = 1_000_000
    h = oracle.hash_table(7, 1, 4096, m)[0]
    cnt = np.bincount(h, minlength=4096)
    e = m / 4096
    chi2 = ((cnt - e) ** 2 / e).sum()
    assert chi2 < 4095 + 4.5 * math.sqrt(2 * 4095)
    # Scattered ids (how the generator presents items, A1): two-sided test, df = 1023.
    rng = np.random.default_rng(5)
    a, c = oracle.hash_params(7, 1)
    ids = rng.choice(2**31, size=100_000, replace=False)
    hv = np.asarray([oracle.item_hash(int(a[0]), int(c[0]), int(x), 1024) for x in ids])
    cnt = np.bincount(hv, minlength=1024)
    e = len(ids) / 1024
    chi2 = ((cnt - e) ** 2 / e).sum()
    assert abs(chi2 - 1023) < 4.5 * math.sqrt(2 * 1023)


def test_theorem2_example_reading_d15():
    g = gold("theorem2_example.json")
    l, b, d = g["l_union"], g["b"], g["d_reading"]
    bound = (1 + d) * (l - 1) / (2 * b)
    prob = 1 - (math.exp(d) / (1 + d) ** (1 + d)) ** (l * (l - 1) / (2 * b))
    assert round(bound, 3) == g["printed_lower_margin"]
    assert round(3 * round(bound, 3), 3) == g["printed_upper_margin"]   # paper multiplies the rounded 0.078
    assert round(prob, 3) == g["printed_probability"]
    # and d = 0.5 as printed does NOT reproduce them (the garble, A23)
    assert round((1.5) * (l - 1) / (2 * b), 3) != g["printed_lower_margin"]


@pytest.mark.parametrize("J_target", [0.1, 0.3, 0.6])
def test_theorem1_monte_carlo(J_target):
    # Theorem 1: J - kappa/l <= P[H(u1)=H(u2)] <= J + 3 kappa/l + O(.)^2.
    # Empirical co-location frequency of the oracle's hash family over many functions,
    # scattered item ids (A1).  kappa/l is bounded via Theorem 2 with d = 1.5 (A23).
    rng = np.random.default_rng(int(J_target * 100))
    l, b, T = 256, 4096, 20000
    inter = int(round(J_target * l))
    m = 10_000_000
    ids = rng.choice(m, size=l, replace=False)
    common, rest = ids[:inter], ids[inter:]
    r1 = rest[: (l - inter) // 2]
    r2 = rest[(l - inter) // 2:]
    P1 = np.sort(np.concatenate([common, r1]))
    P2 = np.sort(np.concatenate([common, r2]))
    J = inter / l
    # compact ids to a table
    uniq = np.unique(np.concatenate([P1, P2]))
    offs, items = csr([np.searchsorted(uniq, P1).tolist(), np.searchsorted(uniq, P2).tolist()])
    a, c = oracle.hash_params(1000 + int(J_target * 10), T)
    htab = np.zeros((T, len(uniq)), np.uint16)
    for f in range(T):
        htab[f] = [oracle.item_hash(int(a[f]), int(c[f]), int(x), b) for x in uniq]
    H = oracle.frh(offs, items, htab)
    p_hat = float((H[:, 0] == H[:, 1]).mean())
    kl = 2.5 * (l - 1) / (2 * b)
    sd = math.sqrt(p_hat * (1 - p_hat) / T)
    assert J - kl - 4 * sd <= p_hat <= J + 3 * kl + 4 * sd


# ----------------------------------------------------------------- FRH
def test_frh_worked_example():
    g = gold("frh_worked_example.json")
    h1 = [x - 1 for x in g["h1_paper_1based"]]
    h2 = [x - 1 for x in g["h2_paper_1based"]]
    htab = np.asarray([h1, h2], np.uint16)
    offs, items = csr([g["profiles"]["u"], g["profiles"]["v"]])
    H = oracle.frh(offs, items, htab)
    e = g["expected_paper_1based"]
    assert H[0].tolist() == [e["H1(u)"] - 1, e["H1(v)"] - 1]
    assert H[1].tolist() == [e["H2(u)"] - 1, e["H2(v)"] - 1]
    cl = oracle.cluster(offs, items, htab, N=10)
    assert partition_sets(cl, 0) == {frozenset([0]), frozenset([1])}   # separated under H1
    assert partition_sets(cl, 1) == {frozenset([0, 1])}                # co-located under H2


def test_sketch_is_the_exclusion_chain():
    # S[d+1] = H\S[d](u) = min{h(i) : h(i) > S[d]} (P:463 applied repeatedly, A5)
    rng = np.random.default_rng(3)
    offs, items = synth.random_instance(rng, 60, 50, 1, 15)
    htab = oracle.hash_table(5, 3, 16, 50)
    sk = oracle.sketch(offs, items, htab, D=6)
    H = oracle.frh(offs, items, htab)
    for f in range(3):
        for u in range(60):
            hv = [int(htab[f][x]) for x in items[offs[u]:offs[u + 1]]]
            chain = [min(hv)]
            while True:
                above = [v for v in hv if v > chain[-1]]
                if not above:
                    break
                chain.append(min(above))
            chain = (chain + [oracle.ABSENT] * 6)[:6]
            assert sk[f, u].tolist() == chain
            assert sk[f, u, 0] == H[f, u]


# ----------------------------------------------------------------- splitting
def fig3_instance():
    g = gold("fig3_split.json")
    rows = []
    for count, its in g["groups"]:
        rows += [its] * count
    offs, items = csr(rows)
    htab = np.asarray([[x - 1 for x in g["h_paper_1based"]]], np.uint16)
    return g, offs, items, htab


def test_fig3_split_sizes():
    g, offs, items, htab = fig3_instance()
    H = oracle.frh(offs, items, htab)[0]
    assert sorted(np.bincount(H).tolist(), reverse=True) == sorted(g["expected_level0_sizes_paper"], reverse=True)
    for form in (0, 1):
        cl = oracle.cluster(offs, items, htab, N=g["N"], formulation=form)
        sizes = sorted(np.diff(cl["offsets"][0][: cl["n_clusters"][0] + 1]).tolist())
        assert sizes == sorted(g["expected_final_sizes_paper"])
        assert cl["n_clusters"][0] == 5


def test_split_threshold_is_strict():
    # A4 / S:275: a cluster of exactly N users is not split
    rows = [[0, 1 + (u % 3)] for u in range(40)]
    offs, items = csr(rows)
    htab = np.asarray([[0, 1, 2, 3]], np.uint16)
    cl = oracle.cluster(offs, items, htab, N=40)
    assert cl["n_clusters"][0] == 1
    cl = oracle.cluster(offs, items, htab, N=39)
    assert cl["n_clusters"][0] == 3


def test_exhausted_users_stay_and_chunk_guard():
    # S:203 / A6 / A8 / A9: every item hashes to the same bucket -> H\eta undefined for all,
    # the residual is the whole node; larger than N -> ceil(s/N) balanced id chunks.
    n, N = 23, 5
    rows = [[u % 4, 4 + u % 3] for u in range(n)]
    offs, items = csr(rows)
    htab = np.zeros((1, 7), np.uint16)
    cl = oracle.cluster(offs, items, htab, N=N)
    mc = math.ceil(n / N)
    assert cl["n_clusters"][0] == mc
    exp = [list(range((j * n) // mc, ((j + 1) * n) // mc)) for j in range(mc)]
    got = [cl["members"][0][cl["offsets"][0][c]:cl["offsets"][0][c + 1]].tolist() for c in range(mc)]
    assert got == exp
    assert cl["stats"]["chunked_residuals"] == 1


def test_b1_closed_form():
    # b = 1: h == 0, one root node; every user is exhausted at depth 1 -> residual = U;
    # N >= n: one cluster; N < n: ceil(n/N) balanced id-contiguous clusters.
    rng = np.random.default_rng(11)
    offs, items = synth.random_instance(rng, 97, 40, 1, 10)
    htab = oracle.hash_table(1, 2, 1, 40)
    assert (htab == 0).all()
    cl = oracle.cluster(offs, items, htab, N=200)
    assert cl["n_clusters"].tolist() == [1, 1]
    cl = oracle.cluster(offs, items, htab, N=10)
    assert cl["n_clusters"].tolist() == [10, 10]
    for f in range(2):
        assert np.diff(cl["offsets"][f][:11]).tolist() == [np.diff([(j * 97) // 10 for j in range(11)])[q] for q in range(10)]
        assert cl["members"][f].tolist() == list(range(97))


@pytest.mark.parametrize("seed", range(12))
def test_two_clustering_formulations_agree(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(20, 300))
    m = int(rng.integers(5, 200))
    offs, items = synth.random_instance(rng, n, m, 1, min(20, m), zipf=1.2)
    t = int(rng.integers(1, 4))
    b = int(rng.choice([1, 2, 3, 8, 64]))
    N = int(rng.integers(2, 60))
    htab = oracle.hash_table(seed, t, b, m)
    a = oracle.cluster(offs, items, htab, N, 0)
    c = oracle.cluster(offs, items, htab, N, 1)
    for key in ("offsets", "members", "cluster_of", "n_clusters"):
        assert (a[key] == c[key]).all()
    assert a["stats"] == c["stats"]


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_formulations_agree_on_configs(cfg):
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    htab = oracle.hash_table(C.hash_seed, C.t, C.b, int(items.max()) + 1)
    a = oracle.cluster(offs, items, htab, C.N, 0)
    c = oracle.cluster(offs, items, htab, C.N, 1)
    for key in ("offsets", "members", "cluster_of", "n_clusters"):
        assert (a[key] == c[key]).all()


def test_partition_invariants():
    C = synth.config("c3")
    offs, items = synth.generate("c3")
    n = len(offs) - 1
    htab = oracle.hash_table(C.hash_seed, C.t, C.b, int(items.max()) + 1)
    cl = oracle.cluster(offs, items, htab, C.N)
    P = 0
    for f in range(C.t):
        nc = cl["n_clusters"][f]
        off = cl["offsets"][f][: nc + 1]
        sizes = np.diff(off)
        assert off[0] == 0 and off[-1] == n and (sizes >= 1).all() and (sizes <= C.N).all()
        mem = cl["members"][f]
        assert np.array_equal(np.sort(mem), np.arange(n))                       # each user exactly once
        firsts = mem[off[:-1]]
        assert (np.diff(firsts) > 0).all()                                       # canonical order
        for c in range(nc):
            seg = mem[off[c]:off[c + 1]]
            assert (np.diff(seg) > 0).all() and (cl["cluster_of"][f][seg] == c).all()
        P += int((sizes * (sizes - 1) // 2).sum())
    assert P == cl["stats"]["pairs"]


# ----------------------------------------------------------------- Jaccard & KNN
def test_jaccard_examples():
    # {1,2,3} vs {3,4,5} -> 1/5; identical -> 1; disjoint -> 0
    offs, items = csr([[1, 2, 3], [3, 4, 5], [1, 2, 3], [6, 7]])
    inter, uni = oracle.pair_counts(offs, items, [0, 0, 0], [1, 2, 3])
    assert [Fraction(int(i), int(u)) for i, u in zip(inter, uni)] == [Fraction(1, 5), Fraction(1), Fraction(0)]


def brute_knn_python(rows, k, users=None):
    """Independent brute force: Python sets + exact Fractions, ties by lower id."""
    n = len(rows)
    S = [set(r) for r in rows]
    out = []
    for u in (range(n) if users is None else users):
        c = []
        for v in range(n):
            if v == u:
                continue
            i = len(S[u] & S[v])
            U = len(S[u] | S[v])
            c.append((-Fraction(i, U), v, i, U))
        c.sort()
        lst = [(v, i, U) for _, v, i, U in c[:k]]
        out.append(lst + [(-1, 0, 0)] * (k - len(lst)))
    return out


def rows_of(offs, items):
    return [items[offs[u]:offs[u + 1]].tolist() for u in range(len(offs) - 1)]


@pytest.mark.parametrize("seed", range(6))
def test_exact_knn_vs_python_brute_force(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 40))
    offs, items = synth.random_instance(rng, n, 25, 1, 8)
    k = int(rng.integers(1, 12))
    nbr, inter, uni = oracle.exact_knn(offs, items, k)
    exp = brute_knn_python(rows_of(offs, items), k)
    for u in range(n):
        assert list(zip(nbr[u].tolist(), inter[u].tolist(), uni[u].tolist())) == exp[u]


@pytest.mark.parametrize("seed", range(6))
def test_b1_unbounded_N_equals_exact_knn(seed):
    # BJ.north_star invariant: b = 1 and N unbounded -> output = exact KNN (every t)
    rng = np.random.default_rng(50 + seed)
    n = int(rng.integers(2, 80))
    offs, items = synth.random_instance(rng, n, 30, 1, 9)
    k = int(rng.integers(1, 15))
    t = int(rng.integers(1, 4))
    g = oracle.build_graph(offs, items, k=k, t=t, b=1, N=n + 5, seed=seed)
    nbr, inter, uni = oracle.exact_knn(offs, items, k)
    assert (g["nbr"] == nbr).all() and (g["inter"] == inter).all() and (g["uni"] == uni).all()
    exp = brute_knn_python(rows_of(offs, items), k)
    assert [list(zip(a.tolist(), b.tolist(), c.tolist())) for a, b, c in zip(nbr, inter, uni)] == exp


@pytest.mark.parametrize("seed", range(6))
def test_local_knn_is_brute_force_within_cluster(seed):
    rng = np.random.default_rng(200 + seed)
    n = int(rng.integers(5, 60))
    offs, items = synth.random_instance(rng, n, 30, 1, 10)
    k = int(rng.integers(1, 10))
    htab = oracle.hash_table(seed, 2, 4, 30)
    cl = oracle.cluster(offs, items, htab, N=12)
    cand = oracle.local_knn(offs, items, cl, k)
    rows = rows_of(offs, items)
    for f in range(2):
        for c in range(cl["n_clusters"][f]):
            mem = cl["members"][f][cl["offsets"][f][c]:cl["offsets"][f][c + 1]].tolist()
            sub = [rows[x] for x in mem]
            exp = brute_knn_python(sub, k)
            for a, u in enumerate(mem):
                e = [(mem[v] if v >= 0 else -1, i, U) for v, i, U in exp[a]]
                got = [(int(x["id"]), int(x["inter"]), int(x["uni"])) for x in cand[f, u]]
                assert got == e


@pytest.mark.parametrize("seed", range(8))
def test_merge_equals_union_of_cluster_mates(seed):
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(10, 150))
    m = int(rng.integers(10, 80))
    offs, items = synth.random_instance(rng, n, m, 1, 12)
    k = int(rng.integers(1, 12))
    t = int(rng.integers(1, 5))
    g = oracle.build_graph(offs, items, k=k, t=t, b=int(rng.choice([2, 4, 16])), N=int(rng.integers(2, 30)),
                           seed=seed)
    nbr, inter, uni = oracle.knn_union(offs, items, g["clusters"], k)
    assert (g["nbr"] == nbr).all() and (g["inter"] == inter).all() and (g["uni"] == uni).all()


def test_merge_order_invariance_and_single_partial():
    offs, items = synth.generate("c1")
    C = synth.config("c1")
    g = oracle.build_graph(offs, items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed)
    nbr2 = oracle.merge(g["cand"][::-1].copy())[0]                  # S:445 permutation invariance
    assert (nbr2 == g["nbr"]).all()
    n1, i1, u1, _ = oracle.merge(g["cand"][:1].copy())               # S:440 one partial -> identity
    c0 = g["cand"][0]
    assert (n1 == c0["id"]).all() and (i1 == c0["inter"]).all() and (u1 == c0["uni"]).all()


def test_identical_tables_equal_single_function():
    rng = np.random.default_rng(9)
    offs, items = synth.random_instance(rng, 120, 40, 1, 10)
    h = oracle.hash_table(3, 1, 8, 40)
    g1 = oracle.build_graph(offs, items, k=7, t=1, b=8, N=15, seed=0, htab=h)
    g3 = oracle.build_graph(offs, items, k=7, t=3, b=8, N=15, seed=0, htab=np.repeat(h, 3, axis=0))
    assert (g1["nbr"] == g3["nbr"]).all() and (g1["inter"] == g3["inter"]).all()


def test_monotone_in_t():
    # A2: a t-function run's functions are a prefix of a (t+1)-function run's -> V_t(u) is a
    # subset of V_{t+1}(u) -> the j-th neighbour never gets worse as t grows.
    offs, items = synth.generate("c1")
    prev = None
    for t in (1, 2, 3, 4):
        g = oracle.build_graph(offs, items, k=10, t=t, b=64, N=500, seed=42)
        cur = g["inter"].astype(np.int64), g["uni"].astype(np.int64)
        if prev is not None:
            # cur_j >= prev_j as fractions (pads are 0/0 -> compare via cross products, pad = 0)
            lhs = cur[0] * np.maximum(prev[1], 1)
            rhs = prev[0] * np.maximum(cur[1], 1)
            assert (lhs >= rhs).all()
        prev = cur


def test_gf_equals_exact_without_collisions():
    # with no GoldFinger collisions (injective bit map) popcount-Jaccard == exact Jaccard
    rng = np.random.default_rng(17)
    offs, items = synth.random_instance(rng, 60, 500, 1, 30)
    gtab = rng.permutation(1024)[:500].astype(np.uint16)
    a = oracle.exact_knn(offs, items, 9)
    b = oracle.exact_knn(offs, items, 9, sim_mode=1, gtab=gtab)
    for x, y in zip(a, b):
        assert (x == y).all()


def test_gf_collisions_are_popcounts():
    rng = np.random.default_rng(18)
    offs, items = synth.random_instance(rng, 30, 300, 1, 40)
    gtab = oracle.gf_table(42, 300)
    nbr, inter, uni = oracle.exact_knn(offs, items, 29, sim_mode=1, gtab=gtab)
    rows = rows_of(offs, items)
    bits = [set(int(gtab[x]) for x in r) for r in rows]
    for u in range(30):
        for v, i, U in zip(nbr[u], inter[u], uni[u]):
            assert i == len(bits[u] & bits[v]) and U == len(bits[u] | bits[v])


def test_oracle_thread_count_independent():
    offs, items = synth.generate("c1")
    C = synth.config("c1")
    a = oracle.build_graph(offs, items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, nthreads=1)
    b = oracle.build_graph(offs, items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, nthreads=7)
    assert (a["nbr"] == b["nbr"]).all() and (a["cand"] == b["cand"]).all()


def test_rejects_malformed_csr():
    for rows in ([[1, 1]], [[2, 1]], [[]], [[-1, 3]]):
        offs = np.zeros(len(rows) + 1, np.int32)
        offs[1:] = np.cumsum([len(r) for r in rows])
        items = np.asarray([x for r in rows for x in r], np.int32)
        with pytest.raises(ValueError):
            oracle.frh(offs, items, np.zeros((1, 8), np.uint16))


# ----------------------------------------------------------------- round-2 pins
def test_item_hash_bigint_non_power_of_two_b():
    # A1/A26: h(x) = floor(((a*x + c) mod 2^64) * b / 2^64) for ANY 1 <= b <= 32768, written
    # here with Python's exact big integers (a third, independent implementation).  A 32-bit
    # (Lemire-style) reduction or a modulo reduction fails this for non-power-of-two b.
    rng = np.random.default_rng(11)
    bs = [3, 5, 7, 10, 100, 1000, 1023, 1025, 3000, 4095, 4097, 10007, 32767]
    for _ in range(400):
        a, c = (int(v) for v in rng.integers(0, 2**63, 2))
        a = a * 2 + 1
        x = int(rng.integers(0, 2**31))
        for b in bs:
            z = (a * x + c) % 2**64
            assert oracle.item_hash(a, c, x, b) == (z * b) >> 64
    # and the table the oracle builds from its SplitMix64 parameters uses the same rule
    a, c = oracle.hash_params(42, 3)
    tab = oracle.hash_table(42, 3, 1000, 500)
    for f in range(3):
        for x in (0, 1, 2, 17, 499):
            z = (int(a[f]) * x + int(c[f])) % 2**64
            assert int(tab[f][x]) == (z * 1000) >> 64


def test_a7_fold_hand_built():
    g = gold("a7_fold.json")
    offs, items = csr(g["profiles"])
    htab = np.asarray([g["h"]], np.uint16)
    for form in (0, 1):  # recursive and prefix-trie formulations
        cl = oracle.cluster(offs, items, htab, g["N"], form)
        got = [cl["members"][0][cl["offsets"][0][c]:cl["offsets"][0][c + 1]].tolist()
               for c in range(cl["n_clusters"][0])]
        assert got == g["expected_clusters"], form
        assert cl["stats"]["split_nodes"] == g["expected_split_nodes"]
        assert cl["stats"]["folded_singletons"] == g["expected_folded_singletons"]


# ----------------------------------------------------------------- C^2/MinHash variant (N3)
def _minhash_py(rows, seed, t, N):
    """Independent big-int MinHash clustering: z = (a x + c) mod 2^64 with Python integers."""
    a, c = oracle.hash_params(seed, t)
    out = []
    for f in range(t):
        groups = {}
        for u, r in enumerate(rows):
            key = min(r, key=lambda x: (((int(a[f]) * x + int(c[f])) % 2**64), x))
            groups.setdefault(key, []).append(u)
        cl = []
        for g in groups.values():
            g = sorted(g)
            s = len(g)
            if s <= N:
                cl.append(g)
            else:
                mc = -(-s // N)
                cl += [g[(j * s) // mc:((j + 1) * s) // mc] for j in range(mc)]
        out.append(sorted(cl))
    return out


@pytest.mark.parametrize("seed", range(6))
def test_minhash_clusters_vs_bigint(seed):
    rng = np.random.default_rng(50 + seed)
    n, m = int(rng.integers(2, 300)), int(rng.integers(2, 200))
    offs, items = synth.random_instance(rng, n, m, 1, 15)
    rows = [items[offs[u]:offs[u + 1]].tolist() for u in range(n)]
    t, N = int(rng.integers(1, 6)), int(rng.choice([2, 5, 40, 10**6]))
    cl = oracle.cluster_minhash(offs, items, 9 + seed, t, N)
    exp = _minhash_py(rows, 9 + seed, t, N)
    for f in range(t):
        got = [cl["members"][f][cl["offsets"][f][c]:cl["offsets"][f][c + 1]].tolist()
               for c in range(cl["n_clusters"][f])]
        assert got == exp[f]


def test_minhash_invariants():
    # one cluster per min-hash ITEM: members share that item, so users with disjoint profiles are
    # never co-clustered; identical profiles always are
    rows = [[1, 2, 3], [4, 5], [1, 2, 3], [6], [6], [7, 8, 9, 10], [11]]
    offs, items = csr(rows)
    cl = oracle.cluster_minhash(offs, items, 3, 64, 10**6)
    for f in range(64):
        cof = cl["cluster_of"][f]
        assert cof[0] == cof[2] and cof[3] == cof[4]
        for u in range(len(rows)):
            for v in range(len(rows)):
                if not set(rows[u]) & set(rows[v]):
                    assert cof[u] != cof[v]
    assert cl["stats"]["split_nodes"] == 0


@pytest.mark.parametrize("J_target", [0.2, 0.5])
def test_minhash_collision_probability_is_jaccard(J_target):
    # Broder's property (S:212 acceptance): P[minhash(u) = minhash(v)] = J for a random
    # permutation; the multiply-add family on scattered ids must match within MC noise + 0.02.
    rng = np.random.default_rng(int(J_target * 10))
    l, T = 100, 4000
    inter = int(round(2 * J_target * l / (1 + J_target)))  # |A| = |B| = l -> J = i / (2l - i)
    ids = rng.choice(2**31 - 1, size=2 * l - inter, replace=False)
    A = np.sort(ids[:l])
    B = np.sort(np.concatenate([ids[:inter], ids[l:]]))
    J = inter / (2 * l - inter)
    offs, items = csr([A.tolist(), B.tolist()])
    cl = oracle.cluster_minhash(offs, items, 77, T, 10**6)
    p_hat = float((cl["cluster_of"][:, 0] == cl["cluster_of"][:, 1]).mean())
    sd = math.sqrt(J * (1 - J) / T)
    assert abs(p_hat - J) <= 4 * sd + 0.02, (p_hat, J)


# ----------------------------------------------------------------- Hyrec (Alg. 2 else-branch, N4)
def _mix64(z):
    z &= 2**64 - 1
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
    return z ^ (z >> 31)


def _hyrec_py(rows, C, f, k, seed):
    """Independent pure-Python Hyrec: random k-graph, then synchronous rounds of
    'compare u with its neighbours' neighbours, keep the k best' until < 0.001 k |C| entries
    change or 30 rounds."""
    SALT = 0x4879726563526E67
    s = len(C)
    sets = [set(rows[u]) for u in C]

    def key(a, b):  # exact order: J desc (cross products), then id asc
        i = len(sets[a] & sets[b])
        U = len(sets[a]) + len(sets[b]) - i
        return (Fraction(-i, U), C[b]), (C[b], i, U)

    N = []
    for a in range(s):
        kk = _mix64(_mix64(((seed ^ SALT) + f) & (2**64 - 1)) + C[a])
        nb, j = [], 0
        while len(nb) < k:
            b = (_mix64(kk + j + 1) * s) >> 64
            j += 1
            if b != a and b not in nb:
                nb.append(b)
        N.append(nb)
    it = 0
    while True:
        upd, Nn, L = 0, [], []
        for a in range(s):
            cand = set(N[a])
            for b in N[a]:
                cand |= set(N[b])
            cand.discard(a)
            best = sorted(cand, key=lambda b: key(a, b)[0])[:k]
            upd += sum(1 for b in best if b not in N[a])
            Nn.append(best)
            L.append([key(a, b)[1] for b in best])
        N = Nn
        it += 1
        if upd * 1000 < k * s or it >= 30:
            return L


@pytest.mark.parametrize("seed", range(3))
def test_hyrec_vs_python(seed):
    rng = np.random.default_rng(70 + seed)
    offs, items = synth.random_instance(rng, 60, 40, 2, 12)
    rows = [items[offs[u]:offs[u + 1]].tolist() for u in range(60)]
    k = 4
    cl = oracle.cluster(offs, items, oracle.hash_table(1, 1, 1, 40), 10**6)  # b = 1: one cluster of 60
    cand = oracle.local_knn(offs, items, cl, k, solver=2, seed=seed)
    C = cl["members"][0][:60].tolist()
    exp = _hyrec_py(rows, C, 0, k, seed)
    for a, u in enumerate(C):
        assert [tuple(int(x) for x in e) for e in cand[0, u]] == exp[a]


def test_hyrec_small_cluster_is_exact():
    # |C| = k + 1: the random initial graph already holds every other member, so Hyrec returns
    # the exact neighbourhoods (= brute force) after one round
    rng = np.random.default_rng(5)
    offs, items = synth.random_instance(rng, 9, 30, 2, 10)
    cl = oracle.cluster(offs, items, oracle.hash_table(1, 1, 1, 30), 10**6)
    a = oracle.local_knn(offs, items, cl, 8, solver=2, seed=1)
    b = oracle.local_knn(offs, items, cl, 8, solver=0)
    assert np.array_equal(a, b)


def test_hyrec_quality_on_planted_clusters():
    # SPEC greedy_knn example: planted clusters -> Hyrec quality (Eq. 2) >= 0.85 of brute force
    rng = np.random.default_rng(8)
    rows = []
    for g in range(10):
        base = rng.choice(np.arange(g * 40, g * 40 + 40), 25, replace=False)
        for _ in range(50):
            rows.append(sorted(set(rng.choice(base, 12, replace=False).tolist()) | set(rng.choice(400, 2).tolist())))
    offs, items = csr(rows)
    k = 10
    cl = oracle.cluster(offs, items, oracle.hash_table(1, 1, 1, 401), 10**6)
    st = {}
    h = oracle.local_knn(offs, items, cl, k, solver=1, seed=2, stats=st)  # 500 >= 5 k^2: Hyrec branch
    e = oracle.local_knn(offs, items, cl, k, solver=0)
    assert st["hyrec_iters"] >= 1

    def qsum(c):
        ok = c["id"] >= 0
        return float((c["inter"][ok] / c["uni"][ok]).sum())
    assert qsum(h) >= 0.85 * qsum(e)

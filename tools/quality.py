"""Quality check of the GPU C^2 graph against exact KNN (a reported check, not a target).

For each config: the GPU graph (c2_build, exact or GoldFinger similarity) is compared with the
oracle's exact KNN (exact Jaccard, ties by lower id) on all users (c1-c3) or a seeded user sample
(c4: 2000, c5: 200):
  recall_strict     |G^(u) ∩ G(u)| / k                                  (neighbour recall, A31)
  recall_tie_aware  #{v in G^(u) : J(u,v) >= J_k(u)} / k, J_k the k-th exact similarity
  quality_eq2       sum_u sum_{v in G^(u)} J(u,v) / sum_u sum_{v in G(u)} J(u,v)
Every J is exact Jaccard recomputed by the oracle (A30: GoldFinger graphs are judged by exact J).
Prints one JSON line per (config, mode).  Usage: python tools/quality.py [c1 c2 ...]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2010_11497_b200 as c2  # noqa: E402

SAMPLE = {"c4": 2000, "c5": 200}


def quality(name, mode):
    C = synth.config(name)
    offs, items = synth.generate(name)
    n = len(offs) - 1
    d_o, d_i = torch.from_numpy(offs).cuda(), torch.from_numpy(items).cuda()
    nbr, _, _, _ = c2.build(d_o, d_i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, sim_mode=mode)
    torch.cuda.synchronize()
    nbr = nbr.cpu().numpy()
    bad = (nbr >= n) | (nbr < -1)
    if bad.any():
        rows = np.nonzero(bad.any(1))[0]
        raise RuntimeError(f"{name}: {int(bad.sum())} neighbour ids out of range in {len(rows)} rows, e.g. row "
                           f"{rows[0]}: {nbr[rows[0]].tolist()}")
    users = np.arange(n, dtype=np.int32)
    if name in SAMPLE:
        users = np.sort(np.random.default_rng(7).choice(n, SAMPLE[name], replace=False)).astype(np.int32)
    t0 = time.time()
    e_nbr, e_int, e_uni = oracle.exact_knn(offs, items, C.k, users=users)
    t_exact = time.time() - t0
    g = nbr[users]
    # exact J of the approximate neighbours
    uu = np.repeat(users, C.k)
    vv = g.reshape(-1)
    ok = vv >= 0
    gi, gu = oracle.pair_counts(offs, items, uu[ok], vv[ok])
    gj = np.zeros(len(vv))
    gj[ok] = gi / gu
    gj = gj.reshape(len(users), C.k)
    ej = np.where(e_nbr >= 0, e_int / np.maximum(e_uni, 1), 0.0)
    strict = np.mean([len(set(a[a >= 0]) & set(b[b >= 0])) / C.k for a, b in zip(g, e_nbr)])
    jk = ej[:, -1:]  # the k-th exact similarity (lists sorted best first)
    tie = np.mean(((gj >= jk - 1e-12) & (g >= 0)).sum(1) / C.k)
    q = gj.sum() / max(ej.sum(), 1e-30)
    return {"config": name, "sim": "gf1024" if mode else "exact", "users": int(len(users)), "k": C.k,
            "recall_strict": round(float(strict), 4), "recall_tie_aware": round(float(tie), 4),
            "quality_eq2": round(float(q), 4), "oracle_exact_knn_s": round(t_exact, 1),
            "oracle_cores": os.cpu_count()}


if __name__ == "__main__":
    cfgs = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
    for name in cfgs:
        for mode in ([0, 1] if name == "c4" else [0]):
            print(json.dumps(quality(name, mode)), flush=True)

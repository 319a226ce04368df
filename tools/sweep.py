"""Sensitivity sweeps and variant ablations on synthetic data (the paper's
Sec. V-D / Fig. 6-8 sweeps over t, b, N and its Table IV / V ablations).

For every setting: the GPU c2_build time (CUDA events, median of 3 after a warm-up), the pair count
P, and the KNN quality of the graph (Eq. 2, exact Jaccard) and neighbour recall against
the oracle's exact KNN on a seeded user sample.  The paper's figures are [FIGURE] placeholders in
PAPER.md, so these are reported shapes on stand-in data, not comparisons with printed values.

usage: python tools/sweep.py [c4] > profiles/r02_sweeps.jsonl      (GPU box)
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

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
C = synth.config(name)
offs, items = synth.generate(C)
n = C.n
d_o, d_i = torch.from_numpy(offs).cuda(), torch.from_numpy(items).cuda()
users = np.sort(np.random.default_rng(7).choice(n, min(n, 1000), replace=False)).astype(np.int32)
t0 = time.time()
e_nbr, e_int, e_uni = oracle.exact_knn(offs, items, C.k, users=users)
ej = np.where(e_nbr >= 0, e_int / np.maximum(e_uni, 1), 0.0)
ctx = c2.Context(0, timing=True)


def measure(t=C.t, b=C.b, N=C.N, mode=0, clustering=0, solver=0):
    ctx.set_option(c2.OPT_CLUSTERING, clustering)
    ctx.set_option(c2.OPT_LOCAL_SOLVER, solver)
    kw = dict(k=C.k, t=t, b=b, N=N, seed=C.hash_seed, sim_mode=mode, ctx=ctx)
    c2.build(d_o, d_i, **kw)
    ms = []
    for _ in range(3):
        nbr, _, _, _ = c2.build(d_o, d_i, **kw)
        torch.cuda.synchronize()
        ms.append(ctx.stats()["ms_total"])
    st = ctx.stats()
    g = nbr.cpu().numpy()[users]
    uu, vv = np.repeat(users, C.k), g.reshape(-1)
    ok = vv >= 0
    gi, gu = oracle.pair_counts(offs, items, uu[ok], vv[ok])
    gj = np.zeros(len(vv))
    gj[ok] = gi / gu
    recall = np.mean([len(set(a[a >= 0]) & set(b[b >= 0])) / C.k for a, b in zip(g, e_nbr)])
    return {"config": name, "t": t, "b": b, "N": N, "sim": "gf1024" if mode else "exact",
            "clustering": "minhash" if clustering else "frh", "solver": "hybrid" if solver else "brute",
            "build_ms": float(np.median(ms)), "pairs": st["pairs"], "clusters": st["clusters"],
            "max_cluster": st["max_cluster_size"], "quality_eq2": round(float(gj.sum() / ej.sum()), 4),
            "recall": round(float(recall), 4), "sample_users": int(len(users))}


rows = []
for t in (1, 2, 4, 8, 12):
    rows.append(measure(t=t))
for b in (256, 1024, 4096):
    rows.append(measure(b=b))
for N in (500, 1000, 2000, 4000):
    rows.append(measure(N=N))
rows.append(measure(mode=1))                 # Table V shape: GoldFinger vs exact sets
rows.append(measure(clustering=1, N=C.N))    # Table IV shape: MinHash instead of FRH (chunked at N)
rows.append(measure(N=8000, solver=1))       # Alg. 2 hybrid: clusters >= 5k^2 = 4500 solved by Hyrec
for r in rows:
    print(json.dumps(r), flush=True)

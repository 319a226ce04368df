"""Write tests/golden/oracle_digests.json: SHA-256 digests of the CPU oracle's full C^2 output
(Alg. 1 + split -> Alg. 2 brute force -> Alg. 3 merge) on every
BASELINE.json config, so the GPU parity tests can compare ALL users of the large configs
(c4, c5) bytewise without re-running the oracle on the GPU box.

This script calls only ``oracle/`` and ``synth/`` (the seeded generator); no value in the
output comes from the CUDA path.  The CSR digest pins the generator output the expected
values belong to.

Usage: python tools/make_golden.py [c1 c2 ...]      (default: all configs, c4 also in GF mode)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_digests.json")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def one(cfg: str, mode: int) -> dict:
    C = synth.config(cfg)
    offs, items = synth.generate(cfg)
    t0 = time.time()
    o = oracle.build_graph(offs, items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, sim_mode=mode)
    dt = time.time() - t0
    cl = o["clusters"]
    rec = {
        "config": cfg, "sim_mode": mode, "n": int(C.n), "nnz": int(len(items)),
        "k": C.k, "t": C.t, "b": C.b, "N": C.N, "seed": C.hash_seed,
        "csr_sha256": digest(offs, items),
        "clusters_sha256": digest(cl["n_clusters"], cl["offsets"], cl["members"], cl["cluster_of"]),
        "nbr_sha256": digest(o["nbr"]),
        "inter_sha256": digest(o["inter"]),
        "uni_sha256": digest(o["uni"]),
        "sim_sha256": digest(o["sim"]),
        "cand_sha256": digest(o["cand"]),
        "pairs": int(cl["stats"]["pairs"]),
        "oracle_seconds": round(dt, 1),
        "oracle_threads": oracle.NTHREADS,
    }
    print(json.dumps(rec), flush=True)
    return rec


def main(argv):
    jobs = [(c, 0) for c in (argv or ["c1", "c2", "c3", "c4", "c5"])]
    if not argv or "c4" in argv:
        jobs.append(("c4", 1))
    db = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for cfg, mode in jobs:
        db[f"{cfg}/{mode}"] = one(cfg, mode)
        with open(OUT, "w") as f:
            json.dump(db, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])

"""Whole-pipeline CPU-oracle timings per config (hash + cluster, Alg. 2 brute force, Alg. 3 merge) on
this host's cores -- the oracle column of BASELINE.md section 2.3 (a reported baseline, not a target)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import synth

for name in sys.argv[1:] or ["c1", "c2", "c3", "c4"]:
    C = synth.config(name)
    offs, items = synth.generate(name)
    t0 = time.perf_counter()
    o = oracle.build_graph(offs, items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed)
    dt = time.perf_counter() - t0
    P = int(o["clusters"]["stats"]["pairs"])
    print(json.dumps({"config": name, "oracle_s": round(dt, 3), "pairs": P, "pairs_per_s": P / dt,
                      "cores": os.cpu_count()}), flush=True)

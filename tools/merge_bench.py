"""Stand-alone Step 3 (c2_merge, Alg. 3) on a real c5 candidate array: CUDA-event time and the
fraction of the measured HBM copy bandwidth (algorithmic bytes: t*n*k*8 read + n*k*12 written)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2010_11497_b200 as c2  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
C = synth.config(name)
offs, items = synth.generate(C)
o, i = torch.from_numpy(offs).cuda(), torch.from_numpy(items).cuda()
ctx = c2.Context(0)
cl = c2.fastrandomhash(o, i, C.t, C.b, C.N, C.hash_seed, ctx=ctx)
cand = c2.local_knn(o, i, cl, C.k, 0, C.hash_seed, ctx=ctx)
n = C.n
out = (torch.empty((n, C.k), dtype=torch.int32, device="cuda"), torch.empty((n, C.k), dtype=torch.uint16, device="cuda"),
       torch.empty((n, C.k), dtype=torch.uint16, device="cuda"), torch.empty((n, C.k), dtype=torch.float32, device="cuda"))
for _ in range(3):
    c2.merge(cand, ctx=ctx)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record()
for _ in range(reps):
    c2.merge(cand, ctx=ctx)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
byts = C.t * n * C.k * 8 + n * C.k * 12
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
print(json.dumps({"kernel": "k_merge", "config": name, "ms": ms, "algorithmic_bytes": byts,
                  "GBps": byts / ms / 1e6, "frac_of_measured_hbm": byts / ms / 1e6 / peaks["hbm_gbs"]}))

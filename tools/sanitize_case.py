"""Small invocations of every libc2 entry point for compute-sanitizer runs (one tool per gpurun call):
c2_build on c1 with t=2 (fused light-row path, survivor overflow with 1 slot, GoldFinger mode,
MinHash clustering, hybrid solver), c2_local_knn + c2_merge (three-call boundary), c2_sketch, and a
random instance with windows.  Exits 0 after checking the fused build against the three-call path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2010_11497_b200 as c2

C = synth.config("c1")
offs, items = synth.generate(C, cache=False)
d_o, d_i = torch.from_numpy(offs).cuda(), torch.from_numpy(items).cuda()
ctx = c2.Context(0)
ref = [x.cpu() for x in c2.build(d_o, d_i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)]
for opt, val in ((c2.OPT_SURVIVORS, 1), (c2.OPT_SURVIVORS, 0)):
    ctx.set_option(opt, val)
    g = [x.cpu() for x in c2.build(d_o, d_i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)]
    assert all(torch.equal(a, b) for a, b in zip(ref, g)), f"option {opt}={val} changed the graph"
ctx.set_option(c2.OPT_SURVIVORS, 256)
c2.build(d_o, d_i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, sim_mode=1, ctx=ctx)
ctx.set_option(c2.OPT_CLUSTERING, 1)
c2.build(d_o, d_i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)
ctx.set_option(c2.OPT_CLUSTERING, 0)
ctx.set_option(c2.OPT_LOCAL_SOLVER, 1)
c2.build(d_o, d_i, k=4, t=2, b=4, N=2000, seed=3, ctx=ctx)
ctx.set_option(c2.OPT_LOCAL_SOLVER, 0)
cl = c2.fastrandomhash(d_o, d_i, C.t, C.b, C.N, C.hash_seed, ctx=ctx)
cand = c2.local_knn(d_o, d_i, cl, C.k, 0, C.hash_seed, ctx=ctx)
nbr, inter, uni, sim = c2.merge(cand, C.k, ctx=ctx)
assert torch.equal(nbr.cpu(), ref[0]) and torch.equal(inter.cpu(), ref[1]), "three-call path differs from c2_build"
c2.sketch(d_o, d_i, 3, 1000, 7, 5, ctx=ctx)
rng = np.random.default_rng(5)
o2, i2 = synth.random_instance(rng, 300, 150000, 1, 80, zipf=0.9)  # item range past one window
c2.build(torch.from_numpy(o2).cuda(), torch.from_numpy(i2).cuda(), k=12, t=3, b=16, N=120, seed=9, ctx=ctx)
torch.cuda.synchronize()
ctx.close()
print("sanitize case ok")

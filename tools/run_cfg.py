"""Run c2_build on one config: warm-up + one build (profiling driver, not the bench)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2010_11497_b200 as c2

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
C = synth.config(name)
offs, items = synth.generate(name)
d_o, d_i = torch.from_numpy(offs).cuda(), torch.from_numpy(items).cuda()
ctx = c2.Context(0)
if os.environ.get("C2_GF_TENSOR"):  # GoldFinger big clusters on the tensor cores (k_gf_mma)
    ctx.set_option(c2.OPT_GF_TENSOR, int(os.environ["C2_GF_TENSOR"]))
for _ in range(reps):
    c2.build(d_o, d_i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, sim_mode=mode, ctx=ctx)
torch.cuda.synchronize()
print("ok", ctx.stats())

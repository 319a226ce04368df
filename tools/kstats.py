"""K7/K8 diagnostic counters per function (C2_OPT_KSTATS) on one config (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2010_11497_b200 as c2

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
C = synth.config(name)
offs, items = synth.generate(name)
d_o, d_i = torch.from_numpy(offs).cuda(), torch.from_numpy(items).cuda()
ctx = c2.Context(0)
ks = torch.zeros(80, dtype=torch.int64, device="cuda")
c2.build(d_o, d_i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)
ctx.set_option(c2.OPT_KSTATS, ks.data_ptr())
c2.build(d_o, d_i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, ctx=ctx)
torch.cuda.synchronize()
k = ks.tolist()
print(f"{name}: k_row_topk rows {k[0]} nq==0 {k[1]/max(k[0],1):.3f} mean nq {k[2]/max(k[0],1):.2f} "
      f"nq>32KS {k[3]/max(k[0],1):.4f} rescans {k[4]} round1 rows {k[6]} exact-fallback rows {k[8]}")
print("  first-scan m histogram (bins of 20): " + " ".join(str(x) for x in k[16:32]))
print(f"  light rows {k[71]} survivors {k[72]} (mean {k[72] / max(k[71], 1):.2f}) prefilter hits {k[74]} (per light row {k[74] / max(k[71], 1):.1f}) overflowed to k_row_topk {k[73]}")
tt = sum(k[32:36]) or 1
for i, nm in enumerate(["mixed", "33-256", "257-1024", ">1024"]):
    mt = max(k[36 + i], 1)
    print(f"  {nm:9s} tiles {k[36 + i]:7d} share {k[32 + i] / tt * 100:5.1f}%  mean cycles {k[32 + i] / mt:8.0f}: "
          f"phase A {k[40 + 3 * i] / mt:8.0f}  light epilogue {k[41 + 3 * i] / mt:7.0f}  count rows {k[42 + 3 * i] / mt:7.0f}")
print(f"  probe of >1024 tiles: busy cycles per warp-step {k[64] / max(k[65], 1):.0f}  steps {k[65]}")
for i, nm in enumerate(["mixed", "33-256", "257-1024", ">1024"]):
    if not k[52 + i]:  # (counted only by a -DC2_KSTATS_STEPS=1 build)
        continue
    nt = max(k[60 + i], 1)
    print(f"  probe balance {nm:9s} light tiles {k[60 + i]:7d}: steps of the busiest warp {k[52 + i] / nt:7.1f}  mean per warp {k[56 + i] / nt / 16:7.1f}")
if k[75]:  # (a -DC2_KSTATS_SURV build)
    print(f"  k_surv_merge: survivors better than the current k-th best {k[75]} ({k[75] / max(k[71], 1):.2f} per light row), "
          f"of those not yet in the list {k[76]} ({k[76] / max(k[71], 1):.2f} per light row)")

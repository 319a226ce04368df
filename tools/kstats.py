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
print(f"{name}: rows {k[0]} nq==0 {k[1]/k[0]:.3f} mean nq {k[2]/k[0]:.2f} nq>32KS {k[3]/k[0]:.4f} overflow {k[4]/k[0]:.5f} "
      f"tiles {k[5]} round1 rows {k[6]} mean s {k[7]/max(k[5],1):.1f} exact-fallback rows {k[8]}")
tot = sum(k[9:14])
print("  warp-cycles: " + " ".join(f"{n} {v / tot * 100:.1f}%" for n, v in
      zip(["phaseA", "round1", "scan", "k8-rest", "k8-wait"], k[9:14])))
print(f"  round1-after-overflow rows {k[14]}  kth_of_queue calls {k[15]}")
print("  first-scan m histogram (bins of 20): " + " ".join(str(x) for x in k[16:32]))
tt = sum(k[32:36]) or 1
print("  tile cycles by class (share, tiles, mean cycles): " + " ".join(
    f"{n}: {k[32 + i] / tt * 100:.1f}% {k[36 + i]} {k[32 + i] / max(k[36 + i], 1):.0f}" for i, n in enumerate(["mixed", "33-256", "257-1024", ">1024"])))
for i, nm in enumerate(["mixed", "33-256", "257-1024", ">1024"]):
    mt = max(k[36 + i], 1)
    b = 40 + 5 * i
    print(f"  {nm:9s} tile (warp 0, mean cycles): build-sum {k[b] / mt:.0f}  probe {k[b + 1] / mt:.0f}  "
          f"phaseA-rest {k[b + 2] / mt:.0f}  K8 {k[b + 3] / mt:.0f}  wait {k[b + 4] / mt:.0f}")
nb = max(k[62], 1)
print(f"  rows of >1024 tiles (warp 0 sample): select {k[60] / nb:.0f} cycles/row  final {k[61] / nb:.0f} cycles/row  rows {k[62]}")
print(f"  probe of >1024 tiles: busy cycles per warp-step {k[64] / max(k[65], 1):.0f}  steps {k[65]}")

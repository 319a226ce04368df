import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import synth, oracle, paper_2010_11497_b200 as c2
for name in ["c1", "c2"]:
    C = synth.config(name); offs, items = synth.generate(name); n = len(offs) - 1
    d_o, d_i = torch.from_numpy(offs).cuda(), torch.from_numpy(items).cuda()
    nbr, inter, uni, sim = c2.build(d_o, d_i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, sim_mode=0)
    torch.cuda.synchronize()
    g = nbr.cpu().numpy()
    o = oracle.build_graph(offs, items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed)
    print(name, "equal:", np.array_equal(g, o["nbr"]), "bad ids:", int(((g >= n) | (g < -1)).sum()), flush=True)
    e = oracle.exact_knn(offs, items, C.k)
    print(name, "exact ok", flush=True)

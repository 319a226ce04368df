"""Rough per-phase timings of c2_build on the configs (dev tool, not the bench)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2010_11497_b200 as c2

cfgs = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
ctx = c2.Context(0, timing=True)
# QT_OPTS="9=1024,11=0": ctx options (C2_OPT_* number = value) for A/B runs
for kv in filter(None, os.environ.get("QT_OPTS", "").split(",")):
    k, v = kv.split("=")
    ctx.set_option(int(k), int(v))
for spec in cfgs:
    # "c5" or "c5:m=16000:N=256" (overrides of the synthetic config, dev experiments)
    name, *kv = spec.split(":")
    over = {k: type(getattr(synth.config(name), k))(v) for k, v in (x.split("=") for x in kv)}
    C = synth.config(name, **over)
    offs, items = synth.generate(C)
    name = spec
    d_o, d_i = torch.from_numpy(offs).cuda(), torch.from_numpy(items).cuda()
    for mode in ([0, 1] if name == "c4" else [0]):
        for rep in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            c2.build(d_o, d_i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, sim_mode=mode, ctx=ctx)
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t0) * 1e3
        s = ctx.stats()
        print(f"{name} mode={mode} wall={wall:.2f}ms total={s['ms_total']:.2f} sketch={s['ms_sketch']:.3f} "
              f"cluster={s['ms_cluster']:.3f} local={s['ms_local']:.3f} merge={s['ms_merge']:.3f} "
              f"P={s['pairs']} pairs/s(local)={s['pairs']/max(s['ms_local'],1e-9)*1e3:.3e} launches={s['launches']} "
              f"syncs={s['host_syncs']} maxdepth={s['max_depth']} split={s['split_nodes']}", flush=True)

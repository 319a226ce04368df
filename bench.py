#!/usr/bin/env python3
"""Benchmark of the B200 Cluster-and-Conquer (C^2) hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--sim exact|gf]
    python bench.py --impl reference ...        # the CPU oracle on a bounded sample

One step = one whole c2_build (validate CSR, FastRandomHash clustering with recursive split,
local brute-force Jaccard top-k, Alg. 3 merge) on the config's synthetic input, resident in
HBM.  metric/unit are BASELINE.json's: Jaccard pair evaluations per second, where a step's
pair count is P = sum over clusters of s(s-1)/2 (reading A21), with the end-to-end
build time as ms_per_step.  Multi-GPU (torchrun, N2): ONE dataset, rank g runs hash functions
[g t/G, (g+1) t/G), one all-to-all of per-user lists by user block, Alg. 3 merge per block
(paper_2010_11497_b200/dist.py) -- strong scaling; value = pairs of the whole t-function job /
max-over-ranks time.  Prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "Jaccard pair evaluations/sec and end-to-end KNN-graph build time (1 B200)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def reduce_over_ranks(ms, pairs, device):
    """The job's step time is the MAX over ranks of the device-timed step; its work the SUM of the
    ranks' pairs (each rank's pairs are those of its own hash functions).  No-op on one process."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(ms), float(pairs)
    tmax = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    tsum = torch.tensor([float(pairs)], dtype=torch.float64, device=device)
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    return float(tmax[0]), float(tsum[0])


def load_json(path):
    try:
        with open(os.path.join(ROOT, path)) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def measured_int_peak():
    """ALU-pipe lane-ops per SM per clock measured on this pool's B200s (tools/microbench/int_peaks.cu,
    profiles/r02_microbench.jsonl): LOP3 / SHF issue on the ALU pipe at 64 lanes/SM/clk."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_microbench.jsonl")) as f:
            rows = [json.loads(x) for x in f if x.strip()]
        lop3 = [r for r in rows if r.get("op") == "LOP3"][0]
        return float(lop3["lane_ops_per_sm_per_clk"]), "measured (profiles/r02_microbench.jsonl, LOP3)"
    except (OSError, IndexError, KeyError, ValueError):
        return 64.0, "fallback (CUDA guide: 64 LOP3 lane-ops/SM/clk)"


def roofline(C, st, tile_ms_step, n_tile, clock, ms_step):
    """Roofline of the dominant kernel, k_local_tile (Step 2, K7+K8), bound by the ALU pipe
    (ncu: ALU is its busiest pipe).

    achieved = ALU-pipe lane-ops of one step's tile launches (sm__inst_executed_pipe_alu.sum x 32,
    summed over the launches of one c5 build in the committed ncu capture) / the live CUDA-event
    time of those launches; peak = the measured 64 ALU lane-ops/SM/clk x 148 SMs x the median SM
    clock sampled during the timed region.  The method's own work rates (pairs/s and the
    SURVEY 8(d) d.3 unit, |P_u|+|P_v| per pair) are reported beside it."""
    per_clk, src = measured_int_peak()
    mhz = clock.get("sm_mhz") or 1965.0
    peak = per_clk * 148 * mhz * 1e6 / 1e12
    ncu = load_json("profiles/r02_ncu_tile_pipes.json")
    achieved, note, traffic = None, "no committed ncu pipe capture for this config", None
    if ncu and ncu.get("config") == C.name:
        alu = float(ncu["alu_warp_inst_per_step"]) * 32
        achieved = alu / (tile_ms_step * 1e-3) / 1e12
        note = f"ALU-pipe warp instructions per step from {ncu['source']}"
        if ncu.get("dram_bytes_per_launch") is not None:
            traffic = ncu["dram_bytes_per_launch"]
    out = {"kernel": "k_local_tile (K7 local Jaccard: phase A + light-row epilogue)", "bound": "alu",
           "achieved": achieved, "peak": peak, "unit": "T lane-ops/s (ALU pipe)",
           "frac": (achieved / peak) if achieved else None, "traffic": traffic,
           "peak_source": f"{src} x 148 SMs x {mhz:.0f} MHz (median SM clock during the timed region)",
           "achieved_source": note, "kernel_ms_per_step": tile_ms_step, "launches_per_step": n_tile,
           "share_of_step": tile_ms_step / ms_step,
           "algorithmic": {"pairs_per_s": st["pairs"] / (tile_ms_step * 1e-3),
                           "work_steps_per_s": st["work_steps"] / (tile_ms_step * 1e-3),
                           "work_steps_note": "SURVEY 8(d) d.3 unit: |P_u|+|P_v| summed over the step's "
                                              "unordered local pairs"}}
    if ncu and ncu.get("config") == C.name and "traffic_note" in ncu:
        out["traffic_note"] = ncu["traffic_note"]
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2010_11497_b200 as c2

    ws, rank, local = dist_env()
    if args.gpus != ws:
        sys.exit(f"bench.py --gpus {args.gpus} needs {args.gpus} ranks (torchrun --nproc-per-node {args.gpus}); "
                 f"WORLD_SIZE={ws}")
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    C = synth.config(args.config)
    offs, items = synth.generate(C)  # the SAME dataset on every rank (strong scaling by hash function)
    n, nnz = len(offs) - 1, len(items)
    d_offs = torch.from_numpy(offs).to(dev)
    d_items = torch.from_numpy(items).to(dev)
    sim_mode = 1 if args.sim == "gf" else 0
    stream = torch.cuda.current_stream(dev)
    ctx = c2.Context(local, stream=stream, timing=True)
    if args.clustering == "minhash":
        ctx.set_option(c2.OPT_CLUSTERING, c2.CLUSTER_MINHASH)
    out = (torch.empty((n, C.k), dtype=torch.int32, device=dev), torch.empty((n, C.k), dtype=torch.uint16, device=dev),
           torch.empty((n, C.k), dtype=torch.uint16, device=dev), torch.empty((n, C.k), dtype=torch.float32, device=dev))
    if ws > 1:
        from paper_2010_11497_b200 import dist as c2d

    def step():
        if ws == 1:
            c2.build(d_offs, d_items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, sim_mode=sim_mode, out=out,
                     ctx=ctx)
        else:  # functions [g t/G, (g+1) t/G) here, one all-to-all, Alg. 3 merge of this rank's users
            c2d.build_sharded(d_offs, d_items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, sim_mode=sim_mode,
                              ctx=ctx, gather=False, local_fn=local_fn)

    snap = {}

    def local_fn(o, i, **kw):  # the rank's fused build; its stats kept before c2_merge resets them
        r = c2d.gpu_local(o, i, ctx=ctx, **kw)
        snap.update(ctx.stats())
        return r

    def stats():
        return dict(ctx.stats(), **snap) if ws > 1 else ctx.stats()

    cold_ms = None
    for wi in range(args.warmup):
        step()
        if wi == 0:
            cold_ms = stats()["ms_total"]  # first call: workspaces allocated, cold caches
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tile_ms, launches, build_ms = [], [], []
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
            st = stats()  # per step: the library synchronised its own events inside the call
            tile_ms.append(st["ms_tile"])
            build_ms.append(st["ms_total"])
            launches.append(st["launches"])
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1) / args.steps
    st = stats()
    ms_max, pairs_all = reduce_over_ranks(ms, st["pairs"], dev)
    value = pairs_all / (ms_max * 1e-3)

    # ---- e2e through the public API with host buffers: H2D of the CSR and D2H of the graph inside
    h_offs = torch.from_numpy(offs).pin_memory()
    h_items = torch.from_numpy(items).pin_memory()
    e2e_steps = max(1, min(args.steps, 5))
    if ws == 1:
        h_out = [torch.empty((n, C.k), dtype=d, pin_memory=True) for d in (torch.int32, torch.int16, torch.int16,
                                                                              torch.float32)]
        np_out = (h_out[0].numpy(), h_out[1].numpy().view(np.uint16), h_out[2].numpy().view(np.uint16),
                  h_out[3].numpy())

        def e2e_step():
            c2.build_host(h_offs.numpy(), h_items.numpy(), k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed,
                          sim_mode=sim_mode, out=np_out, ctx=ctx)
        d2h = n * C.k * (4 + 2 + 2 + 4)
    else:
        blk = c2d.user_block(n, ws, rank)
        h_blk = torch.empty(((blk[1] - blk[0]), C.k), dtype=torch.int32, pin_memory=True)

        def e2e_step():
            o = h_offs.to(dev, non_blocking=True)
            i = h_items.to(dev, non_blocking=True)
            (nb, _, _, _), _ = c2d.build_sharded(o, i, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed,
                                                 sim_mode=sim_mode, ctx=ctx, gather=False)
            h_blk.copy_(nb, non_blocking=True)
        d2h = (blk[1] - blk[0]) * C.k * (4 + 2 + 2 + 4)
    e2e_step()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms, _ = reduce_over_ranks(e0.elapsed_time(e1) / e2e_steps, 0, dev)
    h2d = (n + 1) * 4 + nnz * 4

    if rank == 0:
        clock = clk.summary()
        tile_step = float(np.median(tile_ms))
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "pairs/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max,
            "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak",
            "vs_baseline": None,
            "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": C.name, "n_users": n, "n_items": C.m, "nnz": nnz, "k": C.k, "t": C.t, "b": C.b,
                       "N": C.N, "hash_seed": C.hash_seed, "data_seed": C.data_seed, "sim": args.sim,
                       "clustering": args.clustering, "pairs_per_step": pairs_all,
                       "l2": f"inputs larger than L2 (CSR {4 * (n + 1 + nnz) / 2**20:.0f} MiB + per-step scratch)",
                       "parallelism": ("one dataset; t/G hash functions per rank, one all-to-all of per-user "
                                       f"lists by user block, Alg. 3 merge per block (G={ws})") if ws > 1 else "1 GPU"},
            "roofline": roofline(C, st, tile_step, max(st["tile_launches"], 1), clock, ms),
            "e2e": {"value": pairs_all / (e2e_ms * 1e-3), "unit": "pairs/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": int(np.median(launches)),
            "clocks": clock,
            "phases_ms": {k: st[k] for k in ("ms_sketch", "ms_cluster", "ms_local", "ms_merge", "ms_total")},
            # BJ's second metric, end-to-end build time (library CUDA events, validate -> graph)
            "build_ms": {"median": float(np.median(build_ms)), "min": float(np.min(build_ms)),
                         "cold_first_call": cold_ms},
            "stats": {k: st[k] for k in ("clusters", "max_cluster_size", "split_nodes", "max_depth", "host_syncs",
                                         "work_steps")},
        }
        if not args.no_cpu_baseline and ws == 1:
            line["cpu_baseline"] = cpu_baseline(C, offs, items, args.cpu_seconds)
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()


def oracle_subsample(C, users):
    """The first `users` users of the config's CSR (same generator rows): a c5-shaped sample the
    whole oracle pipeline finishes in seconds."""
    offs, items = synth.generate(C)
    o = offs[: users + 1].copy()
    return o, items[: o[-1]].copy()


def oracle_pipeline(C, offs, items, cores):
    """The whole C^2 pipeline of the CPU oracle, as it stands: FRH clustering with recursive split
    (Alg. 1), brute force per cluster (Alg. 2), Alg. 3 merge; returns (pairs, seconds)."""
    import oracle
    t0 = time.perf_counter()
    o = oracle.build_graph(offs, items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, nthreads=cores)
    return o["clusters"]["stats"]["pairs"], time.perf_counter() - t0


SAMPLE_USERS = {"c5": 150_000}


def cpu_baseline(C, offs, items, seconds):
    cores = os.cpu_count() or 1
    users = SAMPLE_USERS.get(C.name, C.n)
    so, si = oracle_subsample(C, users) if users < C.n else (offs, items)
    P, dt = oracle_pipeline(C, so, si, cores)
    return {"value": P / dt, "unit": "pairs/s", "cores": cores, "kind": "oracle",
            "sample": f"whole oracle pipeline (clustering + Alg. 2 brute force + Alg. 3 merge, t={C.t}) on the "
                      f"first {users} users of {C.name}: {P} pairs in {dt:.1f} s"}


def run_reference(args):
    """The reference arm: the CPU oracle as it stands (no reference implementation exists; the
    reference is a paper), whole pipeline, all host cores, per step a bounded c5-shaped sample."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    C = synth.config(args.config)
    cores = os.cpu_count() or 1
    users = SAMPLE_USERS.get(C.name, C.n)
    so, si = oracle_subsample(C, users) if users < C.n else synth.generate(C)
    for _ in range(args.warmup):
        oracle_pipeline(C, so, si, cores)
    tot_p, tot_t = 0, 0.0
    for _ in range(args.steps):
        P, dt = oracle_pipeline(C, so, si, cores)
        tot_p, tot_t = tot_p + P, tot_t + dt
    v = tot_p / tot_t
    sample = (f"whole oracle pipeline (clustering + Alg. 2 + Alg. 3, t={C.t}) on the first {users} users of "
              f"{C.name} per step ({tot_p // max(args.steps, 1)} pairs)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "pairs/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_t / max(args.steps, 1) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": C.name, "n_users": C.n, "k": C.k, "t": C.t, "b": C.b, "N": C.N, "sim": args.sim,
                   "sample_users": users},
        "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)  # >= 3 (timing rules)
    ap.add_argument("--config", default="c5", choices=sorted(synth.CONFIGS))
    ap.add_argument("--sim", default="exact", choices=["exact", "gf"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--clustering", default="frh", choices=["frh", "minhash"])
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

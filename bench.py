#!/usr/bin/env python3
"""Benchmark of the B200 Cluster-and-Conquer (C^2) hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--sim exact|gf]
    python bench.py --impl reference ...        # the CPU oracle on a bounded sample

One step = one whole c2_build (validate CSR, FastRandomHash clustering with recursive split,
local brute-force Jaccard top-k, Alg. 3 merge) on the config's synthetic input, resident in
HBM.  metric/unit are BASELINE.json's: Jaccard pair evaluations per second, where a step's
pair count is P = sum over clusters of s(s-1)/2 (reading A21), with the end-to-end
build time as ms_per_step.  Multi-GPU (torchrun): every rank builds the graph of its own
dataset (data seed + rank) -- independent problems, no collective on the data path, weak
scaling; value = total pairs of all ranks / max-over-ranks time.  Prints ONE JSON line.
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


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


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
    """Weak scaling over independent datasets: the job's step time is the MAX over ranks of the
    device-timed step, its work the SUM of the ranks' pairs.  No-op on one process."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(ms), float(pairs)
    tmax = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    tsum = torch.tensor([float(pairs)], dtype=torch.float64, device=device)
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    return float(tmax[0]), float(tsum[0])


def cfg_for_rank(name, rank):
    C = synth.config(name)
    return synth.config(name, data_seed=C.data_seed + 1000 * rank) if rank else C


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2010_11497_b200 as c2

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    C = cfg_for_rank(args.config, rank)
    offs, items = synth.generate(C)
    n, nnz = len(offs) - 1, len(items)
    d_offs = torch.from_numpy(offs).to(dev)
    d_items = torch.from_numpy(items).to(dev)
    sim_mode = 1 if args.sim == "gf" else 0
    stream = torch.cuda.current_stream(dev)
    ctx = c2.Context(local, stream=stream, timing=True)
    out = (torch.empty((n, C.k), dtype=torch.int32, device=dev), torch.empty((n, C.k), dtype=torch.uint16, device=dev),
           torch.empty((n, C.k), dtype=torch.uint16, device=dev), torch.empty((n, C.k), dtype=torch.float32, device=dev))

    def step():
        c2.build(d_offs, d_items, k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, sim_mode=sim_mode, out=out, ctx=ctx)

    cold_ms = None
    for wi in range(args.warmup):
        step()
        if wi == 0:
            cold_ms = ctx.stats()["ms_total"]  # first call: workspaces allocated, cold caches
    torch.cuda.synchronize(dev)
    stats0 = ctx.stats()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tile_ms, launches, build_ms = [], [], []
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
            st = ctx.stats()  # per-step: the library synchronised its own events inside the call
            tile_ms.append(st["ms_tile"] / max(st["tile_launches"], 1))
            build_ms.append(st["ms_total"])
            launches.append(st["launches"])
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1) / args.steps
    st = ctx.stats()
    pairs = st["pairs"]
    ms_max, pairs_all = reduce_over_ranks(ms, pairs, dev)
    value = pairs_all / (ms_max * 1e-3)

    # ---- e2e: the same build through the C ABI with host buffers (pinned), copies inside
    h_offs = torch.from_numpy(offs).pin_memory()
    h_items = torch.from_numpy(items).pin_memory()
    h_out = [torch.empty((n, C.k), dtype=d, pin_memory=True) for d in (torch.int32, torch.int16, torch.int16,
                                                                          torch.float32)]
    np_out = (h_out[0].numpy(), h_out[1].numpy().view(np.uint16), h_out[2].numpy().view(np.uint16), h_out[3].numpy())
    e2e_steps = max(1, min(args.steps, 5))
    c2.build_host(h_offs.numpy(), h_items.numpy(), k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed, sim_mode=sim_mode,
                  out=np_out, ctx=ctx)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        c2.build_host(h_offs.numpy(), h_items.numpy(), k=C.k, t=C.t, b=C.b, N=C.N, seed=C.hash_seed,
                      sim_mode=sim_mode, out=np_out, ctx=ctx)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    e2e_ms, _ = reduce_over_ranks(e2e_ms, 0, dev)
    h2d = (n + 1) * 4 + nnz * 4
    d2h = n * C.k * (4 + 2 + 2 + 4)

    if rank == 0:
        peaks, peak_src = load_peaks()
        clock = clk.summary()
        # dominant kernel: the local tile kernel K7; algorithmic work = two-pointer element
        # comparisons |P_u|+|P_v| summed over the unordered pairs it handles
        steps_total = st["work_steps"]
        tile_avg_ms = float(np.median(tile_ms))
        n_tile = max(st["tile_launches"], 1)
        # ALU peak: 148 SMs x 4 SMSP x 32 lanes x 1 int op/clk at sm_max_mhz (B200_PROFILING.md)
        sm_mhz = peaks.get("sm_max_mhz", 1965.0)
        alu_peak = 148 * 128 * sm_mhz * 1e6 / 1e12  # Tops/s
        # DRAM traffic of one K7 launch from the committed ncu --set full capture (profiles/)
        traffic, traffic_note = None, None
        try:
            with open(os.path.join(ROOT, "profiles", "r01_ncu_tile_traffic.json")) as f:
                tj = json.load(f)
            if tj.get("config") == C.name:
                traffic = tj["dram_bytes_read"] + tj["dram_bytes_write"]
                traffic_note = f"bytes per launch, {tj['launch']}; {tj['source']}"
        except (OSError, KeyError, ValueError):
            pass
        achieved = steps_total / n_tile / (tile_avg_ms * 1e-3) / 1e12
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "pairs/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": C.name, "n_users": n, "n_items": C.m, "nnz": nnz, "k": C.k, "t": C.t, "b": C.b,
                       "N": C.N, "hash_seed": C.hash_seed, "data_seed": C.data_seed, "sim": args.sim,
                       "pairs_per_step": pairs, "l2": f"inputs larger than L2 (CSR {4 * (n + 1 + nnz) / 2**20:.0f} MiB"
                       " + per-step scratch)", "parallelism": f"independent datasets per rank x{ws}"},
            "roofline": {"kernel": "k_local_tile (K7 local Jaccard + K8 top-k)", "bound": "alu",
                         "achieved": achieved, "peak": alu_peak, "unit": "Tops/s (two-pointer comparisons)",
                         "frac": achieved / alu_peak, "traffic": traffic,
                         "traffic_note": traffic_note,
                         "peak_source": f"{peak_src}: 148 SM x 128 int lanes x {sm_mhz:.0f} MHz",
                         "kernel_ms_per_launch": tile_avg_ms, "launches_per_step": n_tile,
                         "share_of_step": tile_avg_ms * n_tile / ms},
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


def oracle_sample(C, offs, items, target_pairs):
    """The largest clusters of hash function 0 (canonical order kept) up to ~target_pairs."""
    import oracle
    m = int(items.max()) + 1
    h = oracle.hash_table(C.hash_seed, 1, C.b, m)
    cl = oracle.cluster(offs, items, h, C.N)
    off, nc, mem = cl["offsets"][0], int(cl["n_clusters"][0]), cl["members"][0]
    s = np.diff(off[: nc + 1])
    chosen, P = [], 0
    for c in np.argsort(-s, kind="stable"):
        chosen.append(int(c))
        P += int(s[c]) * (int(s[c]) - 1) // 2
        if P >= target_pairs:
            break
    chosen.sort()
    n = len(offs) - 1
    segs = [mem[off[c]:off[c + 1]] for c in chosen]
    flat = np.concatenate(segs).astype(np.int32)
    sub_off = np.concatenate([[0], np.cumsum([len(x) for x in segs])]).astype(np.int32)
    sub = dict(offsets=np.full((1, n + 1), sub_off[-1], np.int32), members=np.zeros((1, n), np.int32),
               n_clusters=np.asarray([len(chosen)], np.int32))
    sub["offsets"][0, :len(sub_off)] = sub_off
    sub["members"][0, :len(flat)] = flat
    return sub, P, len(chosen)


def cpu_baseline(C, offs, items, seconds):
    import oracle
    cores = os.cpu_count() or 1
    target = int(seconds * 0.7e6 * cores)  # ~0.7M pairs/s/core measured for the oracle
    sub, P, ncl = oracle_sample(C, offs, items, target)
    t0 = time.perf_counter()
    oracle.local_knn(offs, items, sub, C.k, nthreads=cores)
    dt = time.perf_counter() - t0
    return {"value": P / dt, "unit": "pairs/s", "cores": cores, "kind": "oracle",
            "sample": f"local brute-force top-k (Alg. 2) of the {ncl} largest clusters of hash function 0 of "
                      f"{C.name}: {P} pairs in {dt:.1f} s (clustering excluded)"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    C = synth.config(args.config)
    offs, items = synth.generate(C)
    cores = os.cpu_count() or 1
    per_step = max(1, int(args.cpu_seconds * 0.7e6 * cores / max(args.steps + args.warmup, 1)))
    sub, P, ncl = oracle_sample(C, offs, items, per_step)
    for _ in range(args.warmup):
        oracle.local_knn(offs, items, sub, C.k, nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.local_knn(offs, items, sub, C.k, nthreads=cores)
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    v = P / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "pairs/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": C.name, "n_users": C.n, "k": C.k, "t": C.t, "b": C.b, "N": C.N, "sim": args.sim},
        "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": cores, "kind": "oracle",
                         "sample": f"per step: local top-k of the {ncl} largest clusters of hash function 0 "
                                   f"({P} pairs)"},
        "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(synth.CONFIGS))
    ap.add_argument("--sim", default="exact", choices=["exact", "gf"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

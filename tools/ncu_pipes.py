"""ncu pipe counts of every k_local_tile launch of one c2_build -> profiles/<out>.json (read by
bench.py's roofline).  Run on the GPU box AFTER the same command exited 0 without ncu:

    python tools/ncu_pipes.py run c5 gpurun_out/ncu_pipes_c5.csv      # (box) ncu capture
    python tools/ncu_pipes.py summarize gpurun_out/ncu_pipes_c5.csv c5 profiles/r02_ncu_tile_pipes.json
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.sum",
           "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_lsu.sum", "dram__bytes_read.sum",
           "dram__bytes_write.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active"]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(cfg, out_csv):
    cmd = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "-k", "regex:k_local_tile", "--csv",
           "--log-file", out_csv, sys.executable, os.path.join(ROOT, "tools", "run_cfg.py"), cfg, "0", "1"]
    subprocess.check_call(cmd)


def summarize(in_csv, cfg, out_json):
    rows = list(csv.DictReader(io.StringIO("".join(l for l in open(in_csv) if not l.startswith("==")))))
    per = {}
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        v = r["Metric Value"].replace(",", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "ms": 1.0,
                 "msecond": 1.0, "second": 1e3}.get(r.get("Metric Unit", ""), 1.0)  # bytes, ms
        try:
            per.setdefault(key, {})[r["Metric Name"]] = float(v) * scale
        except ValueError:
            pass
    launches = [per[k] for k in sorted(per, key=lambda x: int(x[0]))]
    tot = lambda m: sum(l.get(m, 0.0) for l in launches)  # noqa: E731
    out = {
        "config": cfg, "kernel": "k_local_tile", "launches_per_step": len(launches),
        "alu_warp_inst_per_step": tot("sm__inst_executed_pipe_alu.sum"),
        "fma_warp_inst_per_step": tot("sm__inst_executed_pipe_fma.sum"),
        "lsu_warp_inst_per_step": tot("sm__inst_executed_pipe_lsu.sum"),
        "warp_inst_per_step": tot("smsp__inst_executed.sum"),
        "alu_pct_of_peak_by_launch": [l.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active")
                                      for l in launches],
        "issue_active_pct_by_launch": [l.get("smsp__issue_active.avg.pct_of_peak_sustained_active") for l in launches],
        "dram_bytes_per_launch": (tot("dram__bytes_read.sum") + tot("dram__bytes_write.sum")) / len(launches),
        "traffic_note": "bytes per launch: dram__bytes_read.sum + dram__bytes_write.sum averaged over the "
                        "step's tile launches",
        "duration_ms_by_launch": [l.get("gpu__time_duration.sum") for l in launches],
        "source": os.path.relpath(out_json, ROOT).replace(".json", ".csv") + " (ncu --metrics, --clock-control none)",
    }
    with open(out_json, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if not isinstance(v, list)}))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], sys.argv[3])
    else:
        summarize(sys.argv[2], sys.argv[3], sys.argv[4])

"""Summarise an ncu --set full report: SOL, pipes, stalls, hottest SASS regions."""
import collections, csv, io, re, subprocess, sys

def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout

def summary(rep, regions=True, B=40):
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr = raw[0]
    for row in raw[2:]:
        d = dict(zip(hdr, row))
        print("kernel:", d.get("Kernel Name", "")[:80], "| duration:", d.get("gpu__time_duration.sum"),
              "| regs:", d.get("launch__registers_per_thread"), "| grid:", d.get("launch__grid_size"))
        want = [r"sm__throughput.avg.pct_of_peak_sustained_elapsed$", r"smsp__issue_active.avg.pct_of_peak_sustained_active$",
                r"sm__inst_executed_pipe_(alu|fma|lsu|adu|uniform|xu|cbu)\.avg\.pct_of_peak_sustained_active$",
                r"l1tex__data_pipe_lsu_wavefronts_mem_shared.sum$", r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum$",
                r"smsp__inst_executed.sum$", r"dram__bytes_read.sum$", r"dram__bytes_write.sum$",
                r"l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum$", r"lts__t_bytes.sum$",
                r"smsp__average_warps_issue_stalled_(barrier|long_scoreboard|short_scoreboard|mio_throttle|wait|not_selected|math_pipe_throttle|lg_throttle|membar|branch_resolving|dispatch_stall|no_instruction)_per_issue_active.ratio$",
                r"sm__warps_active.avg.pct_of_peak_sustained_active$", r"smsp__thread_inst_executed_per_inst_executed.ratio$",
                r"l1tex__throughput.avg.pct_of_peak_sustained_active$", r"dram__throughput.avg.pct_of_peak_sustained_elapsed$"]
        for k in hdr:
            if any(re.search(w, k) for w in want):
                print(f"   {k} = {d[k]}")
    if not regions:
        return
    sass = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    h = sass[1]
    data = [dict(zip(h, r)) for r in sass[2:] if len(r) == len(h)]
    f = lambda x: float(x.replace(",", "")) if x else 0.0
    tot = sum(f(d["Instructions Executed"]) for d in data) or 1
    samp = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data) or 1
    for i in range(0, len(data), B):
        seg = data[i:i + B]
        ie = sum(f(d["Instructions Executed"]) for d in seg)
        s = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in seg)
        if ie / tot > 0.02 or s / samp > 0.02:
            ops = collections.Counter(d["Source"].replace("@", "").split()[0] if not d["Source"].strip().startswith("@")
                                      else d["Source"].split()[1] for d in seg).most_common(5)
            print(f"  [{i:5d}] {ie / tot * 100:5.1f}% inst {s / samp * 100:5.1f}% stall  {ops}")

if __name__ == "__main__":
    summary(sys.argv[1], regions="--noregions" not in sys.argv)

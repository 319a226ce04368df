"""Per-CUDA-source-line instruction / stall totals from an ncu report (cuda,sass source view).

usage: python tools/ncu_lines.py REPORT [top] [launch-index]
"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, top=40, which=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    sections, cur_sec = [], None
    hdr = None
    cur_file = ""
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if len(r) >= 2 and r[0] == "Function Name":
            cur_sec = collections.OrderedDict()
            sections.append((r[1], cur_sec))
            continue
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or cur_sec is None or len(r) < 8 or not r[0]:
            continue
        d = dict(zip(hdr[4:], r[4:]))
        try:
            ie = float(d.get("Instructions Executed", "0") or 0)
            ws = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        a = cur_sec.setdefault((cur_file, int(r[0]), r[1].strip()[:70]), [0.0, 0.0])
        a[0] += ie
        a[1] += ws
    name, agg = sections[which]
    print(name)
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    for k, (ie, ws) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{k[0]}:{k[1]:5d} inst {ie / ti * 100:5.1f}% stall {ws / ts * 100:5.1f}%  {k[2]}")
    print(f"total inst {ti:.3e} ({len(sections)} sections)")
    return agg


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, int(sys.argv[3]) if len(sys.argv) > 3 else 0)

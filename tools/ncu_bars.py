"""Per-barrier-interval totals (instructions executed, stall samples) of one kernel in an ncu
report: SASS in program order, split at every BAR.SYNC, so phases of a barrier-structured kernel
get their own line even when their code is made of inlined helpers."""
import csv, io, subprocess, sys

def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    segs = []
    cur = [None, 0.0, 0.0, 0, {}]
    for r in rows:
        if len(r) > 3 and r[0] == "Address":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        src = d["Source"].strip()
        ie = float(d.get("Instructions Executed") or 0)
        ws = float(d.get("Warp Stall Sampling (All Samples)") or 0)
        if cur[0] is None:
            cur[0] = d["Address"]
        cur[1] += ie
        cur[2] += ws
        cur[3] += 1
        op = src.split()[0] if src else ""
        if op.startswith("@"):
            op = src.split()[1]
        cur[4][op.split(".")[0]] = cur[4].get(op.split(".")[0], 0) + ie
        if "BAR.SYNC" in src or "EXIT" == op:
            segs.append(cur)
            cur = [None, 0.0, 0.0, 0, {}]
    segs.append(cur)
    ti = sum(s[1] for s in segs) or 1
    ts = sum(s[2] for s in segs) or 1
    for i, (addr, ie, ws, n, ops) in enumerate(segs):
        top = sorted(ops.items(), key=lambda x: -x[1])[:6]
        print(f"seg{i:2d} @{addr} n={n:5d} inst {ie / ti * 100:5.1f}% stall {ws / ts * 100:5.1f}%  "
              + " ".join(f"{k}:{v / max(ie, 1) * 100:.0f}" for k, v in top))

if __name__ == "__main__":
    main(sys.argv[1])

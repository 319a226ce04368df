"""Stall-reason breakdown per barrier interval (see ncu_bars.py) of an ncu report."""
import csv, io, subprocess, sys, collections

def main(rep, want=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    segs = [collections.Counter()]
    for r in rows:
        if len(r) > 3 and r[0] == "Address":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    segs[-1][k] += float(v or 0)
                except ValueError:
                    pass
        segs[-1]["_inst"] += float(d.get("Instructions Executed") or 0)
        if "BAR.SYNC" in d["Source"]:
            segs.append(collections.Counter())
    tot = sum(sum(v for k, v in s.items() if k != "_inst") for s in segs) or 1
    for i, s in enumerate(segs):
        st = sum(v for k, v in s.items() if k != "_inst")
        if st / tot < 0.02:
            continue
        top = sorted(((k, v) for k, v in s.items() if k != "_inst"), key=lambda x: -x[1])[:6]
        print(f"seg{i:2d} stall {st / tot * 100:5.1f}%  " + " ".join(f"{k[6:]}:{v / st * 100:.0f}" for k, v in top))

if __name__ == "__main__":
    main(sys.argv[1])

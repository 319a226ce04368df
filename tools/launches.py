"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name."""
import collections, csv, sys

def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get('Metric Name') != 'gpu__time_duration.sum':
            continue
        name = d['Kernel Name'].split('(')[0].replace('void ', '')
        v = float(d['Metric Value'].replace(',', ''))
        v *= {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0}[d['Metric Unit']]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    return agg

if __name__ == '__main__' and len(sys.argv) > 2 and sys.argv[2] == '--seq':
    pass
elif __name__ == '__main__':
    agg = load(sys.argv[1])
    tot = sum(v for _, v in agg.values())
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
        print(f"{v:9.3f} ms {v / tot * 100:5.1f}%  x{c:4d}  {k}")
    print(f"total {tot:.3f} ms over {sum(c for c, _ in agg.values())} launches")


def seq(path, pat):
    """Launches whose name contains one of the comma-separated patterns, in launch order."""
    rows = list(csv.reader(open(path)))
    hdr = None
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get('Metric Name') != 'gpu__time_duration.sum':
            continue
        name = d['Kernel Name'].split('(')[0].replace('void ', '')
        if any(p in name for p in pat.split(',')):
            v = float(d['Metric Value'].replace(',', ''))
            v *= {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0}[d['Metric Unit']]
            print(f"{v:9.3f} ms  {name[:60]}")


if __name__ == '__main__' and len(sys.argv) > 2 and sys.argv[2] == '--seq':
    seq(sys.argv[1], sys.argv[3] if len(sys.argv) > 3 else 'k_local_tile,k_surv_merge')

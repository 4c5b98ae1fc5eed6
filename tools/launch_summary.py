"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import sys


def summarise(path, trains=1):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"]) / (1e3 if d["Metric Unit"] == "nsecond" or d["Metric Unit"] == "ns" else 1.0)
        a = agg.setdefault(name, [0.0, 0])
        a[0] += v
        a[1] += 1
    tot = sum(v for v, _ in agg.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total_us':>10s} {'per_train_us':>12s} {'share':>6s}")
    for k, (v, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:40s} {c:8d} {v:10.1f} {v / trains:12.1f} {v / tot:6.1%}")
    return agg


if __name__ == "__main__":
    summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)

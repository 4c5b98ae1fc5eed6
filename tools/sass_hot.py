"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia = hdr.index("Address")
isrc = hdr.index("Source")
iss = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    try:
        data.append((int(r[iss] or 0), r[ia], r[isrc], r[ie]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("total samples", tot)
for s, a, src, ex in sorted(data, reverse=True)[:n]:
    print(f"{s / tot:6.1%} {a} {src[:90]:90s} exec={ex}")

"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0] != "Address"]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iSrc = hdr.index("Source")
tot = sum(f(r[iS]) for r in data)
print("total samples", tot, "instructions", len(data))
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
agg = {}
for r in data:
    for i in stall_cols:
        agg[hdr[i]] = agg.get(hdr[i], 0) + f(r[i])
print("by reason:", sorted(((round(v / tot * 100, 1), k) for k, v in agg.items() if v), reverse=True)[:8])
for r in sorted(data, key=lambda r: -f(r[iS]))[:n]:
    st = sorted([(f(r[i]), hdr[i][6:]) for i in stall_cols], reverse=True)[:2]
    print(f"{f(r[iS]) / tot * 100:5.1f}% {r[0]} {r[iSrc][:64]:64s} {st}")

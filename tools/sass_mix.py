"""Executed-instruction mix and stall split per opcode from `ncu -i REP --page source --csv --print-source sass`
(one or more kernels; each section starts with a "Kernel Name" row).  Usage: sass_mix.py FILE.csv"""
import csv
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1], errors="replace")))
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        secs.append(cur)
    elif cur is not None and r and r[0] == "Address":
        cur[1] = r
    elif cur is not None and cur[1] is not None and len(r) == len(cur[1]):
        cur[2].append(r)
for name, hdr, data in secs:
    iE = hdr.index("Instructions Executed")
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iSrc = hdr.index("Source")
    ex, st = {}, {}
    for r in data:
        t = r[iSrc].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ex[op] = ex.get(op, 0) + f(r[iE])
        st[op] = st.get(op, 0) + f(r[iS])
    te, ts = sum(ex.values()), sum(st.values()) or 1
    print(f"== {name[:100]}\n   warp instructions executed {te:.4g}")
    for op, v in sorted(ex.items(), key=lambda kv: -kv[1])[:16]:
        print(f"   {op:10s} exec {v / te * 100:5.1f}%  stall-samples {st.get(op, 0) / ts * 100:5.1f}%")

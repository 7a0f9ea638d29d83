"""Write profiles/<tag>_configs.txt from tools/profile_configs.sh outputs (gpurun_out/):
the all-config table and, per config, its kernels by total time (ncu launch lists)."""
import csv
import sys
from collections import defaultdict

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = [f"# Round {int(tag[1:])} per-config kernel times -- tools/profile_configs.sh on 1x B200",
       "# (ncu --metrics gpu__time_duration.sum --clock-control none over tools/cfg_apply_time.py <cfg> <prec>:",
       "#  3 warm-up + 10 timed steps of one inverse + one inverse adjoint apply with a random live B_opt;",
       "#  cold-cache, serialised; the cached setup kernels of the first call appear once)", "",
       "## tools/all_configs.py (live CUDA events, CUDA graphs after the second call; fast_path 2 = ring kernels)", ""]
out += [ln.rstrip() for ln in open(f"gpurun_out/allcfg_{tag}.txt") if ln.strip()]
for cfg, prec in [(1, "c128"), (2, "c128"), (3, "c128"), (4, "c128"), (5, "c64")]:
    rows = [r for r in csv.reader(open(f"gpurun_out/launch_cfg{cfg}_{prec}.csv")) if r]
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hi + 1:]:
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        sc = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[iu], 1e-3)
        k = r[ik].split(">(")[0] + ">" if ">(" in r[ik] else r[ik].split("(")[0]
        tot[k] += v * sc
        cnt[k] += 1
    out += ["", f"## config {cfg} {prec}: kernels by total time (us)",
            f"{'kernel':<70} {'launches':>9} {'us/launch':>10}"]
    for k in sorted(tot, key=lambda k: -tot[k])[:12]:
        out.append(f"{k[:70]:<70} {cnt[k]:>9} {tot[k] / cnt[k]:>10.1f}")
open(f"profiles/{tag}_configs.txt", "w").write("\n".join(out) + "\n")
print("\n".join(out[:20]))

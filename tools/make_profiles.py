"""Write profiles/<tag>_launches.{txt,csv}, profiles/<tag>_ncu_full.txt and
profiles/ncu_traffic.json from the outputs of tools/profile_round.sh (gpurun_out/)."""
import csv
import shutil
import subprocess
import sys
from collections import defaultdict

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = f"gpurun_out/launches_{tag}.csv"
rows = [r for r in csv.reader(open(src)) if r]
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[hi + 1:]:
    try:
        v = float(r[iv].replace(",", ""))
    except ValueError:
        continue
    sc = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[iu], 1e-6)
    k = r[ik].split(">(")[0] + ">" if ">(" in r[ik] else r[ik].split("(")[0]
    tot[k] += v * sc
    cnt[k] += 1
apply = [k for k in tot if any(s in k for s in ("k_pass_", "k_spread", "k_gather", "k_ring_halo", "ring::"))]
steps = max(cnt[k] for k in apply)  # 3 warm-up + 3 timed + 3 stage-timed steps of bench.py --steps 3 --warmup 3
app = sum(tot[k] for k in apply)
L = [f"# Round {tag[1:]} launch list -- config 5 (M=2^20, N=2^21 jittered, m=8, sigma=2, 64 RHS, complex128), 1x B200",
     "# Command (tools/profile_round.sh): ncu --metrics gpu__time_duration.sum --clock-control none --csv \\",
     f"#   --log-file launches_{tag}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-configs",
     "# Per-launch times are cold-cache and serialised (ncu); bench.py's live CUDA-event stage times are the",
     "# numbers in the bench line -- the SHARE of each kernel in the step is what must agree.",
     "", f"Apply kernels ({steps} steps = 3 warm-up + 3 timed + 3 with per-stage events; one launch of each per step):",
     f"{'kernel':60s} {'launches':>8s} {'ms/launch':>10s} {'share':>7s}"]
for k in sorted(apply, key=lambda k: -tot[k]):
    L.append(f"{k[:60]:60s} {cnt[k]:8d} {tot[k] / cnt[k]:10.3f} {100 * tot[k] / app:6.1f}%")
L.append(f"sum per step: {app / steps:.3f} ms")
L += ["", "All launches of the process (setup kernels run once, untimed):", f"{'kernel':92s} {'launches':>8s} {'total ms':>10s}"]
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
    L.append(f"{k[:92]:92s} {cnt[k]:8d} {v:10.3f}")
open(f"profiles/{tag}_launches.txt", "w").write("\n".join(L) + "\n")
shutil.copy(src, f"profiles/{tag}_launches.csv")
raw = subprocess.run([sys.executable, "tools/ncu_summary.py", "raw", f"gpurun_out/full_{tag}.ncu-rep"],
                     capture_output=True, text=True).stdout
head = [f"# Round {tag[1:]} ncu --set full summary -- config 5 c128, 64 RHS, one launch of each apply kernel",
        "# Command (tools/profile_round.sh): ncu --set full --import-source on --clock-control none \\",
        "#   -k regex:'k_pass_|k_spread|k_gather|ring::' -c 6 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-configs",
        "# Algorithmic bytes per launch (DESIGN.md 7): spread 4.59 GB, pass A fwd 4.29 GB, pass B fwd 3.22 GB,",
        "#   pass A adj 3.22 GB, pass B adj 4.29 GB, gather 4.59 GB; dram bytes below are what the kernel moved.", ""]
open(f"profiles/{tag}_ncu_full.txt", "w").write("\n".join(head) + raw)
subprocess.check_call([sys.executable, "tools/ncu_traffic.py", f"gpurun_out/full_{tag}.ncu-rep", "profiles/ncu_traffic.json",
                       tag, "c128", "64"], stdout=subprocess.DEVNULL)
print("\n".join(L[:16]))

# hot-path shares: the config-5 c128 launches only (the launch list also holds the per-config
# record's kernels -- config 3 runs the same ring templates at < 0.3 ms, config 5 c64 the float ones)
sel = [("spread", "ring::k_spread_ring<double, 8>", 0.3), ("fft_forward", "k_pass_a_ip<double, (int)-1, 0, 1024", 0.0),
       ("trunc_deconv", "k_pass_b_ip<double, (int)-1, 0, 2048", 0.0), ("deconv_pad", "k_pass_a_ip<double, 1, 1, 1024", 0.0),
       ("fft_inverse", "k_pass_b_ip<double, 1, 1, 2048", 0.0), ("gather", "ring::k_gather_ring<double, 8>", 0.3)]
acc = {s[0]: [0.0, 0] for s in sel}
for r in rows[hi + 1:]:
    try:
        v = float(r[iv].replace(",", ""))
    except ValueError:
        continue
    ms = v * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[iu], 1e-6)
    for name, pat, lo in sel:
        if pat in r[ik] and ms > lo:
            acc[name][0] += ms
            acc[name][1] += 1
tot5 = sum(a[0] for a in acc.values())
S = ["# config-5 c128 hot-path kernels in the launch list of `bench.py --steps 3 --warmup 3` (cold, serialised",
     "# ncu durations; the config-3 launches of the same kernel templates, < 0.3 ms, excluded)",
     f"{'stage':14s} {'launches':>8s} {'ms/launch':>10s} {'share':>7s}"]
for name, _, _ in sel:
    t, c = acc[name]
    S.append(f"{name:14s} {c:8d} {t / max(c, 1):10.4f} {100 * t / tot5:6.1f}%")
open(f"profiles/{tag}_launch_shares.txt", "w").write("\n".join(S) + "\n")
print("\n".join(S))

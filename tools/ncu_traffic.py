"""Per-stage DRAM traffic from one `ncu --set full` capture of the apply kernels
(tools/profile_round.sh) -> profiles/ncu_traffic.json, read by bench.py for the
roofline's "traffic" field.

    python tools/ncu_traffic.py gpurun_out/full_r01.ncu-rep profiles/ncu_traffic.json r01 [c128] [64]
"""
import csv
import io
import json
import re
import subprocess
import sys

# kernel-name pattern -> bench stage (fused 1-D path, see include/inft.h stage list)
STAGES = [
    (r"k_spread", "spread"),
    (r"k_pass_a(_ip)?<(double|float), \(int\)-1, 0,", "fft_forward"),
    (r"k_pass_b(_ip)?<(double|float), \(int\)-1, 0,", "trunc_deconv"),
    (r"k_pass_a(_ip)?<(double|float), 1, 1,", "deconv_pad"),
    (r"k_pass_b(_ip)?<(double|float), 1, 1,", "fft_inverse"),
    (r"k_gather", "gather"),
]


def main():
    rep, out, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    prec = sys.argv[4] if len(sys.argv) > 4 else "c128"
    rhs = int(sys.argv[5]) if len(sys.argv) > 5 else 64
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ik = hdr.index("Kernel Name")
    ir, iw, it = (hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum"),
                  hdr.index("gpu__time_duration.sum"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tscale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
    stages = {}
    for r in rows[2:]:
        name = r[ik]
        for pat, st in STAGES:
            if re.search(pat, name) and st not in stages:
                rd = float(r[ir].replace(",", "")) * scale[units[ir]]
                wr = float(r[iw].replace(",", "")) * scale[units[iw]]
                stages[st] = {"kernel": name.split(">(")[0] + ">", "dram_read": rd, "dram_write": wr,
                              "dram_bytes": rd + wr,
                              "ncu_ms": float(r[it].replace(",", "")) * tscale[units[it]]}
    doc = {"source": f"profiles/{tag}_ncu_full.txt (ncu --set full --clock-control none, one launch per kernel)",
           "prec": prec, "rhs": rhs, "stages": stages}
    with open(out, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()

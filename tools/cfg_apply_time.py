"""Apply timing of one BASELINE config on its own RHS count (stage profile), random B_opt."""
import sys

import numpy as np
import torch

import paper_1811_05335_b200 as P
import synth as S

cid = int(sys.argv[1])
prec = sys.argv[2] if len(sys.argv) > 2 else "c128"
c = S.config(cid)
x = S.make_nodes(c)
M = c["M"][0] if c["d"] == 1 else c["M"]
sigma, m, R = c["sigma"], c["m"], c["R"] if cid != 5 else 64
rng = np.random.default_rng(0)
# live slots = the support of the window matrix B (positive Kaiser-Bessel weights)
live = P.Plan(x, M, sigma, m).precompute("plain").get_bopt() != 0
w = rng.standard_normal(live.shape) * live
plan = P.Plan(x, M, sigma, m, precision=prec).set_bopt(w, "alg2")
dt = torch.complex128 if prec == "c128" else torch.complex64
Mt = int(np.prod(M))
f = torch.randn(R, x.shape[0], dtype=dt, device="cuda")
h = torch.randn(R, Mt, dtype=dt, device="cuda")
for _ in range(3):
    plan.apply(f)
    plan.adjoint_apply(h)
torch.cuda.synchronize()
plan.set_profiling(True)
plan.get_profile(reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 10
e0.record()
for _ in range(K):
    plan.apply(f)
    plan.adjoint_apply(h)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
prof = plan.get_profile()
info = plan.info()
print(f"config {cid} {prec} R={R}: step {ms:.3f} ms ({2 * R / ms * 1e3:.0f} solves/s) fast_path={info['fast_path']} "
      f"fused_fft={info['fused_fft']} perm_identity={info['perm_identity']}")
print({k: round(v[0] / max(v[1], 1), 4) for k, v in prof.items()})

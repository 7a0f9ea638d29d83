"""Apply timing of every BASELINE config (its own R, random live B_opt), c128 and c64:
one table for DESIGN.md / profiles.  Step = one inverse + one inverse adjoint apply."""
import numpy as np
import torch

import paper_1811_05335_b200 as P
import synth as S

rows = []
for cid in (1, 2, 3, 4, 5):
    c = S.config(cid)
    x = S.make_nodes(c)
    M = c["M"][0] if c["d"] == 1 else c["M"]
    sigma, m = c["sigma"], c["m"]
    R = c["R"] if cid != 5 else 64
    # live slots = the support of the window matrix B (positive Kaiser-Bessel weights)
    live = P.Plan(x, M, sigma, m).precompute("plain").get_bopt() != 0
    w = np.random.default_rng(cid).standard_normal(live.shape) * live
    for prec in ("c128", "c64"):
        plan = P.Plan(x, M, sigma, m, precision=prec).set_bopt(w, "alg2")
        dt = torch.complex128 if prec == "c128" else torch.complex64
        f = torch.randn(R, x.shape[0], dtype=dt, device="cuda")
        h = torch.randn(R, int(np.prod(M)), dtype=dt, device="cuda")
        for _ in range(3):
            plan.apply(f)
            plan.adjoint_apply(h)
        torch.cuda.synchronize()
        K = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            plan.apply(f)
            plan.adjoint_apply(h)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        info = plan.info()
        rows.append((cid, prec, R, ms, 2 * R / ms * 1e3, info["fast_path"], info["fused_fft"]))
print(f"{'cfg':>3} {'prec':>5} {'R':>4} {'ms/step':>9} {'solves/s':>12} fast_path fused_fft")
for r in rows:
    print(f"{r[0]:>3} {r[1]:>5} {r[2]:>4} {r[3]:9.4f} {r[4]:12.0f} {r[5]:>9} {r[6]:>9}")

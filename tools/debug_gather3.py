import os, subprocess, sys
CASE = r'''
import numpy as np, torch, sys, os
sys.path.insert(0, ".")
import synth as S, oracle as O
import paper_1811_05335_b200 as P
N, M, R = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
m = 8
x = S.jittered(N, 4)
w = np.random.default_rng(1).standard_normal((N, 2*m+1)) * O.slot_live(x, 2*M, m)
prec = os.environ["PREC"]
plan = P.Plan(x, M, 2.0, m, precision=prec).set_bopt(w, "alg2")
dt = torch.complex64 if prec == "c64" else torch.complex128
g = torch.Generator(device="cuda").manual_seed(5)
h = torch.randn(R, M, dtype=dt, device="cuda", generator=g)
outs = [plan.adjoint_apply(h).cpu().numpy().astype(np.complex128) for _ in range(4)]
np.save("/tmp/o_%s_%s.npy" % (os.environ["INFT_FORCE_REG"], os.environ.get("INFT_DEBUG_SPREAD","0")), np.stack(outs))
'''
import numpy as np
for prec in ("c64", "c128"):
    ref = None
    for reg, dbg in (("1", "0"), ("0", "0"), ("0", "16"), ("0", "32"), ("0", "48")):
        env = {**os.environ, "INFT_FORCE_REG": reg, "INFT_DEBUG_SPREAD": dbg, "PREC": prec}
        r = subprocess.run([sys.executable, "-c", CASE, str(1 << 21), str(1 << 20), "64"], capture_output=True, text=True, timeout=600, env=env)
        if r.returncode:
            print(prec, reg, dbg, "rc", r.returncode, r.stderr[-300:]); continue
        o = np.load("/tmp/o_%s_%s.npy" % (reg, dbg))
        if ref is None:
            ref = o[0]
        tol = 1e-5 if prec == "c64" else 1e-12
        errs = [float(np.max(np.abs(oo - ref)) / np.max(np.abs(ref))) for oo in o]
        nbad = [int((np.abs(oo - ref).max(axis=1) > tol * np.abs(ref).max()).sum()) for oo in o]
        print(prec, "reg", reg, "dbg", dbg, "maxerr", ["%.1e" % e for e in errs], "bad rows", nbad, flush=True)

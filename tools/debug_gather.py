"""c64 staged gather vs register gather at config-5 scale, repeated (race check)."""
import os
import subprocess
import sys

CASE = r'''
import numpy as np, torch, sys
sys.path.insert(0, ".")
import synth as S, oracle as O
import paper_1811_05335_b200 as P
prec, N, M, R = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
m = 8
x = S.jittered(N, 4)
w = np.random.default_rng(1).standard_normal((N, 2*m+1)) * O.slot_live(x, 2*M, m)
plan = P.Plan(x, M, 2.0, m, precision=prec).set_bopt(w, "alg2")
dt = torch.complex128 if prec == "c128" else torch.complex64
g = torch.Generator(device="cuda").manual_seed(5)
h = torch.randn(R, M, dtype=dt, device="cuda", generator=g)
outs = [plan.adjoint_apply(h).cpu().numpy().astype(np.complex128) for _ in range(3)]
ref = O.apply_adjoint(x, M, 2.0, m, w, 1.0, h[:1].cpu().numpy().astype(np.complex128))
print("errs", [O.rel_l2(o[:1], ref) for o in outs], "rep", O.rel_l2(outs[0], outs[1]), O.rel_l2(outs[1], outs[2]))
'''
for env_reg in ("0", "1"):
    for c in [("c64", 1 << 21, 1 << 20, 64), ("c64", 1 << 18, 1 << 17, 64), ("c128", 1 << 21, 1 << 20, 64)]:
        env = {**os.environ, "INFT_FORCE_REG": env_reg}
        r = subprocess.run([sys.executable, "-c", CASE, *map(str, c)], capture_output=True, text=True, timeout=600, env=env)
        out = (r.stdout + r.stderr).strip().splitlines()
        print("reg", env_reg, c, "rc", r.returncode, (out[-1] if out else "")[:300], flush=True)

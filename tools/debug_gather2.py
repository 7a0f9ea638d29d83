"""Locate staged-gather discrepancies (RHS rows, node positions) vs the register gather."""
import os
import subprocess
import sys

CASE = r'''
import numpy as np, torch, sys, os
sys.path.insert(0, ".")
import synth as S, oracle as O
import paper_1811_05335_b200 as P
N, M, R = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
m = 8
x = S.jittered(N, 4)
w = np.random.default_rng(1).standard_normal((N, 2*m+1)) * O.slot_live(x, 2*M, m)
plan = P.Plan(x, M, 2.0, m, precision=os.environ.get("PREC","c128")).set_bopt(w, "alg2")
g = torch.Generator(device="cuda").manual_seed(5)
h = torch.randn(R, M, dtype=(torch.complex64 if os.environ.get("PREC")=="c64" else torch.complex128), device="cuda", generator=g)
a = [plan.adjoint_apply(h).cpu().numpy().astype(np.complex128) for _ in range(3)][-1]
np.save("/tmp/out_%s.npy" % os.environ.get("INFT_FORCE_REG","0"), a)
'''
for env_reg in ("1", "0"):
    env = {**os.environ, "INFT_FORCE_REG": env_reg, "PREC": "c64"}
    r = subprocess.run([sys.executable, "-c", CASE, str(1 << 21), str(1 << 20), "64"], capture_output=True, text=True, timeout=600, env=env)
    print("reg", env_reg, r.returncode, r.stderr[-300:], flush=True)
import numpy as np
a = np.load("/tmp/out_1.npy"); b = np.load("/tmp/out_0.npy")
err = np.abs(a - b) / np.abs(a).max()
rows = np.nonzero(err.max(axis=1) > 1e-5)[0]
print("bad rows", rows.tolist()[:64], "count", len(rows))
if len(rows):
    r0 = rows[0]
    bad = np.nonzero(err[r0] > 1e-5)[0]
    print("row", r0, "bad nodes", len(bad), "first", bad[:20].tolist(), "last", bad[-10:].tolist())
    # per-chunk (32 segments x 16 nodes = 512 nodes) histogram of bad nodes
    ch = np.bincount(bad // 512)
    nz = np.nonzero(ch)[0]
    print("chunks with bad nodes", len(nz), nz[:30].tolist(), ch[nz[:30]].tolist())
    for rr in rows[:8]:
        bb = np.nonzero(err[rr] > 1e-5)[0]
        print("row", rr, "nbad", len(bb), "chunks", np.unique(bb // 512)[:10].tolist())

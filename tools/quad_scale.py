"""Quadratic case at scale (fast summation): plan (a, b by the ln|sin| fast summation) and
apply / adjoint times for N = 2^14..2^22 jittered nodes, R = 16, with the exactness check on a
sparse fhat (8 frequencies: f = A fhat by 8 exponentials per node).

    python tools/quad_scale.py
"""
import os
import sys
import time

import numpy as np
import torch

_ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, _ROOT)
import paper_1811_05335_b200 as P  # noqa: E402
import synth as S  # noqa: E402

R = 16
print(f"{'N':>9} {'plan s':>8} {'apply ms':>9} {'adjoint ms':>11} {'solves/s':>10} {'rel err fhat':>13} {'rel err f':>10}")
for lg in range(14, 23, 2):
    N = 1 << lg
    y = S.jittered(N, 1)
    t0 = time.perf_counter()
    q = P.QuadPlan(y)
    torch.cuda.synchronize()
    tp = time.perf_counter() - t0
    rng = np.random.default_rng(lg)
    ks = rng.choice(N, 8, replace=False)
    fh = np.zeros((R, N), dtype=np.complex128)
    fh[:, ks] = rng.standard_normal((R, 8)) + 1j * rng.standard_normal((R, 8))
    yt = torch.as_tensor(y, device="cuda")
    kk = torch.as_tensor(ks - N // 2, device="cuda", dtype=torch.float64)
    E = torch.exp(2j * np.pi * torch.outer(yt, kk).to(torch.complex128))       # [N][8]
    f = (torch.as_tensor(fh[:, ks], device="cuda") @ E.T).contiguous()          # A fhat
    fs = torch.zeros(R, N, dtype=torch.complex128, device="cuda")
    js = rng.choice(N, 8, replace=False)
    fs[:, js] = torch.as_tensor(rng.standard_normal((R, 8)) + 1j * rng.standard_normal((R, 8)), device="cuda")
    kall = torch.arange(-N // 2, N // 2, device="cuda", dtype=torch.float64)
    h = (fs[:, js] @ torch.exp(-2j * np.pi * torch.outer(yt[js], kall).to(torch.complex128))).contiguous()  # A^* f
    out = q.apply(f)
    oa = q.adjoint_apply(h)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    for _ in range(5):
        q.apply(f, out=out)
    ev[1].record()
    for _ in range(5):
        q.adjoint_apply(h, out=oa)
    ev[2].record()
    torch.cuda.synchronize()
    ta, tb = ev[0].elapsed_time(ev[1]) / 5, ev[1].elapsed_time(ev[2]) / 5
    e1 = (torch.linalg.norm(out - torch.as_tensor(fh, device="cuda")) / np.linalg.norm(fh)).item()
    e2 = (torch.linalg.norm(oa - fs) / torch.linalg.norm(fs)).item()
    print(f"{N:>9} {tp:>8.3f} {ta:>9.3f} {tb:>11.3f} {2 * R / (ta + tb) * 1e3:>10.0f} {e1:>13.2e} {e2:>10.2e}", flush=True)

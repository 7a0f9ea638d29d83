"""Where the quadratic case's 1e-9 parity bar comes from.

For jittered nodes at N = 1024, 4096, 16384 print
  * max |atilde|, max |btilde| -- the log-domain sums, O(N) in magnitude;
  * the oracle's own rounding floor: float64 direct sums against numpy longdouble ones
    (absolute error of atilde/btilde = RELATIVE error of a = e^{atilde + s}, b = e^{btilde - s});
  * GPU direct sums (INFT_QUAD_DIRECT=1) and GPU fast summation against the oracle: relative
    error of a, b and relative l2 error of both applies;
  * the cancellation factor of the Lagrange sums, sum_j |f_j b_j cot| / |sum_j f_j b_j cot|.

Run on a GPU box:  PYTHONPATH=. python tools/quad_error_budget.py
"""
import os

import numpy as np
import torch

import oracle as O
import paper_1811_05335_b200 as P
import synth as S
from oracle import quadratic as Q


def ld_logs(y, x):
    yl, xl = y.astype(np.longdouble), x.astype(np.longdouble)
    pi = np.longdouble(np.pi) + np.longdouble(1.2246467991473532e-16)  # pi to ~1e-32
    at = np.empty(x.size, dtype=np.longdouble)
    bt = np.empty(y.size, dtype=np.longdouble)
    for i in range(x.size):
        at[i] = np.log(np.abs(np.sin(pi * (xl[i] - yl)))).sum()
    for j in range(y.size):
        d = np.abs(np.sin(pi * (yl[j] - yl)))
        d[j] = 1
        bt[j] = -np.log(d).sum()
    return at, bt


def main():
    for N in (1024, 4096, 16384):
        y = S.jittered(N, N)
        x = Q.targets(N)
        atil, _, btil, _ = Q.log_coeffs(y, x)
        line = f"N = {N}: max|atilde| {np.abs(atil).max():.1f}, max|btilde| {np.abs(btil).max():.1f}"
        if N <= 4096:
            al, bl = ld_logs(y, x)
            line += (f"; oracle float64 vs longdouble: |d atilde| {float(np.abs(atil - al).max()):.1e}, "
                     f"|d btilde| {float(np.abs(btil - bl).max()):.1e}")
        print(line)
        xo, ao, bo, so = Q.coeffs(y)
        qf = P.QuadPlan(y)
        os.environ["INFT_QUAD_DIRECT"] = "1"
        try:
            qd = P.QuadPlan(y)
        finally:
            del os.environ["INFT_QUAD_DIRECT"]
        for name, q in (("GPU direct", qd), ("GPU fast  ", qf)):
            _, a, b, s = q.coeffs()
            print(f"  {name} vs oracle: rel a {np.abs(a / ao - 1).max():.1e}, rel b {np.abs(b / bo - 1).max():.1e}, "
                  f"|s - s_o| {abs(s - so):.1e}", end="")
            if N <= 4096:
                f = S.normal_complex(3, N, 1)
                h = S.normal_complex(3, N, 2)
                ei = O.rel_l2(q.apply(torch.from_numpy(f).cuda()).cpu().numpy(), Q.inverse(y, f))
                ea = O.rel_l2(q.adjoint_apply(torch.from_numpy(h).cuda()).cpu().numpy(), Q.adjoint(y, h))
                print(f"; inverse {ei:.1e}, adjoint {ea:.1e}")
            else:
                print()
        _, af, bf, _ = qf.coeffs()
        _, ad, bd, _ = qd.coeffs()
        print(f"  GPU fast vs GPU direct: rel a {np.abs(af / ad - 1).max():.1e}, rel b {np.abs(bf / bd - 1).max():.1e}")
        if N <= 4096:
            f = S.normal_complex(1, N, 1)[0]
            C = 1.0 / np.tan(np.pi * (x[:, None] - y[None, :]))
            t = (f * bo)[None, :] * C
            canc = np.abs(t).sum(axis=1) / np.abs(t.sum(axis=1))
            print(f"  cancellation of sum_j f_j b_j cot(pi (x_l - y_j)): median {np.median(canc):.1e}, max {canc.max():.1e}")


if __name__ == "__main__":
    main()

"""The paper's numerical experiments on the GPU, qualitatively: the
figures' PDFs are not in the container, so the output is tables of the same quantities.

  E1  Alg. 1 Frobenius norms ||A D^* F^* B^* - M I_N||_F, window B vs B_opt   (Ex. P:968-1049)
  E2  Alg. 1 setup time, B-spline vs Dirichlet, m = 2, sigma = 1, N = 128     (Fig. P:1024-1030)
  E3  Alg. 2 Frobenius norms ||F D A^* B - I_{M_sigma}||_F, B vs B_opt         (Ex. P:1367-1451)
  E4  Alg. 2 setup time, B-spline vs Dirichlet, m = 2, sigma = 1, M = 128     (Fig. P:1425-1431)
  E5  Alg. 1 errors per node, inverse and inverse adjoint                     (Ex. P:1052-1143)
  E6  Alg. 2 errors per node, inverse and inverse adjoint                     (Ex. P:1467-1552)
  E7  quadratic case errors per node (Lagrange inverse, fast summation)      (Ex. P:501-544)

Every setup and apply runs in the library (libinft.so); the dense matrices of the metrics
(A, F, D, B from the plan's own weights and deconvolution table) are formed with torch on
the GPU.  Inputs: jittered nodes (eq. jittered_nodes, jitter 1/4), Chebyshev nodes, fhat_k
uniform in [1, 100].

    python tools/experiments.py [--quick] > profiles/r01_experiments.txt
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

_ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, _ROOT)
import paper_1811_05335_b200 as P  # noqa: E402
import synth as S  # noqa: E402

dev = torch.device("cuda")
c128 = torch.complex128


def mat_A(x, M):
    k = torch.arange(-M // 2, M // 2, device=dev, dtype=torch.float64)
    return torch.exp(2j * np.pi * torch.outer(torch.as_tensor(x, device=dev), k).to(c128))


def mat_F(M, Ms):
    l = torch.arange(-Ms // 2, Ms // 2, device=dev, dtype=torch.float64)
    k = torch.arange(-M // 2, M // 2, device=dev, dtype=torch.float64)
    return torch.exp(2j * np.pi * torch.outer(l, k).to(c128) / Ms)


def dense_B(plan, Ms):
    """B (N x M_sigma, columns l = -Ms/2..Ms/2-1) from the plan's slot weights and bins."""
    w = torch.as_tensor(plan.get_bopt(), device=dev).to(c128)
    l0, _, _ = plan.get_bins()
    N, Pw = w.shape
    cols = (torch.as_tensor(l0, device=dev, dtype=torch.int64)[:, None] + torch.arange(Pw, device=dev)[None, :]
            + Ms // 2) % Ms
    B = torch.zeros(N, Ms, dtype=c128, device=dev)
    B.index_put_((torch.arange(N, device=dev)[:, None].expand(N, Pw), cols), w, accumulate=True)
    return B


def D_of(plan, s):
    return torch.as_tensor(plan.get_deconv(), device=dev).to(c128) / s  # d = s/(Ms what)


def nodes(kind, N, seed=0):
    return S.jittered(N, seed) if kind == "jittered" else S.chebyshev(N)


def fhat_uniform(R, M, seed):
    return np.random.default_rng(seed).uniform(1.0, 100.0, (R, M)).astype(np.complex128)


def errs(est, ref, N):
    d = (est - ref).reshape(-1)
    r = ref.reshape(-1)
    out = []
    for p in (2, float("inf")):
        a = torch.linalg.vector_norm(d, p).item()
        out += [a / N, a / (N * torch.linalg.vector_norm(r, p).item())]
    return out  # e2abs/N, e2rel/N, einf_abs/N, einf_rel/N


def plan_for(x, M, sigma, m, window, method):
    p = P.Plan(x, M, sigma, m, window=window)
    p.precompute(method)
    return p


def e1(cs, rows):
    print("## E1  Alg. 1: ||A D^* F^* B^* - M I_N||_F (window B) vs B_opt; N = 128 jittered unless noted")
    print(f"{'nodes':>10} {'N':>4} {'m':>2} {'sig':>4} {'M':>5} {'B-spline B':>12} {'B-spline Bopt':>14} {'Dirichlet Bopt':>15}")
    for kind, N, m, sigma in rows:
        x = nodes(kind, N, 1)
        for c in cs:
            M = 1 << c
            Ms = int(sigma * M)
            if m > Ms // 2:
                continue
            A, F = mat_A(x, M), mat_F(M, Ms)
            vals = []
            for window, method in (("bspline", "plain"), ("bspline", "alg1"), ("dirichlet", "alg1")):
                p = plan_for(x, M, sigma, m, window, method)
                s = 1.0 / M if method == "alg1" else 1.0
                D = D_of(p, s)
                X = A @ (D.conj()[:, None] * (F.conj().T @ dense_B(p, Ms).conj().T))
                vals.append(torch.linalg.norm(X - M * torch.eye(N, device=dev, dtype=c128)).item())
            print(f"{kind:>10} {N:>4} {m:>2} {sigma:>4} {M:>5} {vals[0]:>12.3e} {vals[1]:>14.3e} {vals[2]:>15.3e}")
    print()


def setup_time(x, M, sigma, m, window, method):
    plan_for(x, M, sigma, m, window, method)  # warm (cuFFT plans, tables)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan_for(x, M, sigma, m, window, method)
    return time.perf_counter() - t0


def e2(cs):
    print("## E2  Alg. 1 setup time on the GPU (s, includes plan creation), m = 2, sigma = 1, N = 128 jittered")
    print(f"{'M':>6} {'B-spline':>10} {'Dirichlet':>10}")
    x = nodes("jittered", 128, 1)
    for c in cs:
        M = 1 << c
        print(f"{M:>6} {setup_time(x, M, 1.0, 2, 'bspline', 'alg1'):>10.4f} {setup_time(x, M, 1.0, 2, 'dirichlet', 'alg1'):>10.4f}")
    print()


def e3(cs, rows):
    print("## E3  Alg. 2: ||F D A^* B - I_Msigma||_F (window B) vs B_opt; M = 128; rank bound sqrt(Msigma - M)")
    print(f"{'nodes':>10} {'m':>2} {'sig':>4} {'N':>6} {'B-spline B':>12} {'B-spline Bopt':>14} {'Dirichlet Bopt':>15} {'bound':>8}")
    M = 128
    for kind, m, sigma in rows:
        Ms = int(sigma * M)
        F = mat_F(M, Ms)
        for c in cs:
            N = 1 << c
            x = nodes(kind, N, 2)
            A = mat_A(x, M)
            vals = []
            for window, method in (("bspline", "plain"), ("bspline", "alg2"), ("dirichlet", "alg2")):
                p = plan_for(x, M, sigma, m, window, method)
                D = D_of(p, 1.0)
                X = F @ (D[:, None] * (A.conj().T @ dense_B(p, Ms)))
                vals.append(torch.linalg.norm(X - torch.eye(Ms, device=dev, dtype=c128)).item())
            print(f"{kind:>10} {m:>2} {sigma:>4} {N:>6} {vals[0]:>12.3e} {vals[1]:>14.3e} {vals[2]:>15.3e} "
                  f"{np.sqrt(Ms - M):>8.3f}")
    print()


def e4(cs):
    print("## E4  Alg. 2 setup time on the GPU (s, includes plan creation), m = 2, sigma = 1, M = 128 jittered")
    print(f"{'N':>6} {'B-spline':>10} {'Dirichlet':>10}")
    for c in cs:
        N = 1 << c
        x = nodes("jittered", N, 2)
        print(f"{N:>6} {setup_time(x, 128, 1.0, 2, 'bspline', 'alg2'):>10.4f} "
              f"{setup_time(x, 128, 1.0, 2, 'dirichlet', 'alg2'):>10.4f}")
    print()


def err_table(title, cases, method):
    print(title)
    print(f"{'N':>6} {'M':>6} {'m':>3} | inverse: {'e2abs/N':>9} {'e2rel/N':>9} {'einf/N':>9} {'einfrel/N':>9} | "
          f"adjoint: {'e2abs/N':>9} {'e2rel/N':>9} {'einf/N':>9} {'einfrel/N':>9}")
    for N, M, m in cases:
        Ms = 2 * M
        m = min(m, Ms // 2)
        x = nodes("jittered", N, 3)
        p = plan_for(x, M, 2.0, m, "dirichlet", method)
        A = mat_A(x, M)
        fh = torch.as_tensor(fhat_uniform(1, M, N + M), device=dev)
        f = (A @ fh.T).T.contiguous()
        fc = p.apply(f)
        # Alg. 1 (underdetermined) compares A fcheck with f (eq. errors_per_node_underdet,
        # P:1061-1065); Alg. 2 compares fcheck with fhat (eq. errors_per_node_lagrange)
        inv = errs((A @ fc.T).T, f, N) if method == "alg1" else errs(fc, fh, N)
        h = (A.conj().T @ f.T).T.contiguous()
        adj = errs(p.adjoint_apply(h), f, N)
        print(f"{N:>6} {M:>6} {m:>3} |          {inv[0]:>9.2e} {inv[1]:>9.2e} {inv[2]:>9.2e} {inv[3]:>9.2e} | "
              f"         {adj[0]:>9.2e} {adj[1]:>9.2e} {adj[2]:>9.2e} {adj[3]:>9.2e}")
    print()


def e7(cs):
    print("## E7  quadratic case M = N (Lagrange inverse; fast summation for N >= 512, direct sums below): errors per node, jittered, fhat in [1,100]")
    print(f"{'N':>6} {'e2abs/N':>9} {'e2rel/N':>9} {'einf/N':>9} {'einfrel/N':>9} {'ms':>8}")
    for c in cs:
        N = 1 << c
        y = nodes("jittered", N, 4)
        fh = torch.as_tensor(fhat_uniform(1, N, N), device=dev)
        k = torch.arange(-N // 2, N // 2, device=dev, dtype=torch.float64)
        yt = torch.as_tensor(y, device=dev)
        f = torch.zeros(1, N, dtype=c128, device=dev)
        for j0 in range(0, N, 4096):
            Aj = torch.exp(2j * np.pi * torch.outer(yt[j0:j0 + 4096], k).to(c128))
            f[0, j0:j0 + 4096] = Aj @ fh[0]
        q = P.QuadPlan(y)
        q.apply(f)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        est = q.apply(f)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        e = errs(est, fh, N)
        print(f"{N:>6} {e[0]:>9.2e} {e[1]:>9.2e} {e[2]:>9.2e} {e[3]:>9.2e} {dt:>8.2f}")
    print()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="smaller sweeps (CI smoke)")
    a = ap.parse_args()
    q = a.quick
    print("# NEXT-4: the paper's experiments on 1x B200 (tools/experiments.py); quantities of the figures,")
    print("# values from this build (no numeric targets exist: the figure PDFs are not in the container)\n")
    e1(range(4, 9 if q else 13), [("jittered", 128, 2, 1.0), ("jittered", 128, 2, 2.0), ("jittered", 128, 4, 1.0)]
       + ([] if q else [("chebyshev", 16, 2, 1.0), ("chebyshev", 64, 2, 1.0), ("chebyshev", 128, 2, 1.0)]))
    e2(range(4, 9 if q else 13))
    e3(range(2, 9 if q else 15), [("jittered", 2, 1.0), ("jittered", 2, 2.0), ("jittered", 4, 1.0)]
       + ([] if q else [("chebyshev", 2, 1.0)]))
    e4(range(2, 9 if q else 15))
    n1 = range(1, 8 if q else 13)
    err_table("## E5  Alg. 1 (Dirichlet, sigma = 2, jittered): errors per node (inverse: ||A fcheck - f||, "
              "adjoint: ||ftilde - f||); (a) M = 4N, m = 4",
              [(1 << c, 4 << c, 4) for c in n1], "alg1")
    err_table("## E5  Alg. 1: (b) N = 512, M = 2048, m = 4..12", [(512, 2048, m) for m in range(4, 13)], "alg1")
    err_table("## E6  Alg. 2 (Dirichlet, sigma = 2, jittered): errors per node (inverse: ||fcheck - fhat||, "
              "adjoint: ||ftilde - f||; the Dirichlet D zeroes k = -M/2, reading A21, so fcheck_{-M/2} = 0 "
              "bounds the inverse error by |fhat_{-M/2}|); (a) N = 4M, m = 4",
              [(4 << c, 1 << c, 4) for c in n1], "alg2")
    err_table("## E6  Alg. 2: (b) N = 2048, M = 512, m = 4..12", [(2048, 512, m) for m in range(4, 13)], "alg2")
    e7(range(1, 9 if q else 15))


if __name__ == "__main__":
    main()

"""GPU: seeded random problems at sizes where the hot-path kernels run with many chunks and
tiles (M up to 2^17, ring kernels m in {4, 8, 16}, fused four-step FFT passes, multiple row
groups, CUDA-graph replay), element-wise against the oracle's C apply."""
import os

import numpy as np
import pytest

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def P():
    import paper_1811_05335_b200 as P
    return P


def _case(seed):
    rng = np.random.default_rng(7000 + seed)
    M = int(rng.choice([1 << 14, 1 << 15, 1 << 16, 1 << 17]))
    m = int(rng.choice([4, 8, 16]))
    N = int(M * rng.choice([1.0, 2.0, 1.5]))
    N -= N % 2
    kind = rng.choice(["jittered", "cluster", "cheb", "cells", "dense"])
    if kind == "jittered":
        x = S.jittered(N, seed)
    elif kind == "cheb":
        x = S.chebyshev(N)
    elif kind == "cells":  # several nodes per grid cell (repeated slot bases), whole circle
        Ms = 2 * M
        x = np.sort((np.floor(rng.random(N) * Ms) + rng.random(N) * 0.3) / Ms - 0.5)
    elif kind == "dense":  # 4 N nodes: every segment far above the chunk target
        N *= 4
        x = np.sort(rng.random(N) - 0.5)
    else:
        x = np.sort(np.clip(np.concatenate([rng.normal(0.1, 0.02, N // 2), rng.random(N - N // 2) - 0.5]),
                            -0.5, 0.5 - 1e-12))
    R = int(rng.choice([17, 40, 64]))
    prec = "c64" if rng.random() < 0.3 else "c128"
    return M, m, x, R, prec, kind


# INFT_RANDOM_LARGE=n widens the sweep
@pytest.mark.parametrize("seed", range(int(os.environ.get("INFT_RANDOM_LARGE", "24"))))
def test_random_large(P, torch, seed):
    M, m, x, R, prec, kind = _case(seed)
    sigma = 2.0
    live = O.slot_live(x, O.msigma(M, sigma), m)
    w = np.random.default_rng(seed).standard_normal(live.shape) * live
    plan = P.Plan(x, M, sigma, m, precision=prec).set_bopt(w, "alg2")
    info = plan.info()
    # complex64 with m = 4 has no ring kernel (a 16-node batch is one 8-byte box): register kernels
    assert info["fast_path"] == (1 if (prec == "c64" and m == 4) else 2) and info["fused_fft"] == 1, (info, M, m, prec)
    dt = torch.complex128 if prec == "c128" else torch.complex64
    f = torch.from_numpy(S.normal_complex(R, x.size, seed)).to("cuda", dt)
    h = torch.from_numpy(S.normal_complex(R, M, seed + 1)).to("cuda", dt)
    c = lambda t: t.cpu().numpy().astype(np.complex128)  # noqa: E731
    ref_i = O.apply_inverse(x, M, sigma, m, w, 1.0, c(f))
    ref_a = O.apply_adjoint(x, M, sigma, m, w, 1.0, c(h))
    tol = 1e-12 if prec == "c128" else 1e-5
    oi = torch.empty(R, M, dtype=dt, device="cuda")
    oa = torch.empty(R, x.size, dtype=dt, device="cuda")
    for _ in range(3):  # plain, capture, replay
        plan.apply(f, out=oi)
        plan.adjoint_apply(h, out=oa)
        assert O.rel_l2(c(oi), ref_i) <= tol, (seed, M, m, kind, R, prec)
        assert O.rel_l2(c(oa), ref_a) <= tol, (seed, M, m, kind, R, prec)


@pytest.mark.parametrize("seed", range(max(4, int(os.environ.get("INFT_RANDOM_LARGE", "24")) // 6)))
def test_random_large_2d(P, torch, seed):
    """2-D tile kernels (heavy tiles split, partial sums combined) at larger sizes."""
    rng = np.random.default_rng(8000 + seed)
    M = (int(rng.choice([64, 128, 256])), int(rng.choice([64, 128, 256])))
    m = int(rng.integers(2, 7))
    N = int(rng.choice([1 << 15, 1 << 16, 1 << 17]))
    if seed % 2:
        x = np.clip(rng.normal(0.0, 0.08, (N, 2)), -0.5, 0.5 - 1e-12)
    else:
        x = rng.random((N, 2)) - 0.5
    l1 = O.slot_live(x[:, 0], O.msigma(M[0], 2.0), m)
    l2 = O.slot_live(x[:, 1], O.msigma(M[1], 2.0), m)
    live = (l1[:, :, None] & l2[:, None, :]).reshape(N, -1)
    w = rng.standard_normal(live.shape) * live
    prec = "c64" if seed == 3 else "c128"
    plan = P.Plan(x, M, 2.0, m, precision=prec).set_bopt(w, "alg2")
    dt = torch.complex128 if prec == "c128" else torch.complex64
    R = int(rng.choice([17, 64]))
    f = torch.from_numpy(S.normal_complex(R, N, seed)).to("cuda", dt)
    h = torch.from_numpy(S.normal_complex(R, M[0] * M[1], seed + 1)).to("cuda", dt)
    c = lambda t: t.cpu().numpy().astype(np.complex128)  # noqa: E731
    tol = 1e-12 if prec == "c128" else 1e-5
    assert O.rel_l2(c(plan.apply(f)), O.apply_inverse(x, M, 2.0, m, w, 1.0, c(f))) <= tol, (seed, M, m, N)
    assert O.rel_l2(c(plan.adjoint_apply(h)), O.apply_adjoint(x, M, 2.0, m, w, 1.0, c(h))) <= tol, (seed, M, m, N)

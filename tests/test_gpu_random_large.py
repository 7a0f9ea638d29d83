"""GPU: seeded random problems at sizes where the hot-path kernels run with many chunks and
tiles (M up to 2^17, ring kernels m in {4, 8, 16}, fused four-step FFT passes, multiple row
groups, CUDA-graph replay), element-wise against the oracle's C apply."""
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
    kind = rng.choice(["jittered", "cluster", "cheb"])
    if kind == "jittered":
        x = S.jittered(N, seed)
    elif kind == "cheb":
        x = S.chebyshev(N)
    else:
        x = np.sort(np.clip(np.concatenate([rng.normal(0.1, 0.02, N // 2), rng.random(N - N // 2) - 0.5]),
                            -0.5, 0.5 - 1e-12))
    R = int(rng.choice([17, 40, 64]))
    prec = "c64" if rng.random() < 0.3 else "c128"
    return M, m, x, R, prec, kind


@pytest.mark.parametrize("seed", range(12))
def test_random_large(P, torch, seed):
    M, m, x, R, prec, kind = _case(seed)
    sigma = 2.0
    live = O.slot_live(x, O.msigma(M, sigma), m)
    w = np.random.default_rng(seed).standard_normal(live.shape) * live
    plan = P.Plan(x, M, sigma, m, precision=prec).set_bopt(w, "alg2")
    info = plan.info()
    assert info["fast_path"] == 2 and info["fused_fft"] == 1, (info, M, m, prec)
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

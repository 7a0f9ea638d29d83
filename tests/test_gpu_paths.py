"""GPU: every apply path against the oracle on sizes that exercise it -- non-power-of-two
grids (cuFFT path), sigma != 2, odd and even m (ring kernels for m in {4, 8, 16}, register
kernels otherwise), 1-D and 2-D, both precisions, ragged batches crossing the 32-RHS lanes."""
import numpy as np
import pytest

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu

# (M, sigma, m, N, nodes)
CASES_1D = [
    (300, 2.0, 5, 700, "jittered"),      # M_sigma = 600: cuFFT path, register kernels
    (1024, 1.25, 4, 1500, "iid"),        # M_sigma = 1280, sigma = 1.25
    (2048, 2.0, 8, 4096, "jittered"),    # ring kernels, fused FFT
    (4096, 2.0, 16, 8192, "jittered"),   # ring kernels m = 16
    (2048, 3.0, 3, 3000, "chebyshev"),   # M_sigma = 6144 (not a power of two), odd m
    (512, 2.0, 7, 900, "iid"),           # m = 7
]
CASES_2D = [((32, 48), 2.0, 3, 2000), ((64, 64), 1.5, 5, 3000), ((48, 32), 2.0, 7, 1500)]


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def P():
    import paper_1811_05335_b200 as P
    return P


def _nodes(kind, N, seed):
    if kind == "jittered":
        return S.jittered(N, seed)
    if kind == "chebyshev":
        return S.chebyshev(N)
    return S.iid_sorted(N, seed)


def _check(P, torch, x, M, sigma, m, live, prec, R):
    rng = np.random.default_rng(R)
    w = rng.standard_normal(live.shape) * live
    plan = P.Plan(x, M, sigma, m, precision=prec).set_bopt(w, "alg2")
    dt = torch.complex128 if prec == "c128" else torch.complex64
    g = torch.Generator(device="cuda").manual_seed(R)
    f = torch.randn(R, x.shape[0], dtype=dt, device="cuda", generator=g)
    h = torch.randn(R, int(np.prod(M)), dtype=dt, device="cuda", generator=g)
    tol = 1e-12 if prec == "c128" else 1e-5
    c = lambda t: t.cpu().numpy().astype(np.complex128)  # noqa: E731
    assert O.rel_l2(c(plan.apply(f)), O.apply_inverse(x, M, sigma, m, w, 1.0, c(f))) <= tol
    assert O.rel_l2(c(plan.adjoint_apply(h)), O.apply_adjoint(x, M, sigma, m, w, 1.0, c(h))) <= tol
    return plan.info()


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("case", CASES_1D, ids=[f"M{c[0]}s{c[1]:g}m{c[2]}" for c in CASES_1D])
def test_paths_1d(P, torch, case, prec):
    M, sigma, m, N, kind = case
    x = _nodes(kind, N, M + m)
    live = O.slot_live(x, O.msigma(M, sigma), m)
    for R in (1, 37):
        info = _check(P, torch, x, M, sigma, m, live, prec, R)
    Ms = O.msigma(M, sigma)
    assert info["fused_fft"] == (1 if (Ms & (Ms - 1)) == 0 and Ms >= 256 else 0) or prec == "c64"


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("case", CASES_2D, ids=[f"M{c[0][0]}x{c[0][1]}m{c[2]}" for c in CASES_2D])
def test_paths_2d(P, torch, case, prec):
    M, sigma, m, N = case
    rng = np.random.default_rng(m)
    x = rng.random((N, 2)) - 0.5
    l1 = O.slot_live(x[:, 0], O.msigma(M[0], sigma), m)
    l2 = O.slot_live(x[:, 1], O.msigma(M[1], sigma), m)
    live = (l1[:, :, None] & l2[:, None, :]).reshape(N, -1)
    for R in (1, 37):
        _check(P, torch, x, M, sigma, m, live, prec, R)

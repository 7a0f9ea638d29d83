"""GPU: the fused four-step FFT passes (a3+a4, a5+a6 in fft.cu) against the
unfused path (cuFFT + separate truncation/deconvolution and padding kernels,
selected with INFT_NO_FUSED_FFT=1 at plan creation) and against the oracle, over
grid lengths M_sigma = 2^9 .. 2^20 (square and non-square N1 x N2 splits,
sigma = 2 and 4), both precisions, a ragged batch of right-hand sides."""
import os

import numpy as np
import pytest

import oracle as O
import synth.nodes as SN

pytestmark = pytest.mark.gpu

# (M, sigma, m, N): M_sigma = sigma M is a power of two
CASES = [(256, 2.0, 4, 300), (1024, 2.0, 6, 2000), (4096, 4.0, 5, 5000), (1 << 14, 2.0, 8, 20000),
         (1 << 15, 2.0, 7, 40000), (1 << 17, 2.0, 8, 100000), (1 << 19, 2.0, 6, 300000)]
R = 3


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def P():
    import paper_1811_05335_b200 as P
    return P


def _plan(P, x, M, sigma, m, w, prec, fused):
    old = os.environ.get("INFT_NO_FUSED_FFT")
    os.environ["INFT_NO_FUSED_FFT"] = "0" if fused else "1"
    try:
        plan = P.Plan(x, M, sigma, m, precision=prec).set_bopt(w, "alg2")
    finally:
        if old is None:
            del os.environ["INFT_NO_FUSED_FFT"]
        else:
            os.environ["INFT_NO_FUSED_FFT"] = old
    return plan


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("case", CASES, ids=[f"M{c[0]}s{c[1]:g}" for c in CASES])
def test_fused_fft_matches_unfused_and_oracle(P, torch, case, prec):
    M, sigma, m, N = case
    x = SN.jittered(N, seed=M + N)
    Ms = O.msigma(M, sigma)
    rng = np.random.default_rng(M)
    w = rng.standard_normal((N, 2 * m + 1)) * O.slot_live(x, Ms, m)
    pf = _plan(P, x, M, sigma, m, w, prec, True)
    pu = _plan(P, x, M, sigma, m, w, prec, False)
    assert pf.info()["fused_fft"] == 1, "fused FFT path not selected"
    assert pu.info()["fused_fft"] == 0
    dt = torch.complex128 if prec == "c128" else torch.complex64
    g = torch.Generator(device="cuda").manual_seed(M)
    f = torch.randn(R, N, dtype=dt, device="cuda", generator=g)
    h = torch.randn(R, M, dtype=dt, device="cuda", generator=g)
    a_f, a_u = pf.apply(f), pu.apply(f)
    b_f, b_u = pf.adjoint_apply(h), pu.adjoint_apply(h)
    tol = 1e-13 if prec == "c128" else 2e-6
    c = lambda t: t.cpu().numpy().astype(np.complex128)  # noqa: E731
    assert O.rel_l2(c(a_f), c(a_u)) <= tol
    assert O.rel_l2(c(b_f), c(b_u)) <= tol
    if Ms <= (1 << 16):  # the oracle finishes these in well under a second per RHS
        tol_o = 1e-12 if prec == "c128" else 1e-5
        r = R - 1
        assert O.rel_l2(c(a_f[r:r + 1]), O.apply_inverse(x, M, sigma, m, w, 1.0, c(f[r:r + 1]))) <= tol_o
        assert O.rel_l2(c(b_f[r:r + 1]), O.apply_adjoint(x, M, sigma, m, w, 1.0, c(h[r:r + 1]))) <= tol_o

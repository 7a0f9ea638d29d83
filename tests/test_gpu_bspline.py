"""GPU: the B-spline window (INFT_BSPLINE, reading A24; the window of the paper's experiments,
P:987) against the oracle -- deconvolution table, plain window
weights (ordinary NFFT), GPU Alg. 2 / Alg. 1 setups reaching the oracle's per-column /
per-node optimum, and the apply with a shared B_opt."""
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


@pytest.mark.parametrize("M,sigma,m", [(256, 2.0, 4), (1024, 1.0, 2), (48, 1.5, 3), (128, 2.0, 12)])
def test_bspline_deconv_and_plain_weights(P, M, sigma, m):
    x = S.jittered(200, m)
    plan = P.Plan(x, M, sigma, m, window="bspline").precompute("plain")
    ref = O.deconv_vector(M, sigma, m, 1.0, window="bspline")
    assert np.abs(plan.get_deconv() / ref - 1).max() < 1e-13
    w = plan.get_bopt()
    wo = O.window_slot_weights(x, M, sigma, m, window="bspline")
    assert np.abs(w - wo).max() <= 1e-13 * np.abs(wo).max()


def test_bspline_plain_nfft_matches_ndft(P, torch):
    """The GPU ordinary NFFT with the B-spline window (adjoint apply = B F D, s = 1) against
    the NDFT: error at the window's level, falling in m."""
    M, sigma, N = 512, 2.0, 700
    x = S.jittered(N, 5)
    fh = S.normal_complex(3, M, 6)
    ref = O.ndft(x, fh, M)
    errs = []
    for m in (2, 4, 8):
        plan = P.Plan(x, M, sigma, m, window="bspline").precompute("plain")
        got = plan.adjoint_apply(torch.from_numpy(fh).cuda()).cpu().numpy()
        errs.append(O.rel_l2(got, ref))
    assert errs[0] > 10 * errs[1] > 100 * errs[2], errs
    assert errs[2] < 1e-6, errs


def test_bspline_alg2_gpu_setup(P, torch):
    M, sigma, m, N = 64, 2.0, 2, 200
    x = S.jittered(N, 7)
    plan = P.Plan(x, M, sigma, m, window="bspline").precompute("alg2")
    wg = plan.get_bopt()
    wo, _ = O.alg2_setup(x, M, sigma, m, form="gram", window="bspline")
    og = O.objective_alg2(x, M, sigma, m, wg, window="bspline")
    oo = O.objective_alg2(x, M, sigma, m, wo, window="bspline")
    assert og <= oo * (1 + 1e-9) + 1e-9
    ow = O.objective_alg2(x, M, sigma, m, O.window_slot_weights(x, M, sigma, m, window="bspline"), window="bspline")
    assert og < ow  # the optimisation improves on the window matrix
    f = torch.from_numpy(S.normal_complex(2, N, 8)).cuda()
    assert O.rel_l2(plan.apply(f).cpu().numpy(),
                    O.apply_inverse(x, M, sigma, m, wg, 1.0, f.cpu().numpy(), window="bspline")) <= 1e-12


@pytest.mark.parametrize("mode", ["dense", "gram"])
def test_bspline_alg1_gpu_setup(P, mode):
    import os
    M, sigma, m, N = 512, 1.0, 2, 128
    x = S.jittered(N, 9)
    old = os.environ.get("INFT_ALG1")
    os.environ["INFT_ALG1"] = mode
    try:
        plan = P.Plan(x, M, sigma, m, window="bspline").precompute("alg1")
    finally:
        if old is None:
            del os.environ["INFT_ALG1"]
        else:
            os.environ["INFT_ALG1"] = old
    wg = plan.get_bopt()
    wo, _ = O.alg1_setup(x, M, sigma, m, window="bspline")
    K = O.K_kernel_matrix(x, M, sigma, m, window="bspline")
    Ms = O.msigma(M, sigma)
    l0 = O.node_base(x, Ms, m)
    for j in range(N):
        cols = np.mod(l0[j] + np.arange(2 * m + 1) + Ms // 2, Ms)
        e = np.zeros(N)
        e[j] = M
        assert np.linalg.norm(K[:, cols] @ wg[j] - e) <= np.linalg.norm(K[:, cols] @ wo[j] - e) * (1 + 1e-6) + 1e-9 * M


def test_bspline_window_limits(P):
    with pytest.raises(P.InftError):
        P.Plan(S.jittered(64, 1), 64, 2.0, 17, window="bspline")  # order 2m > 32

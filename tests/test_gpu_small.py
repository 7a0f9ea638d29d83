"""GPU: the single-launch path for small 1-D problems (one CTA per RHS: spread, radix-2 FFT in
shared memory and deconvolution in one kernel; configs 1-2 are launch-latency bound) against
the oracle and against the multi-kernel pipeline on the same plans' weights: real and complex
weights, both precisions, aliasing (2m+1 > M_sigma), configs 1 and 2."""
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


def _plan(P, small, *a, **k):
    old = os.environ.get("INFT_NO_SMALL")
    os.environ["INFT_NO_SMALL"] = "0" if small else "1"
    try:
        return P.Plan(*a, **k)
    finally:
        if old is None:
            del os.environ["INFT_NO_SMALL"]
        else:
            os.environ["INFT_NO_SMALL"] = old


CASES = [  # M, sigma, m, N, nodes, R, complex weights
    (256, 2.0, 4, 512, "jittered", 1, False),     # config 1 shape
    (1024, 2.0, 6, 512, "iid", 4, False),         # config 2 shape (R M_sigma <= 8192)
    (64, 2.0, 5, 100, "iid", 7, True),
    (16, 1.0, 8, 20, "jittered", 3, False),       # 2m+1 > M_sigma: aliased slots
    (512, 4.0, 3, 900, "jittered", 2, True),
]


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("case", CASES, ids=[f"M{c[0]}s{c[1]:g}m{c[2]}R{c[5]}" for c in CASES])
def test_small_path_parity(P, torch, case, prec):
    M, sigma, m, N, kind, R, cplx = case
    x = S.jittered(N, M) if kind == "jittered" else S.iid_sorted(N, M)
    live = O.slot_live(x, O.msigma(M, sigma), m)
    rng = np.random.default_rng(M + m)
    w = rng.standard_normal(live.shape) * live
    if cplx:
        w = w + 1j * rng.standard_normal(live.shape) * live
    ps = _plan(P, True, x, M, sigma, m, precision=prec).set_bopt(w, "alg2")
    pr = _plan(P, False, x, M, sigma, m, precision=prec).set_bopt(w, "alg2")
    dt = torch.complex128 if prec == "c128" else torch.complex64
    f = torch.from_numpy(S.normal_complex(R, N, 1)).to("cuda", dt)
    h = torch.from_numpy(S.normal_complex(R, M, 2)).to("cuda", dt)
    tol = 1e-12 if prec == "c128" else 1e-5
    c = lambda t: t.cpu().numpy().astype(np.complex128)  # noqa: E731
    n0 = ps.kernel_launches()
    for _ in range(3):  # plain, graph capture, replay
        gi, ga = ps.apply(f), ps.adjoint_apply(h)
        assert O.rel_l2(c(gi), O.apply_inverse(x, M, sigma, m, w, 1.0, c(f))) <= tol
        assert O.rel_l2(c(ga), O.apply_adjoint(x, M, sigma, m, w, 1.0, c(h))) <= tol
        assert O.rel_l2(c(gi), c(pr.apply(f))) <= tol and O.rel_l2(c(ga), c(pr.adjoint_apply(h))) <= tol
    assert ps.kernel_launches() - n0 == 6  # one launch per direction and call


def test_small_path_configs_setup(P, torch):
    """Configs 1 (Alg. 2) and 2 (Alg. 1) end to end with GPU-optimised B_opt on the small path."""
    for cid, method in ((1, "alg2"), (2, "alg1")):
        cfg = S.config(cid)
        x = S.make_nodes(cfg)
        M, sigma, m = cfg["M"][0], cfg["sigma"], cfg["m"]
        ps = _plan(P, True, x, M, sigma, m).precompute(method)
        pr = _plan(P, False, x, M, sigma, m).precompute(method)
        R = min(cfg["R"], 4)  # the small path takes R M_sigma <= 8192
        f = torch.from_numpy(S.normal_complex(R, x.size, 3)).cuda()
        h = torch.from_numpy(S.normal_complex(R, M, 4)).cuda()
        assert O.rel_l2(ps.apply(f).cpu().numpy(), pr.apply(f).cpu().numpy()) <= 1e-12
        assert O.rel_l2(ps.adjoint_apply(h).cpu().numpy(), pr.adjoint_apply(h).cpu().numpy()) <= 1e-12

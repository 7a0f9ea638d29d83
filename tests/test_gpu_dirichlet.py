"""GPU: the Dirichlet-kernel variant (Remarks P:934-957, P:1343-1358,
reading A21) against the oracle -- deconvolution table, GPU Alg. 2 / Alg. 1 setups and the
apply with a shared B_opt."""
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


def _cfg(i):
    c = S.config(i)
    x = S.make_nodes(c)
    M = c["M"][0] if c["d"] == 1 else c["M"]
    return c, x, M, c["sigma"], c["m"]


def test_dirichlet_deconv_table(P):
    for M, sigma, m in [(256, 2.0, 4), (1024, 2.0, 6), (24, 1.5, 3)]:
        x = S.jittered(64, 1)
        plan = P.Plan(x, M, sigma, m, window="dirichlet")
        np.testing.assert_array_equal(plan.get_deconv(), O.deconv_vector(M, sigma, m, 1.0, window="dirichlet"))


def test_dirichlet_plain_nfft_rejected(P):
    plan = P.Plan(S.jittered(64, 1), 32, 2.0, 4, window="dirichlet")
    with pytest.raises(P.InftError):
        plan.precompute("plain")


def test_dirichlet_alg2_gpu_setup_cfg1(P, torch):
    c, x, M, sigma, m = _cfg(1)
    plan = P.Plan(x, M, sigma, m, window="dirichlet").precompute("alg2")
    wg = plan.get_bopt()
    wo, info_o = O.alg2_setup(x, M, sigma, m, form="gram", window="dirichlet")
    og = O.objective_alg2(x, M, sigma, m, wg, window="dirichlet")
    oo = O.objective_alg2(x, M, sigma, m, wo, window="dirichlet")
    assert og <= oo * (1 + 1e-9) + 1e-9
    fh = S.make_rhs(c)
    f = O.ndft(x, fh, M)
    got = plan.apply(torch.from_numpy(np.ascontiguousarray(f)).cuda()).cpu().numpy()
    assert O.rel_l2(got, O.apply_inverse(x, M, sigma, m, wg, 1.0, f, window="dirichlet")) <= 1e-12
    assert O.rel_l2(got, O.apply_inverse(x, M, sigma, m, wo, 1.0, f, window="dirichlet")) < 1e-8


def test_dirichlet_alg1_gpu_setup_cfg2(P, torch):
    c, x, M, sigma, m = _cfg(2)
    plan = P.Plan(x, M, sigma, m, window="dirichlet").precompute("alg1")
    wg = plan.get_bopt()
    wo, _ = O.alg1_setup(x, M, sigma, m, window="dirichlet")
    f = S.make_rhs(c, kind="adjoint")
    h = O.ndft_adjoint(x, f, M)
    got = plan.adjoint_apply(torch.from_numpy(np.ascontiguousarray(h)).cuda()).cpu().numpy()
    ref = O.apply_adjoint(x, M, sigma, m, wg, 1.0 / M, h, window="dirichlet")
    # this B_opt is ill-conditioned (|w| up to ~10^3): measure the error against the scale of
    # the summands, |B| |F D h| / M, so that cancellation in the gather is not charged to the
    # kernels (the bar stays 1e-12)
    Ms = O.msigma(M, sigma)
    Bd = O.dense_from_slots(np.abs(wg), O.node_base(x, Ms, m), Ms)
    g = (O.matrix_F(M, Ms) @ np.diag(O.deconv_vector(M, sigma, m, 1.0, window="dirichlet")) @ h.T)
    scale = np.abs(Bd) @ np.abs(g) / M
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(scale).max()
    # per-node objective ||K_j b - M e_j|| reaches the oracle's minimum
    K = O.K_kernel_matrix(x, M, sigma, m, window="dirichlet")
    Ms = O.msigma(M, sigma)
    l0 = O.node_base(x, Ms, m)
    for j in range(0, x.size, 37):
        cols = np.mod(l0[j] + np.arange(2 * m + 1) + Ms // 2, Ms)
        e = np.zeros(x.size)
        e[j] = M
        assert np.linalg.norm(K[:, cols] @ wg[j] - e) <= np.linalg.norm(K[:, cols] @ wo[j] - e) * (1 + 1e-6) + 1e-9 * M


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_dirichlet_apply_parity_shared_bopt(P, torch, prec):
    """Config 3 nodes (1-D fast path) and config 4 nodes (2-D tile kernels) with a shared
    random live B_opt: the only change from the KB apply is d."""
    for cid in (3, 4):
        c, x, M, sigma, m = _cfg(cid)
        rng = np.random.default_rng(cid)
        if c["d"] == 1:
            live = O.slot_live(x, O.msigma(M, sigma), m)
        else:
            l1 = O.slot_live(x[:, 0], O.msigma(M[0], sigma), m)
            l2 = O.slot_live(x[:, 1], O.msigma(M[1], sigma), m)
            live = (l1[:, :, None] & l2[:, None, :]).reshape(x.shape[0], -1)
        w = rng.standard_normal(live.shape) * live
        plan = P.Plan(x, M, sigma, m, precision=prec, window="dirichlet").set_bopt(w, "alg2")
        dt = torch.complex128 if prec == "c128" else torch.complex64
        R = 3
        f = torch.randn(R, x.shape[0], dtype=dt, device="cuda")
        h = torch.randn(R, int(np.prod(M)), dtype=dt, device="cuda")
        tol = 1e-12 if prec == "c128" else 1e-5
        c128 = lambda t: t.cpu().numpy().astype(np.complex128)  # noqa: E731
        assert O.rel_l2(c128(plan.apply(f)), O.apply_inverse(x, M, sigma, m, w, 1.0, c128(f), window="dirichlet")) <= tol
        assert O.rel_l2(c128(plan.adjoint_apply(h)),
                        O.apply_adjoint(x, M, sigma, m, w, 1.0, c128(h), window="dirichlet")) <= tol

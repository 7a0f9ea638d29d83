"""GPU: Alg. 1 (node-wise) with the Gram matrices assembled by grid pairs
(DESIGN.md "Alg. 1 at scale"): every node's normal equations from one
node sum Sp(q), 2m+1 correlations and 2m+1 FFTs of length M_sigma instead of the dense
K = A D^* F^*.  Each solution is checked against the oracle's minimum of ||K_j b - M e_j||
(eq. opt_ansatz1) on the node's live slots, with K_j formed by the oracle from its
own kernel (direct sums for Kaiser-Bessel, the closed form D_{M/2-1}/M_sigma for Dirichlet)."""
import os
import time

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


def _precompute(P, x, M, sigma, m, window, mode):
    old = os.environ.get("INFT_ALG1")
    os.environ["INFT_ALG1"] = mode
    try:
        plan = P.Plan(x, M, sigma, m, window=window)
        t0 = time.perf_counter()
        plan.precompute("alg1")
        return plan, time.perf_counter() - t0
    finally:
        if old is None:
            del os.environ["INFT_ALG1"]
        else:
            os.environ["INFT_ALG1"] = old


def _kernel(dx, M, sigma, m, window):
    if window == "dirichlet":
        return O.dirichlet_kernel(dx, M) / O.msigma(M, sigma)
    return O.Kplus_kernel(dx, M, sigma, m, window)


def _node_residuals(x, M, sigma, m, w, nodes, window):
    """(GPU residual, oracle minimum) of ||K_j b - M e_j|| for the sampled nodes."""
    Ms = O.msigma(M, sigma)
    l0 = O.node_base(x, Ms, m)
    live = O.slot_live(x, Ms, m)
    out = []
    for j in nodes:
        ts = np.nonzero(live[j])[0]
        Kj = _kernel(O.wrap_diff(x[:, None] - (l0[j] + ts)[None, :] / Ms), M, sigma, m, window)
        e = np.zeros(x.size, dtype=np.complex128)
        e[j] = M
        bo, _ = O.lstsq_minnorm_svd(Kj, e, O.TAU_DEFAULT, real=True)
        out.append((np.linalg.norm(Kj @ w[j, ts] - e), np.linalg.norm(Kj @ bo - e)))
    return out


def test_alg1_gram_equals_dense_cfg2(P):
    """Config 2 (the Alg. 1 configuration): both assemblies reach the same per-node optimum."""
    c = S.config(2)
    x = S.make_nodes(c)
    M, sigma, m = c["M"][0], c["sigma"], c["m"]
    pd, _ = _precompute(P, x, M, sigma, m, "kb", "dense")
    pg, _ = _precompute(P, x, M, sigma, m, "kb", "gram")
    wd, wg = pd.get_bopt(), pg.get_bopt()
    K = O.K_kernel_matrix(x, M, sigma, m)
    Ms = O.msigma(M, sigma)
    l0 = O.node_base(x, Ms, m)
    for j in range(x.size):
        cols = np.mod(l0[j] + np.arange(2 * m + 1) + Ms // 2, Ms)
        e = np.zeros(x.size)
        e[j] = M
        rd = np.linalg.norm(K[:, cols] @ wd[j] - e)
        rg = np.linalg.norm(K[:, cols] @ wg[j] - e)
        assert rg <= rd * (1 + 1e-6) + 1e-9 * M, (j, rg, rd)
    # both recover f from h = A^* f equally well (the weights themselves agree only to the
    # conditioning of these rank-deficient systems, ~1e-8 here)
    f = S.normal_complex(2, x.size, 4)
    h = np.ascontiguousarray(O.ndft_adjoint(x, f, M))
    eg = O.rel_l2(pg.adjoint_apply(h).cpu().numpy(), f)
    ed = O.rel_l2(pd.adjoint_apply(h).cpu().numpy(), f)
    assert eg <= ed * 1.01 + 1e-12, (eg, ed)
    assert pg.info()["n_rank_deficient"] == pd.info()["n_rank_deficient"]


@pytest.mark.parametrize("window", ["kb", "dirichlet"])
@pytest.mark.parametrize("N,M,sigma,m", [(2048, 4096, 2.0, 6), (4096, 2048, 2.0, 8), (3000, 2000, 1.5, 5)])
def test_alg1_gram_sampled_nodes(P, window, N, M, sigma, m):
    """Under- and overdetermined, sigma = 1.5 (frequencies fold onto the M_sigma grid): sampled
    nodes reach the oracle's per-node minimum."""
    x = S.jittered(N, 11)
    plan, _ = _precompute(P, x, M, sigma, m, window, "gram")
    w = plan.get_bopt()
    assert np.all(np.isfinite(w))
    nodes = np.random.default_rng(1).choice(N, 12, replace=False)
    for rg, ro in _node_residuals(x, M, sigma, m, w, nodes, window):
        assert rg <= ro * (1 + 1e-6) + 1e-9 * M, (rg, ro)


def test_alg1_gram_beyond_dense_limit(P):
    """N M_sigma = 2^36, far past the dense form's 2^28 limit (which refuses): Dirichlet
    window (closed-form K_j for the oracle), iid nodes, M = 2N (underdetermined, the case
    Alg. 1 is for)."""
    N, M, sigma, m = 1 << 17, 1 << 18, 2.0, 4
    x = np.sort(np.random.default_rng(7).random(N) - 0.5)
    with pytest.raises(P.InftError):
        _precompute(P, x, M, sigma, m, "dirichlet", "dense")
    plan, dt = _precompute(P, x, M, sigma, m, "dirichlet", "auto")
    print(f"Alg. 1 (Gram by grid pairs) N = 2^17, M = 2^18, m = 4: {dt:.2f} s")
    w = plan.get_bopt()
    assert np.all(np.isfinite(w))
    nodes = np.random.default_rng(2).choice(N, 6, replace=False)
    for rg, ro in _node_residuals(x, M, sigma, m, w, nodes, "dirichlet"):
        assert rg <= ro * (1 + 1e-6) + 1e-9 * M, (rg, ro)

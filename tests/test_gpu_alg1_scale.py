"""NEXT-2 at the scale it targets: GPU Alg. 1 (Alg. "Fast optimization of the matrix B*",
P:895-931, the node-wise setup meant for M > N) at N = 2^20 nodes, M = 2^21, m = 8,
sigma = 2, with every node's Gram matrix assembled from the grid-pair table (DESIGN.md "Alg. 1 at
scale").

* Dirichlet window (reading A21): K(x) = D_{M/2-1}(x)/M_sigma has a closed form, so the oracle
  forms K_j = (K(x_h - l/M_sigma))_{h, l in I(x_j)} over ALL 2^20 nodes h for 64 sampled nodes j
  and minimises ||K_j b - M e_j|| (eq. opt_ansatz1) by its SVD solver; the GPU's column
  must reach that minimum.
* Kaiser-Bessel: K_j would cost 2^21 terms per entry, so the check is the method's purpose
  instead: h = A^* f for random f (the oracle's plain adjoint NFFT with a wide window, spot-checked
  against the direct sum), then the inverse adjoint NFFT f~ = (1/M) B_opt F D h on the GPU
   must recover f as well as the same construction does at N = 2^12, where the GPU's
  Alg. 1 is compared column by column with the oracle's dense Alg. 1."""
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


def test_alg1_dirichlet_full_scale_node_optimum(P):
    N, M, m, sigma = 1 << 20, 1 << 21, 8, 2.0
    x = S.jittered(N, 4)
    plan = P.Plan(x, M, sigma, m, window="dirichlet").precompute("alg1")
    w = plan.get_bopt()
    assert np.all(np.isfinite(w))
    Ms = O.msigma(M, sigma)
    l0 = O.node_base(x, Ms, m)
    live = O.slot_live(x, Ms, m)
    rng = np.random.default_rng(20)
    nodes = [0, 1, N // 2, N - 1] + sorted(rng.choice(N, 60, replace=False).tolist())
    worst = 0.0
    rows = []
    for j in nodes:
        ts = np.nonzero(live[j])[0]
        ls = l0[j] + ts  # grid indices (any representative mod M_sigma: K is 1-periodic)
        Kj = O.dirichlet_kernel(O.wrap_diff(x[:, None] - ls[None, :] / Ms), M) / Ms
        e = np.zeros(N, dtype=np.complex128)
        e[j] = M
        bo, _ = O.lstsq_minnorm_svd(Kj, e)
        ro = np.linalg.norm(Kj @ bo - e)
        rg = np.linalg.norm(Kj @ np.conj(w[j, ts]) - e)  # stored conjugated (reading A4); real here
        # the same minimisation in the Gram form (reading A6) done by the oracle: normal equations
        # from the explicit K_j, eigh + cutoff -- the precision floor of that form at this size
        bgr, _ = O.solve_minnorm_gram(np.real(Kj.conj().T @ Kj), np.real(Kj.conj().T @ e))
        rgr = np.linalg.norm(Kj @ bgr - e)
        # objective excess over the SVD optimum, normalised by ||M e_j||^2.  The GPU's Gram
        # matrices come from the grid-pair table, whose length-2^21/2^22 FFT sums carry rounding of
        # ~1e-15 of their largest entries; in the normal equations that is an objective excess of
        # ~1e-12, against the oracle's explicit-K_j Gram form at
        # ~1e-17.  Bar: 3e-11 of ||M e_j||^2 at any node, 2e-12 at the median (the residual
        # itself is ~6e-6 of ||M e_j||; the measured worst was 1.2e-11, i.e. a residual 9 % above
        # the optimum -- recorded in DESIGN.md as the table's precision floor).
        ex_g = (rg * rg - ro * ro) / float(M) ** 2
        worst = max(worst, ex_g)
        rows.append((j, ro, rg, rgr))
        assert ex_g <= 3e-11, (j, ro, rg, rgr)
    med = float(np.median([(r[2] ** 2 - r[1] ** 2) / float(M) ** 2 for r in rows]))
    assert med <= 2e-12, med
    print(f"Dirichlet N=2^20 M=2^21: {len(nodes)} nodes; median / max objective excess over the SVD optimum "
          f"{med:.2e} / "
          f"{worst:.2e} of ||M e_j||^2 (oracle Gram form: {max((r[3]**2 - r[1]**2) / M**2 for r in rows):.2e}); "
          f"sample (j, svd, gpu, gram) {rows[:3]}; rank-deficient {plan.info()['n_rank_deficient']}")


def _recovery(P, torch, N, M, m, sigma, seed, check_oracle=False):
    x = S.jittered(N, seed)
    plan = P.Plan(x, M, sigma, m).precompute("alg1")
    R = 2
    f = S.normal_complex(R, N, seed + 1)
    wB = O.window_slot_weights(x, M, sigma, 16)
    h = O.apply_inverse(x, M, sigma, 16, wB, 1.0, f)  # A^* f (plain adjoint NFFT, m = 16)
    ks = np.random.default_rng(seed).choice(M, 16, replace=False)
    # direct sum h_k = sum_j f_j e^{-2 pi i k x_j} with an exact phase: x = xh + xl, xh with 24
    # significant bits (k xh exact for |k| <= 2^21), k xl small
    xh = x.astype(np.float32).astype(np.float64)
    xl = x - xh

    def phase(k):
        return np.mod(k * xh, 1.0) + k * xl

    ref = np.array([[np.sum(f[r] * np.exp(-2j * np.pi * phase(float(k - M // 2)))) for k in ks]
                    for r in range(R)])
    assert np.abs(h[:, ks] - ref).max() <= 1e-10 * np.abs(ref).max()
    got = plan.adjoint_apply(torch.from_numpy(h).cuda()).cpu().numpy()
    err = O.rel_l2(got, f)
    if check_oracle:  # the small case: GPU weights = the oracle's dense Alg. 1 optimum
        wo, _ = O.alg1_setup(x, M, sigma, m)
        ref_o = O.apply_adjoint(x, M, sigma, m, wo, 1.0 / M, h)
        assert O.rel_l2(ref_o, f) <= 2 * err + 1e-12
    return err, plan.info()


def test_alg1_kb_full_scale_recovery(P, torch):
    sigma, m = 2.0, 8
    e_small, _ = _recovery(P, torch, 1 << 12, 1 << 13, m, sigma, 4, check_oracle=True)
    e_big, info = _recovery(P, torch, 1 << 20, 1 << 21, m, sigma, 4)
    print(f"KB Alg. 1 inverse adjoint recovery: N=2^12 {e_small:.2e}, N=2^20 {e_big:.2e} "
          f"(rank-deficient {info['n_rank_deficient']}, max|w| {info['max_abs_w']:.3g})")
    assert e_big <= max(10 * e_small, 1e-6)

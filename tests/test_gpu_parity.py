"""GPU parity: the CUDA path through the C ABI against the CPU oracle on the
same seeded inputs.  Bar (BASELINE north_star): relative l2 per RHS <= 1e-12
(complex128), <= 1e-5 (complex64); integer bins / permutation bit-exact.
Apply parity uses a SHARED B_opt (imported with inft_set_bopt or exported
with inft_get_bopt) -- reading D6 in DESIGN.md."""
import numpy as np
import pytest

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-12, "c64": 1e-5}


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


def _live_random_weights(x, M, sigma, m, seed):
    rng = np.random.default_rng(seed)
    x = np.asarray(x)
    if x.ndim == 1:
        Ms = O.msigma(M, sigma)
        live = O.slot_live(x, Ms, m)
    else:
        l1 = O.slot_live(x[:, 0], O.msigma(M[0], sigma), m)
        l2 = O.slot_live(x[:, 1], O.msigma(M[1], sigma), m)
        live = (l1[:, :, None] & l2[:, :, None].transpose(0, 2, 1)).reshape(x.shape[0], -1)
    return rng.standard_normal(live.shape) * live


def _dev(torch, a, prec="c128"):
    dt = torch.complex128 if prec == "c128" else torch.complex64
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dt)


# ------------------------------------------------------------------ a0: plan integers
@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_bins_bit_exact(P, cid):
    c, x, M, sigma, m = _cfg(cid)
    plan = P.Plan(x, M, sigma, m)
    l0, b, perm = plan.get_bins()
    info = plan.info()
    if c["d"] == 1:
        Ms = O.msigma(M, sigma)
        l0r, n0r, br, permr = O.bins_1d(x, Ms, m, info["tile"][0])
        np.testing.assert_array_equal(l0, l0r)
    else:
        S1, S2 = info["tile"]
        Ms = [O.msigma(v, sigma) for v in M]
        l0r = np.stack([O.node_base(x[:, 0], Ms[0], m), O.node_base(x[:, 1], Ms[1], m)], axis=1)
        np.testing.assert_array_equal(l0, l0r)
        n0 = np.mod(l0r, Ms)
        nseg2 = -(-Ms[1] // S2)
        br = (n0[:, 0] // S1) * nseg2 + n0[:, 1] // S2
        permr = np.argsort(br, kind="stable")
    np.testing.assert_array_equal(b, br)
    np.testing.assert_array_equal(perm, permr)


def test_deconv_table(P):
    for M, sigma, m in [(256, 2.0, 4), (1024, 2.0, 6), (1 << 20, 2.0, 8), (24, 1.5, 3)]:
        x = S.jittered(8, 0)
        plan = P.Plan(x, M, sigma, m)
        np.testing.assert_allclose(plan.get_deconv(), O.deconv_vector(M, sigma, m, 1.0), rtol=1e-14)


# ------------------------------------------------------------------ apply parity, shared B_opt
def test_cfg1_inverse_parity_oracle_bopt(P, torch):
    c, x, M, sigma, m = _cfg(1)
    w, _ = O.alg2_setup(x, M, sigma, m, form="gram")
    fh = S.make_rhs(c)
    f = O.ndft(x, fh, M)
    plan = P.Plan(x, M, sigma, m).set_bopt(w, "alg2")
    got = plan.apply(_dev(torch, f)).cpu().numpy()
    ref = O.apply_inverse(x, M, sigma, m, w, 1.0, f)
    assert O.rel_l2(got, ref) <= TOL["c128"]
    assert O.rel_l2(got, fh) < 1e-4  # the method recovers fhat (sanity, not parity)


def test_cfg2_adjoint_parity_oracle_bopt(P, torch):
    c, x, M, sigma, m = _cfg(2)
    w, _ = O.alg1_setup(x, M, sigma, m)
    f = S.make_rhs(c, kind="adjoint")
    h = O.ndft_adjoint(x, f, M)
    plan = P.Plan(x, M, sigma, m).set_bopt(w, "alg1")
    assert abs(plan.info()["scale"] - 1.0 / M) < 1e-18
    got = plan.adjoint_apply(_dev(torch, h)).cpu().numpy()
    ref = O.apply_adjoint(x, M, sigma, m, w, 1.0 / M, h)
    assert O.rel_l2(got, ref) <= TOL["c128"]


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_cfg3_inverse_parity_random_bopt(P, torch, prec):
    c, x, M, sigma, m = _cfg(3)
    w = _live_random_weights(x, M, sigma, m, 3)
    R = 40  # ragged vs the 32-RHS warp tiles
    f = S.normal_complex(R, x.size, 7)
    plan = P.Plan(x, M, sigma, m, precision=prec).set_bopt(w, "alg2")
    got = plan.apply(_dev(torch, f, prec)).cpu().numpy().astype(np.complex128)
    ref = O.apply_inverse(x, M, sigma, m, w, 1.0, f)
    assert O.rel_l2(got, ref) <= TOL[prec]
    h = S.normal_complex(R, M, 8)
    got = plan.adjoint_apply(_dev(torch, h, prec)).cpu().numpy().astype(np.complex128)
    ref = O.apply_adjoint(x, M, sigma, m, w, 1.0, h)
    assert O.rel_l2(got, ref) <= TOL[prec]


def test_cfg4_2d_parity_random_bopt(P, torch):
    c, x, M, sigma, m = _cfg(4)
    w = _live_random_weights(x, M, sigma, m, 4)
    R = 3
    f = S.normal_complex(R, x.shape[0], 9)
    plan = P.Plan(x, M, sigma, m).set_bopt(w, "alg2")
    got = plan.apply(_dev(torch, f)).cpu().numpy()
    ref = O.apply_inverse(x, M, sigma, m, w, 1.0, f)
    assert O.rel_l2(got, ref) <= TOL["c128"]
    h = S.normal_complex(R, M[0] * M[1], 10)
    got = plan.adjoint_apply(_dev(torch, h)).cpu().numpy()
    ref = O.apply_adjoint(x, M, sigma, m, w, 1.0, h)
    assert O.rel_l2(got, ref) <= TOL["c128"]


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_cfg5_full_size_sampled_parity(P, torch, prec):
    """Full config-5 size in the bench launch configuration (R = 64 per GPU);
    the oracle recomputes 2 sampled right-hand sides completely."""
    c, x, M, sigma, m = _cfg(5)
    w = _live_random_weights(x, M, sigma, m, 5)
    R = 64
    plan = P.Plan(x, M, sigma, m, precision=prec).set_bopt(w, "alg2")
    rng = np.random.default_rng(12)
    dt = torch.complex128 if prec == "c128" else torch.complex64
    g = torch.Generator(device="cuda").manual_seed(5)
    f = torch.randn(R, x.size, dtype=dt, device="cuda", generator=g)
    out = plan.apply(f)
    h = torch.randn(R, M, dtype=dt, device="cuda", generator=g)
    outa = plan.adjoint_apply(h)
    # every RHS of the batch: fast path vs the generic kernels (complex weights with
    # zero imaginary part take the one-thread-per-output path) -- catches races in any row
    pg = P.Plan(x, M, sigma, m, precision=prec).set_bopt(w + 0j, "alg2")
    tol_full = 1e-13 if prec == "c128" else 1e-5
    ga = pg.apply(f)
    gb = pg.adjoint_apply(h)
    assert O.rel_l2(out.cpu().numpy().astype(np.complex128), ga.cpu().numpy().astype(np.complex128)) <= tol_full
    assert O.rel_l2(outa.cpu().numpy().astype(np.complex128), gb.cpu().numpy().astype(np.complex128)) <= tol_full
    for r in sorted(rng.choice(R, 2, replace=False)):
        fr = f[r:r + 1].cpu().numpy().astype(np.complex128)
        ref = O.apply_inverse(x, M, sigma, m, w, 1.0, fr)
        assert O.rel_l2(out[r:r + 1].cpu().numpy().astype(np.complex128), ref) <= TOL[prec]
        hr = h[r:r + 1].cpu().numpy().astype(np.complex128)
        ref = O.apply_adjoint(x, M, sigma, m, w, 1.0, hr)
        assert O.rel_l2(outa[r:r + 1].cpu().numpy().astype(np.complex128), ref) <= TOL[prec]


# ------------------------------------------------------------------ setup on the GPU
def test_plain_nfft_window_weights_and_ndft(P, torch):
    """INFT_PLAIN_NFFT: the GPU forms the window matrix B itself; its apply must
    equal the oracle's plain NFFT and approximate the NDFT."""
    M, sigma, m, N = 256, 2.0, 6, 256
    x = np.random.default_rng(5).random(N) - 0.5
    plan = P.Plan(x, M, sigma, m).precompute("plain")
    wref = O.window_slot_weights(x, M, sigma, m)
    wg = plan.get_bopt()
    assert np.abs(wg - wref).max() <= 1e-13 * np.abs(wref).max()
    fh = S.uniform_complex(2, M, 1)
    fe = O.ndft(x, fh, M)
    got = plan.adjoint_apply(_dev(torch, fh)).cpu().numpy()
    assert O.rel_l2(got, O.apply_adjoint(x, M, sigma, m, wref, 1.0, fh)) <= 1e-12
    assert np.abs(got - fe).max() <= 1e-10 * np.abs(fe).max()
    got = plan.apply(_dev(torch, fe)).cpu().numpy()
    he = O.ndft_adjoint(x, fe, M)
    assert np.abs(got - he).max() <= 1e-10 * np.abs(he).max()


def test_alg2_gpu_setup_cfg1(P, torch):
    """GPU Alg. 2 (Gram form + Jacobi) against the oracle's Gram solution on
    config 1 (full rank: the minimiser is unique, reading D6 part P2)."""
    c, x, M, sigma, m = _cfg(1)
    plan = P.Plan(x, M, sigma, m).precompute("alg2")
    info = plan.info()
    assert info["n_rank_deficient"] == 0 and info["max_col_size"] == 8 and info["n_empty_cols"] == 0
    wg = plan.get_bopt()
    wo, _ = O.alg2_setup(x, M, sigma, m, form="gram")
    assert np.abs(wg - wo).max() <= 1e-7 * np.abs(wo).max()
    # objective at the rank bound sqrt(Ms - M) (sigma = 2)
    assert abs(O.objective_alg2(x, M, sigma, m, wg) - np.sqrt(O.msigma(M, sigma) - M)) < 1e-6
    fh = S.make_rhs(c)
    f = O.ndft(x, fh, M)
    got = plan.apply(_dev(torch, f)).cpu().numpy()
    assert O.rel_l2(got, O.apply_inverse(x, M, sigma, m, wg, 1.0, f)) <= TOL["c128"]
    assert O.rel_l2(got, O.apply_inverse(x, M, sigma, m, wo, 1.0, f)) < 1e-9


def test_alg1_gpu_setup_cfg2(P, torch):
    c, x, M, sigma, m = _cfg(2)
    plan = P.Plan(x, M, sigma, m).precompute("alg1")
    wg = plan.get_bopt()
    wo, _ = O.alg1_setup(x, M, sigma, m)
    f = S.make_rhs(c, kind="adjoint")
    h = O.ndft_adjoint(x, f, M)
    got = plan.adjoint_apply(_dev(torch, h)).cpu().numpy()
    assert O.rel_l2(got, O.apply_adjoint(x, M, sigma, m, wg, 1.0 / M, h)) <= TOL["c128"]
    # per-node objective ||K_j b - M e_j|| equal to the oracle's (unique minimum value)
    K = O.K_kernel_matrix(x, M, sigma, m)
    Ms = O.msigma(M, sigma)
    l0 = O.node_base(x, Ms, m)
    for j in range(0, x.size, 37):
        cols = np.mod(l0[j] + np.arange(2 * m + 1) + Ms // 2, Ms)
        e = np.zeros(x.size)
        e[j] = M
        rg = np.linalg.norm(K[:, cols] @ wg[j] - e)
        ro = np.linalg.norm(K[:, cols] @ wo[j] - e)
        assert rg <= ro * (1 + 1e-6) + 1e-9 * M


def test_alg2_full_support_exact_on_gpu(P, torch):
    """sigma = 1, m = M_sigma/2: K^*B = I attainable -> exact recovery."""
    M, N = 8, 16
    x = S.jittered(N, 7)
    plan = P.Plan(x, M, 1.0, 4).precompute("alg2")
    fh = S.uniform_complex(3, M, 2)
    got = plan.apply(_dev(torch, O.ndft(x, fh, M))).cpu().numpy()
    assert O.rel_l2(got, fh) < 1e-6


def test_alg1_full_support_exact_on_gpu(P, torch):
    M, N = 8, 6
    x = S.jittered(N, 9)
    plan = P.Plan(x, M, 2.0, 8).precompute("alg1")
    f = S.normal_complex(3, N, 1)
    got = plan.adjoint_apply(_dev(torch, O.ndft_adjoint(x, f, M))).cpu().numpy()
    assert O.rel_l2(got, f) < 1e-9


# ------------------------------------------------------------------ edge cases and invariants
def test_edge_cases(P, torch):
    M, sigma, m = 64, 2.0, 4
    x = S.jittered(100, 3)
    plan = P.Plan(x, M, sigma, m)
    with pytest.raises(P.InftError) as e:
        plan.apply(torch.zeros(1, 100, dtype=torch.complex128, device="cuda"))
    assert e.value.status == 4
    with pytest.raises(P.InftError) as e:
        P.Plan(np.array([0.1, 0.5]), M, sigma, m)
    assert e.value.status == 2
    with pytest.raises(P.InftError):
        P.Plan(np.array([0.1, np.nan]), M, sigma, m)
    with pytest.raises(P.InftError):
        P.Plan(x, 63, sigma, m)  # M odd
    with pytest.raises(P.InftError):
        P.Plan(x, M, 1.3, m)  # sigma M not an even integer
    w = _live_random_weights(x, M, sigma, m, 1)
    plan.set_bopt(w, "alg2")
    empty = torch.zeros(0, 100, dtype=torch.complex128, device="cuda")
    assert plan.apply(empty).shape == (0, M)
    # N = 0: inverse of nothing is zero
    p0 = P.Plan(np.zeros(0), M, sigma, m).set_bopt(np.zeros((0, 9)), "alg2")
    z = p0.apply(torch.zeros(2, 0, dtype=torch.complex128, device="cuda")).cpu().numpy()
    assert np.all(z == 0)


def test_unsorted_nodes_boundary_and_on_grid(P, torch):
    """Non-identity permutation, nodes at -1/2 and exactly on grid points (slot 2m live)."""
    M, sigma, m = 64, 2.0, 3
    Ms = 128
    x = np.concatenate([S.iid_sorted(150, 2)[::-1], [-0.5, 0.0, 5.0 / Ms, -17.0 / Ms, 0.5 - 1.0 / Ms]])
    rng = np.random.default_rng(1)
    x = x[rng.permutation(x.size)]
    w = _live_random_weights(x, M, sigma, m, 2)
    assert w[:, 2 * m].any()
    plan = P.Plan(x, M, sigma, m).set_bopt(w, "alg2")
    assert plan.info()["perm_identity"] == 0
    for R in (1, 33):
        f = S.normal_complex(R, x.size, R)
        got = plan.apply(_dev(torch, f)).cpu().numpy()
        assert O.rel_l2(got, O.apply_inverse(x, M, sigma, m, w, 1.0, f)) <= TOL["c128"]
        h = S.normal_complex(R, M, R + 1)
        got = plan.adjoint_apply(_dev(torch, h)).cpu().numpy()
        assert O.rel_l2(got, O.apply_adjoint(x, M, sigma, m, w, 1.0, h)) <= TOL["c128"]
    np.testing.assert_array_equal(plan.get_bopt(), w)


def test_aliasing_full_support_generic_path(P, torch):
    """2m+1 > M_sigma: aliased slots (reading A5) handled by the generic kernels."""
    M, sigma, m = 8, 1.0, 4
    x = S.jittered(16, 7)
    w = _live_random_weights(x, M, sigma, m, 3)
    plan = P.Plan(x, M, sigma, m).set_bopt(w, "alg2")
    f = S.normal_complex(2, 16, 3)
    got = plan.apply(_dev(torch, f)).cpu().numpy()
    assert O.rel_l2(got, O.apply_inverse(x, M, sigma, m, w, 1.0, f)) <= TOL["c128"]


def test_complex_weights_generic_equals_oracle_and_fast_path(P, torch):
    M, sigma, m = 128, 2.0, 4
    x = S.jittered(256, 4)
    w = _live_random_weights(x, M, sigma, m, 5)
    wc = w + 1j * _live_random_weights(x, M, sigma, m, 6)
    pc = P.Plan(x, M, sigma, m).set_bopt(wc, "alg2")
    f = S.normal_complex(5, 256, 4)
    got = pc.apply(_dev(torch, f)).cpu().numpy()
    assert O.rel_l2(got, O.apply_inverse(x, M, sigma, m, wc, 1.0, f)) <= TOL["c128"]
    h = S.normal_complex(5, M, 5)
    got = pc.adjoint_apply(_dev(torch, h)).cpu().numpy()
    assert O.rel_l2(got, O.apply_adjoint(x, M, sigma, m, wc, 1.0, h)) <= TOL["c128"]
    # generic (complex with zero imaginary part) vs fast (real) kernels
    pr = P.Plan(x, M, sigma, m).set_bopt(w, "alg2")
    pz = P.Plan(x, M, sigma, m).set_bopt(w + 0j, "alg2")
    assert pr.info()["fast_path"] >= 1
    a = pr.apply(_dev(torch, f)).cpu().numpy()
    b = pz.apply(_dev(torch, f)).cpu().numpy()
    assert O.rel_l2(a, b) < 1e-14


def test_host_buffers_equal_device(P, torch):
    """The C ABI accepts host pointers (pageable numpy and pinned torch)."""
    M, sigma, m = 512, 2.0, 8
    x = S.jittered(1024, 5)
    w = _live_random_weights(x, M, sigma, m, 7)
    plan = P.Plan(x, M, sigma, m).set_bopt(w, "alg2")
    f = S.normal_complex(70, 1024, 2)
    ref = plan.apply(_dev(torch, f)).cpu().numpy()
    got = plan.apply(f)  # numpy in, numpy out
    np.testing.assert_array_equal(got, ref)
    fp = torch.from_numpy(f).pin_memory()
    outp = torch.empty(70, M, dtype=torch.complex128).pin_memory()
    plan.apply(fp, out=outp)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(outp.numpy(), ref)
    h = S.normal_complex(70, M, 3)
    refa = plan.adjoint_apply(_dev(torch, h)).cpu().numpy()
    np.testing.assert_array_equal(plan.adjoint_apply(h), refa)


def test_gpu_adjointness_and_batch_invariance(P, torch):
    c, x, M, sigma, m = _cfg(1)
    plan = P.Plan(x, M, sigma, m).precompute("alg2")
    f = S.normal_complex(40, x.size, 1)
    h = S.normal_complex(40, M, 2)
    A = plan.apply(_dev(torch, f)).cpu().numpy()
    B = plan.adjoint_apply(_dev(torch, h)).cpu().numpy()
    for r in range(3):
        a = np.vdot(h[r], A[r])
        b = np.vdot(B[r], f[r])
        assert abs(a - b) <= 1e-12 * abs(a)
    one = plan.apply(_dev(torch, f[7:8])).cpu().numpy()
    assert O.rel_l2(one, A[7:8]) <= 1e-15


def test_binding_rejects_mismatched_buffers(P, torch):
    """The C side trusts R*N / R*M elements at the plan's precision: the binding checks dtype,
    trailing size, output size and device before passing raw pointers (no silent overrun)."""
    M, sigma, m = 64, 2.0, 4
    x = S.jittered(100, 3)
    plan = P.Plan(torch.from_numpy(x).to(torch.float32).cuda(), M, sigma, m)  # float32 nodes: converted
    np.testing.assert_array_equal(plan.get_bins()[0], O.node_base(x.astype(np.float32).astype(np.float64), 128, m))
    plan = P.Plan(x, M, sigma, m).set_bopt(_live_random_weights(x, M, sigma, m, 1), "alg2")
    f = torch.zeros(2, 100, dtype=torch.complex128, device="cuda")
    with pytest.raises(TypeError):
        plan.apply(f.to(torch.complex64))
    with pytest.raises(ValueError):
        plan.apply(torch.zeros(2, 99, dtype=torch.complex128, device="cuda"))
    with pytest.raises(ValueError):
        plan.apply(f, out=torch.zeros(1, M, dtype=torch.complex128, device="cuda"))
    with pytest.raises(ValueError):  # config-5-like trap: adjoint output sized [R][M] with N > M
        plan.adjoint_apply(torch.zeros(2, M, dtype=torch.complex128, device="cuda"),
                           out=torch.zeros(2, M, dtype=torch.complex128, device="cuda"))
    with pytest.raises(ValueError):
        P.Plan(np.zeros((10, 2)), M, sigma, m)  # 2-D nodes for a 1-D plan
    assert plan.apply(f).shape == (2, M)

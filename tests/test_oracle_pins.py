"""Pins of the CPU oracle against what the paper and the mathematics fix
(DESIGN.md "Oracle pins").  No GPU.  Citations: P:<n> = PAPER.md line n."""
import os

import numpy as np
import pytest
import scipy.special
from scipy.integrate import quad

import oracle as O
import synth as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ window
def test_i0_series_matches_scipy():
    x = np.concatenate([np.linspace(0, 60, 301), [1e-3, 37.7, 50.26]])
    np.testing.assert_allclose(O.i0(x), scipy.special.i0(x), rtol=1e-14)


@pytest.mark.parametrize("Ms,m,sigma", [(64, 6, 2.0), (32, 4, 2.0), (40, 3, 1.25)])
def test_kb_pair_by_quadrature(Ms, m, sigma):
    """what(k) = int w(x) e^{-2 pi i k x} dx (eq. fourier_transform)
    for the closed-form KB pair of reading A7, |k| <= M/2.  Integrating the
    truncated w_m instead of w differs by the window's truncation error, which
    decays like e^{-b m} (b = pi (2 - 1/sigma)); that is the tolerance."""
    M = int(Ms / sigma)
    for k in (0, 1, M // 4, M // 2):
        val = quad(lambda t: O.kb_w(np.array([t]), Ms, m, sigma)[0] * np.cos(2 * np.pi * k * t),
                   -m / Ms, m / Ms, limit=400, epsabs=0, epsrel=1e-13)[0]
        assert abs(val / O.kb_what(k, Ms, m, sigma) - 1) < 10 * np.exp(-O.kb_b(sigma) * m)


def test_window_properties():
    Ms, m, s = 32, 4, 2.0
    wh = O.window_hat_vector(16, s, m)
    assert np.all(wh > 0)
    np.testing.assert_allclose(wh[1:], wh[1:][::-1], rtol=1e-15)  # even: k <-> -k
    x = np.linspace(-0.49, 0.49, 97)
    np.testing.assert_allclose(O.kb_w_periodic(x, Ms, m, s), O.kb_w_periodic(x + 1, Ms, m, s), rtol=1e-12)
    far = np.array([m / Ms + 1e-9, 0.3, -0.4])
    assert np.all(O.kb_w(far, Ms, m, s) == 0)


def test_deconv_vector_is_matrix_D():
    """d_k = s / (M_sigma what(k)) (eq. matrix_D) with scale s (A2)."""
    d = O.deconv_vector(8, 2.0, 2, s=0.5)
    np.testing.assert_allclose(d, 0.5 / (16 * O.kb_what(np.arange(-4, 4), 16, 2, 2.0)), rtol=0)


# --------------------------------------------------------------- index sets
def _read_golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as fh:
        for line in fh:
            line = line.split("#")[0].strip()
            if line:
                lhs, rhs = line.split("|")
                rows.append((lhs.split(), [float(v) for v in rhs.split()]))
    return rows


def test_index_sets_golden():
    for lhs, members in _read_golden("index_sets.txt"):
        x, Ms, m = float(lhs[0]), int(lhs[1]), int(lhs[2])
        assert O.index_set_node_bruteforce(x, Ms, m) == [int(v) for v in members]
        # slot layout l0 + live slots gives the same set (wrapped to [-Ms/2, Ms/2))
        live = O.slot_live(np.array([x]), Ms, m)[0]
        l0 = O.node_base(np.array([x]), Ms, m)[0]
        got = sorted(((l0 + t + Ms // 2) % Ms) - Ms // 2 for t in np.nonzero(live)[0])
        assert got == [int(v) for v in members]


def test_slot_layout_matches_definition_random():
    rng = np.random.default_rng(11)
    for Ms, m in [(16, 2), (64, 8), (10, 5), (8, 4), (6, 3)]:
        xs = np.concatenate([rng.random(60) - 0.5, np.arange(-Ms // 2, Ms // 2) / Ms])  # incl. on-grid
        live = O.slot_live(xs, Ms, m)
        l0 = O.node_base(xs, Ms, m)
        for j, x in enumerate(xs):
            want = O.index_set_node_bruteforce(x, Ms, m)
            got = sorted(((l0[j] + t + Ms // 2) % Ms) - Ms // 2 for t in np.nonzero(live[j])[0])
            assert got == want
            # D4: slots 0..2m-1 live unless aliased; slot 2m live iff Ms x in Z
            if 2 * m + 1 <= Ms:
                assert live[j, 2 * m] == (np.float64(Ms) * x == np.round(np.float64(Ms) * x))


def test_index_set_duality():
    """j in I(l) <=> l in I(x_j) (eqs. set_xj / set_l)."""
    x = S.jittered(40, 3)
    Ms, m = 32, 3
    sets = O.grid_node_sets(x, Ms, m)
    for n in range(Ms):
        l = n - Ms if n >= Ms // 2 else n
        js = sorted(j for (j, t) in sets[n])
        want = [j for j in range(x.size) if l in O.index_set_node_bruteforce(x[j], Ms, m)]
        assert js == want


def test_jittered_column_sizes():
    """Jittered nodes with N = M_sigma: every |I(l)| = 2m (config-5 structure)."""
    for N, m in [(64, 8), (128, 4)]:
        x = S.jittered(N, 4)
        sets = O.grid_node_sets(x, N, m)
        assert all(len(s) == 2 * m for s in sets)


def test_bins_stable_permutation():
    x = S.iid_sorted(200, 9)[::-1].copy()
    l0, n0, b, perm = O.bins_1d(x, 64, 3, 16)
    assert np.all(np.diff(n0[perm]) >= 0) and np.all(np.diff(b[perm]) >= 0)
    for v in np.unique(n0):  # stable: ties keep original order
        idx = perm[n0[perm] == v]
        assert np.all(np.diff(idx) > 0)
    assert np.all(n0 == np.mod(l0, 64))
    # increasing nodes -> the sorted order is a cyclic shift of the caller order
    xs = S.jittered(512, 4)
    _, _, _, pj = O.bins_1d(xs, 512, 8, 16)
    assert np.all(pj == (np.arange(512) + pj[0]) % 512)


def test_node_generators_golden():
    for lhs, vals in _read_golden("nodes.txt"):
        kind, N = lhs[0], int(lhs[1])
        if kind == "chebyshev":
            np.testing.assert_allclose(S.chebyshev(N), vals, atol=1e-16)
        elif kind == "jittered0":
            np.testing.assert_allclose(S.jittered(N, 0, jitter=0.0), vals, atol=0)
    x = S.jittered(1000, 1)
    assert np.all(np.diff(x) > 0) and x.min() >= -0.5 and x.max() < 0.5
    xp = S.polar(16, 16)
    assert xp.min() >= -0.5 and xp.max() < 0.5


# --------------------------------------------------------------------- NDFT
def test_equispaced_identities():
    """A^*A = N I_M for M <= N and A A^* = M I_N for N | M."""
    for N, M in [(16, 8), (16, 16), (12, 6)]:
        A = O.matrix_A(S.equispaced(N), M)
        np.testing.assert_allclose(A.conj().T @ A, N * np.eye(M), atol=1e-12)
    for N, M in [(8, 16), (8, 8), (6, 12)]:
        A = O.matrix_A(S.equispaced(N), M)
        np.testing.assert_allclose(A @ A.conj().T, M * np.eye(N), atol=1e-12)


def test_ndft_adjointness():
    x = S.jittered(30, 2)
    fh = S.uniform_complex(1, 16, 1)[0]
    f = S.normal_complex(1, 30, 2)[0]
    lhs = np.vdot(f, O.ndft(x, fh[None], 16)[0])
    rhs = np.vdot(O.ndft_adjoint(x, f[None], 16)[0], fh)
    assert abs(lhs - rhs) < 1e-12 * abs(lhs)


@pytest.mark.parametrize("n", [1, 2, 8, 64, 6, 12])
def test_oracle_dft_against_definition(n):
    x = S.normal_complex(1, n, n)[0]
    q = np.arange(n)
    for sign in (-1, 1):
        want = np.exp(sign * 2j * np.pi * np.outer(q, q) / n) @ x
        np.testing.assert_allclose(O.dft(x, sign), want, atol=1e-12 * max(1, np.abs(want).max()))
    np.testing.assert_allclose(O.dft(x, -1), np.fft.fft(x), atol=1e-12 * max(1, np.abs(x).sum()))


# -------------------------------------------------------------------- apply
def test_plain_nfft_vs_ndft_decays_in_m():
    """With the window matrix B (s = 1) the fast pair is the ordinary NFFT /
    adjoint NFFT (A ~ BFD P:229, A^* ~ D^*F^*B^* P:288).  KB, sigma = 2,
    M = N = 256: error <= 1e-10 at m = 6 and decreasing in m.
    This pins the D, F, B sign and index conventions (A9) and the window (A7)."""
    M, N, s = 256, 256, 2.0
    x = np.random.default_rng(5).random(N) - 0.5
    fh = S.uniform_complex(2, M, 1)
    fe = O.ndft(x, fh, M)
    he = O.ndft_adjoint(x, fe, M)
    errs = []
    for m in (2, 4, 6, 8):
        w = O.window_slot_weights(x, M, s, m)
        ef = np.abs(O.apply_adjoint(x, M, s, m, w, 1.0, fh) - fe).max() / np.abs(fe).max()
        eh = np.abs(O.apply_inverse(x, M, s, m, w, 1.0, fe) - he).max() / np.abs(he).max()
        errs.append(max(ef, eh))
    assert errs[2] <= 1e-10
    assert all(a > b for a, b in zip(errs, errs[1:]))


def test_plain_nfft_2d_vs_ndft():
    """Tensor reading A12: 2-D plain NFFT against the 2-D NDFT."""
    M, s, m = (16, 12), 2.0, 6
    x = np.random.default_rng(6).random((70, 2)) - 0.5
    w = O.window_slot_weights_2d(x, M, s, m)
    fh = S.uniform_complex(2, 16 * 12, 3)
    fe = O.ndft(x, fh, M)
    assert np.abs(O.apply_adjoint(x, M, s, m, w, 1.0, fh) - fe).max() < 1e-9 * np.abs(fe).max()
    he = O.ndft_adjoint(x, fe, M)
    assert np.abs(O.apply_inverse(x, M, s, m, w, 1.0, fe) - he).max() < 1e-9 * np.abs(he).max()


@pytest.mark.parametrize("cplx", [False, True])
def test_fast_oracle_equals_dense_literal_1d(cplx):
    """C loops == s D^* F^* B^* f and s B F D h as explicit matrices."""
    rng = np.random.default_rng(2)
    M, s, m = 24, 2.0, 3
    x = S.jittered(40, 1)
    w = rng.standard_normal((40, 2 * m + 1))
    if cplx:
        w = w + 1j * rng.standard_normal(w.shape)
    f = S.normal_complex(3, 40, 2)
    h = S.normal_complex(3, M, 3)
    assert O.rel_l2(O.apply_inverse(x, M, s, m, w, 0.7, f), O.dense_inverse(x, M, s, m, w, 0.7, f)) < 1e-13
    assert O.rel_l2(O.apply_adjoint(x, M, s, m, w, 0.7, h), O.dense_adjoint(x, M, s, m, w, 0.7, h)) < 1e-13


def test_fast_oracle_equals_dense_literal_2d_and_nonpow2():
    rng = np.random.default_rng(3)
    M, m = (8, 6), 2
    x = rng.random((50, 2)) - 0.5
    w = rng.standard_normal((50, 25))
    f = S.normal_complex(2, 50, 1)
    h = S.normal_complex(2, 48, 1)
    assert O.rel_l2(O.apply_inverse(x, M, 2.0, m, w, 0.3, f), O.dense_inverse(x, M, 2.0, m, w, 0.3, f)) < 1e-13
    assert O.rel_l2(O.apply_adjoint(x, M, 2.0, m, w, 0.3, h), O.dense_adjoint(x, M, 2.0, m, w, 0.3, h)) < 1e-13
    # M_sigma = 12*1.5 = 18: not a power of two (plain DFT branch)
    x1 = S.jittered(30, 4)
    w1 = rng.standard_normal((30, 5))
    f1 = S.normal_complex(2, 30, 5)
    assert O.rel_l2(O.apply_inverse(x1, 12, 1.5, 2, w1, 1.0, f1), O.dense_inverse(x1, 12, 1.5, 2, w1, 1.0, f1)) < 1e-13


def test_apply_pair_adjointness_and_linearity():
    """<inverse(f), h> = <f, inverse_adjoint(h)> for the same B_opt and real s
    (the two maps are conjugate transposes: (s D^*F^*B^*)^* = s B F D)."""
    rng = np.random.default_rng(4)
    M, s, m = 32, 2.0, 4
    x = S.jittered(48, 6)
    w = rng.standard_normal((48, 9))
    f = S.normal_complex(1, 48, 7)
    h = S.normal_complex(1, M, 8)
    a = np.vdot(h[0], O.apply_inverse(x, M, s, m, w, 0.25, f)[0])
    b = np.vdot(O.apply_adjoint(x, M, s, m, w, 0.25, h)[0], f[0])
    assert abs(a - b) < 1e-13 * abs(a)
    f2 = S.normal_complex(2, 48, 9)
    lin = O.apply_inverse(x, M, s, m, w, 1.0, 2.0 * f2[:1] - 3j * f2[1:])
    sep = 2.0 * O.apply_inverse(x, M, s, m, w, 1.0, f2[:1]) - 3j * O.apply_inverse(x, M, s, m, w, 1.0, f2[1:])
    assert O.rel_l2(lin, sep) < 1e-14
    batch = O.apply_inverse(x, M, s, m, w, 1.0, f2)
    one = O.apply_inverse(x, M, s, m, w, 1.0, f2[1:])
    np.testing.assert_array_equal(batch[1:], one)


# -------------------------------------------------------------------- setup
def test_alg2_columns_equal_textbook_lstsq():
    """Each column of Alg. 2 is min ||L_l b - e_l|| over real b;
    full-rank columns must equal numpy.linalg.lstsq on the real-stacked system."""
    M, s, m = 32, 2.0, 3
    x = S.jittered(64, 2)
    Ms = 64
    w, info = O.alg2_setup(x, M, s, m, form="explicit")
    sets = O.grid_node_sets(x, Ms, m)
    for n in (0, 5, 31, 40, 63):
        js = [j for (j, t) in sets[n]]
        ts = [t for (j, t) in sets[n]]
        l = n - Ms if n >= Ms // 2 else n
        # L_l from its definition, entry by entry (eq. matrix_Ll)
        k = np.arange(-M // 2, M // 2)
        wh = O.window_hat_vector(M, s, m)
        svals = np.arange(-Ms // 2, Ms // 2)
        L = np.array([[np.sum(np.exp(2j * np.pi * k * (sv / Ms - x[j])) / wh) / Ms for j in js] for sv in svals])
        e = np.zeros(Ms)
        e[l + Ms // 2] = 1
        b = np.linalg.lstsq(np.vstack([L.real, L.imag]), np.concatenate([e, 0 * e]), rcond=None)[0]
        np.testing.assert_allclose(w[js, ts], b, rtol=1e-9, atol=1e-12 * np.abs(b).max())


def test_alg2_gram_equals_explicit():
    """Gram identity (L^*L)_{jj'} = G(x_j - x_j'), L^*e_l = K+(x_j - l/M_sigma)
    (from F^*F = M_sigma I_M) gives the same solution as the explicit form."""
    M, s, m = 64, 2.0, 4
    x = S.jittered(128, 0)
    we, _ = O.alg2_setup(x, M, s, m, form="explicit")
    wg, _ = O.alg2_setup(x, M, s, m, form="gram")
    assert np.abs(we - wg).max() < 1e-8 * np.abs(we).max()
    f = S.normal_complex(2, 128, 1)
    assert O.rel_l2(O.apply_inverse(x, M, s, m, wg, 1.0, f), O.apply_inverse(x, M, s, m, we, 1.0, f)) < 1e-11


def test_alg2_objective_bounds():
    """Window B is feasible => ||K^*B_opt - I|| <= ||K^*B - I||; rank(K^*B) <= M
    => objective >= sqrt(M_sigma - M); at sigma = 2 it attains the bound."""
    M, s, m = 32, 2.0, 4
    x = S.jittered(96, 3)
    w, _ = O.alg2_setup(x, M, s, m)
    obj = O.objective_alg2(x, M, s, m, w)
    win = O.objective_alg2(x, M, s, m, O.window_slot_weights(x, M, s, m))
    assert obj <= win
    assert abs(obj - np.sqrt(64 - 32)) < 1e-6 * np.sqrt(32)
    # per-column residuals sum to the objective (column decomposition P:1220-1224)
    _, info = O.alg2_setup(x, M, s, m, form="gram")
    assert abs(np.sqrt(sum(r * r for r in info["resid"].values())) - obj) < 1e-6 * obj


def test_alg2_full_support_exact_inverse():
    """sigma = 1, m = M_sigma/2 (all grid points in every I(x_j)), N >= 2M:
    K^*B = I is attainable, so D^*F^*B_opt^* A = I_M and consistent data is
    recovered exactly (special case of P:1190-1194 = textbook LS)."""
    M, N = 8, 16
    x = S.jittered(N, 7)
    w, _ = O.alg2_setup(x, M, 1.0, 4)
    fh = S.uniform_complex(3, M, 2)
    assert O.rel_l2(O.apply_inverse(x, M, 1.0, 4, w, 1.0, O.ndft(x, fh, M)), fh) < 1e-10


def test_alg2_full_support_2d():
    rng = np.random.default_rng(3)
    M = (4, 4)
    x = rng.random((40, 2)) - 0.5
    w, _ = O.alg2_setup(x, M, 1.0, 2)
    fh = S.uniform_complex(2, 16, 2)
    assert O.rel_l2(O.apply_inverse(x, M, 1.0, 2, w, 1.0, O.ndft(x, fh, M)), fh) < 1e-10
    # separable Gram (reading A12): Re(G1 G2) gives the explicit solution
    wg, _ = O.alg2_setup(x, M, 1.0, 2, form="gram")
    assert O.rel_l2(O.apply_inverse(x, M, 1.0, 2, wg, 1.0, O.ndft(x, fh, M)), fh) < 1e-7


def test_alg1_full_support_exact():
    """m = M_sigma/2, M >= N, sigma = 2: K B^* = M I_N attainable, so the inverse
    adjoint (1/M) B_opt F D h recovers f from h = A^* f (Remark P:1091-1107)
    and A fcheck = g for the inverse."""
    M, N = 8, 6
    x = S.jittered(N, 9)
    w, _ = O.alg1_setup(x, M, 2.0, 8)
    f = S.normal_complex(3, N, 1)
    h = O.ndft_adjoint(x, f, M)
    assert O.rel_l2(O.apply_adjoint(x, M, 2.0, 8, w, 1.0 / M, h), f) < 1e-12
    g = S.normal_complex(2, N, 3)
    assert O.rel_l2(O.ndft(x, O.apply_inverse(x, M, 2.0, 8, w, 1.0 / M, g), M), g) < 1e-12


def test_alg1_objective_decreases_in_m():
    """'increasing the cut-off m expectedly leads to better results';
    optimized beats the window matrix B."""
    N, M, s = 64, 256, 2.0
    x = S.jittered(N, 3)
    objs = []
    for m in (2, 4, 6):
        w, _ = O.alg1_setup(x, M, s, m)
        objs.append(O.objective_alg1(x, M, s, m, w))
    assert objs[0] > objs[1] > objs[2]
    win = O.objective_alg1(x, M, s, 4, O.window_slot_weights(x, M, s, 4))
    assert objs[1] < win


def test_alg1_columns_equal_textbook_lstsq():
    N, M, s, m = 20, 64, 2.0, 3
    x = S.jittered(N, 5)
    w, _ = O.alg1_setup(x, M, s, m)
    Ms = 128
    live = O.slot_live(x, Ms, m)
    l0 = O.node_base(x, Ms, m)
    k = np.arange(-M // 2, M // 2)
    wh = O.window_hat_vector(M, s, m)
    for j in (0, 7, 19):
        ts = np.nonzero(live[j])[0]
        ls = l0[j] + ts
        # K_j from eq. matrix_Kj, entry by entry (KB what is even: what(-k) = what(k), A8)
        Kj = np.array([[np.sum(np.exp(2j * np.pi * k * (x[h] - l / Ms)) / wh) / Ms for l in ls] for h in range(N)])
        e = np.zeros(N)
        e[j] = M
        b = np.linalg.lstsq(np.vstack([Kj.real, Kj.imag]), np.concatenate([e, 0 * e]), rcond=None)[0]
        np.testing.assert_allclose(w[j, ts], b, rtol=1e-9, atol=1e-12 * np.abs(b).max())


def test_alg2_adjoint_fails_for_N_gt_M():
    """'our optimization was not successful in the case N>M'."""
    M, s, m = 32, 2.0, 4
    x = S.jittered(64, 1)
    w, _ = O.alg2_setup(x, M, s, m, form="gram")
    f = S.normal_complex(2, 64, 2)
    err = O.rel_l2(O.apply_adjoint(x, M, s, m, w, 1.0, O.ndft_adjoint(x, f, M)), f)
    assert err > 0.3


def test_alg2_config1_recovery_accuracy():
    """Config 1 (M=256, N=512 jittered, sigma=2, m=4): the inverse recovers fhat;
    the paper prints no value (figures absent) -- a sanity envelope, not a pin."""
    c = S.config(1)
    x = S.make_nodes(c)
    M, m, s = c["M"][0], c["m"], c["sigma"]
    w, info = O.alg2_setup(x, M, s, m, form="gram")
    assert info["n_rank_deficient"] == 0 and info["max_col_size"] == 8
    fh = S.make_rhs(c)
    err = O.rel_l2(O.apply_inverse(x, M, s, m, w, 1.0, O.ndft(x, fh, M)), fh)
    assert err < 1e-4

"""Pins of the oracle's Dirichlet-kernel variant (Remarks P:934-957 and
P:1343-1358, reading A21): what(k) = 1 for |k| < M/2 and the unpaired entry k = -M/2 of D^*
set to zero.  Every pin compares the oracle's direct sums / matrix products with the paper's
closed forms or with a mathematically exact special case -- never with a retyped formula."""
import numpy as np

import oracle as O
import synth as S


def test_dirichlet_kernel_closed_form():
    """G and K+ of the Dirichlet variant are (1/M_sigma) D_{M/2-1}(x), eq. kernel_Dirichlet
    P:937-944: sum_{k=-M/2+1}^{M/2-1} e^{2 pi i k x} = sin((M-1) pi x)/sin(pi x)."""
    rng = np.random.default_rng(0)
    for M, sigma in [(16, 2.0), (64, 1.5), (256, 2.0)]:
        Ms = O.msigma(M, sigma)
        x = rng.random(200) - 0.5
        ref = O.dirichlet_kernel(x, M) / Ms
        for fn in (O.G_kernel, O.Kplus_kernel):
            v = fn(x, M, sigma, 4, window="dirichlet")
            assert np.abs(v.imag).max() < 1e-13 * M / Ms
            assert np.abs(v.real - ref).max() < 1e-12 * M / Ms
        # value at 0 = M - 1 terms
        assert abs(O.G_kernel(0.0, M, sigma, 4, window="dirichlet").real - (M - 1) / Ms) < 1e-13


def test_dirichlet_deconvolution():
    d = O.deconv_vector(32, 2.0, 4, 0.5, window="dirichlet")
    assert d[0] == 0.0 and np.all(d[1:] == 0.5 / 64)


def test_dirichlet_L_matrix_closed_form():
    """L_l = F D H_l (eq. matrix_Ll) equals [(1/M_sigma) D_{M/2-1}(l/M_sigma - x_j)] with rows
    l = -M_sigma/2 .. M_sigma/2 - 1 (Remark P:1343-1358)."""
    M, sigma, m = 32, 2.0, 3
    Ms = O.msigma(M, sigma)
    xs = S.jittered(7, 2)
    L = O.L_explicit(5, xs, M, sigma, m, window="dirichlet")
    rows = np.arange(Ms) - Ms // 2
    ref = O.dirichlet_kernel(rows[:, None] / Ms - xs[None, :], M) / Ms
    assert np.abs(L - ref).max() < 1e-12


def test_dirichlet_K_matrix_closed_form():
    """K = A D^* F^* equals [(1/M_sigma) D_{M/2-1}(x_h - l/M_sigma)] (Remark P:934-957)."""
    M, sigma, m = 32, 2.0, 3
    Ms = O.msigma(M, sigma)
    x = S.jittered(9, 4)
    K = O.K_kernel_matrix(x, M, sigma, m, window="dirichlet")
    cols = np.arange(Ms) - Ms // 2
    ref = O.dirichlet_kernel(x[:, None] - cols[None, :] / Ms, M) / Ms
    assert np.abs(K - ref).max() < 1e-12


def test_dirichlet_alg2_gram_equals_explicit():
    M, s, m = 64, 2.0, 4
    x = S.jittered(128, 5)
    we, _ = O.alg2_setup(x, M, s, m, form="explicit", window="dirichlet")
    wg, _ = O.alg2_setup(x, M, s, m, form="gram", window="dirichlet")
    f = S.normal_complex(2, 128, 1)
    a = O.apply_inverse(x, M, s, m, we, 1.0, f, window="dirichlet")
    b = O.apply_inverse(x, M, s, m, wg, 1.0, f, window="dirichlet")
    assert O.rel_l2(b, a) < 1e-9


def test_dirichlet_alg1_full_support_exact():
    """m = M_sigma/2 and N <= M - 1: K B^* = M I_N is attainable although D^* drops k = -M/2,
    so (1/M) B_opt F D h recovers f from h = A^* f."""
    M, N = 8, 6
    x = S.jittered(N, 9)
    w, _ = O.alg1_setup(x, M, 2.0, 8, window="dirichlet")
    f = S.normal_complex(3, N, 1)
    h = O.ndft_adjoint(x, f, M)
    assert O.rel_l2(O.apply_adjoint(x, M, 2.0, 8, w, 1.0 / M, h, window="dirichlet"), f) < 1e-12
    assert O.objective_alg1(x, M, 2.0, 8, w, window="dirichlet") < 1e-10


def test_dirichlet_fast_equals_dense_literal():
    M, sigma, m = 16, 2.0, 3
    x = S.jittered(24, 6)
    w = np.random.default_rng(1).standard_normal((24, 2 * m + 1)) * O.slot_live(x, O.msigma(M, sigma), m)
    f = S.normal_complex(2, 24, 2)
    h = S.normal_complex(2, M, 3)
    assert O.rel_l2(O.apply_inverse(x, M, sigma, m, w, 1.0, f, window="dirichlet"),
                    O.dense_inverse(x, M, sigma, m, w, 1.0, f, window="dirichlet")) < 1e-13
    assert O.rel_l2(O.apply_adjoint(x, M, sigma, m, w, 1.0, h, window="dirichlet"),
                    O.dense_adjoint(x, M, sigma, m, w, 1.0, h, window="dirichlet")) < 1e-13

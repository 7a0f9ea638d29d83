"""Pins of the oracle's B-spline window (reading A24; the window of the paper's experiments,
P:987) against textbook facts: closed values of M_2, M_4;
partition of unity; unit integral; the Fourier transform sinc^{2m} checked by Gauss-Legendre
quadrature (exact on each polynomial piece); and the ordinary NFFT with this window against
the NDFT, with the error falling in m."""
import numpy as np
import pytest

import oracle as O
import synth as S


def test_closed_values():
    v = np.linspace(-1.5, 1.5, 31)
    assert np.allclose(O.bspline_centred(v, 2), np.clip(1 - np.abs(v), 0, None), atol=1e-15)
    assert abs(O.bspline_centred(0.0, 4) - 2.0 / 3.0) < 1e-15
    assert abs(O.bspline_centred(1.0, 4) - 1.0 / 6.0) < 1e-15
    assert O.bspline_centred(2.0, 4) == 0.0


@pytest.mark.parametrize("n", [2, 4, 8, 16, 24])
def test_partition_of_unity_and_symmetry(n):
    v = np.random.default_rng(n).random(50) - 0.5
    tot = sum(O.bspline_centred(v - l, n) for l in range(-n, n + 1))
    assert np.abs(tot - 1.0).max() < 1e-13
    assert np.abs(O.bspline_centred(v, n) - O.bspline_centred(-v, n)).max() < 1e-14


@pytest.mark.parametrize("m", [1, 2, 4, 6])
def test_fourier_transform_by_quadrature(m):
    """what(k) = int w(x) e^{-2 pi i k x} dx: w = M_2m(Msig x) is a polynomial of degree 2m-1 on
    each cell [j, j+1]/Msig, so Gauss-Legendre with 2m + 8 points per cell integrates the
    product with the exponential to rounding (the exponential is smooth on a cell)."""
    Ms = 64
    g, wq = np.polynomial.legendre.leggauss(2 * m + 24)
    ks = np.array([0, 1, 5, 16, 31])
    tot = np.zeros(ks.size, dtype=np.complex128)
    for j in range(-m, m):
        x = (j + 0.5 + 0.5 * g) / Ms
        tot += (O.bspline_w(x, Ms, m) * wq * 0.5 / Ms) @ np.exp(-2j * np.pi * np.outer(x, ks))
    ref = O.bspline_what(ks, Ms, m)
    assert np.abs(tot - ref).max() < 1e-14 * max(1.0, np.abs(ref).max() * Ms) / Ms
    assert abs(tot[0] * 1.0 - 1.0 / Ms) < 1e-15  # unit integral of M_2m (what(0) = 1/Ms)


def test_plain_nfft_bspline_accuracy_falls_in_m():
    """Ordinary NFFT (B F D with the B-spline window, eqs. matrix_B/F/D) vs the NDFT: the error
    falls with m like (2 sigma - 1)^{-2m}."""
    M, sigma, N = 64, 2.0, 100
    x = S.jittered(N, 3)
    fh = S.normal_complex(2, M, 4)
    ref = O.ndft(x, fh, M)
    errs = []
    for m in (2, 4, 6, 8):
        w = O.window_slot_weights(x, M, sigma, m, window="bspline")
        got = O.dense_adjoint(x, M, sigma, m, w, 1.0, fh, window="bspline")
        errs.append(O.rel_l2(got, ref))
    assert all(a > 2 * b for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 3.0 ** (-16) * 1e3, errs

"""Pins of the oracle's quadratic case (oracle/quadratic.py, SURVEY
8(f) NEXT-3) against what the mathematics fixes -- never against a retyped formula:
the Lagrange relation is exact for trigonometric polynomials of degree N (duro95 Thm 2.3,
P:369-372), so the inverse must return fhat from f = A fhat (A = the NDFT matrix, eq.
matrix_A) and the adjoint must return f from h = A^* f; the stabilised coefficients must
equal the plain products of sines; the shift must balance the exponents."""
import numpy as np
import pytest

import oracle as O
from oracle import quadratic as Q
import synth as S


@pytest.mark.parametrize("N", [2, 4, 8, 16, 32, 64, 128])
def test_inverse_recovers_fhat(N):
    y = S.jittered(N, N)
    fhat = S.normal_complex(3, N, N + 1)
    f = O.ndft(y, fhat, N)
    assert O.rel_l2(Q.inverse(y, f), fhat) < 1e-11


@pytest.mark.parametrize("N", [2, 8, 32, 128])
def test_adjoint_recovers_f(N):
    y = S.jittered(N, 3 * N)
    f = S.normal_complex(2, N, N + 5)
    h = O.ndft_adjoint(y, f, N)
    assert O.rel_l2(Q.adjoint(y, h), f) < 1e-11


def test_iid_nodes_and_other_offsets():
    """iid nodes (less regular than jittered) and a target offset other than the midpoint:
    the recovery is exact either way (any equispaced targets disjoint from y)."""
    N = 24
    y = np.sort(np.random.default_rng(5).random(N) - 0.5)
    fhat = S.normal_complex(2, N, 9)
    f = O.ndft(y, fhat, N)
    for delta in (None, 0.3 / N, 0.9 / N):
        assert O.rel_l2(Q.inverse(y, f, delta), fhat) < 1e-8


def test_stabilized_product_equals_direct_product():
    N = 20
    y = S.jittered(N, 7)
    x, a, b, s = Q.coeffs(y)
    a_direct = np.array([np.prod(np.sin(np.pi * (xl - y))) for xl in x])
    b_direct = np.array([np.prod([1.0 / np.sin(np.pi * (y[j] - y[n])) for n in range(N) if n != j])
                         for j in range(N)])
    assert np.allclose(np.outer(a, b), np.outer(a_direct, b_direct), rtol=1e-12, atol=0)
    assert s != 0.0 or np.isclose(np.abs(a).max(), np.abs(b).max())


def test_stabilization_shift_balances():
    assert Q.stabilization_shift(np.full(4, -100.0), np.full(5, 100.0)) == 100.0
    assert Q.stabilization_shift(np.array([1.0, 3.0]), np.array([1.0, 3.0])) == 0.0
    y = S.jittered(64, 2)
    x, a, b, _ = Q.coeffs(y)
    assert np.isclose(np.log(np.abs(a)).max(), np.log(np.abs(b)).max())


def test_constant_polynomial():
    N = 16
    y = S.jittered(N, 4)
    fc = Q.inverse(y, np.full((1, N), 2.5 - 1.0j))
    e0 = np.zeros(N, dtype=np.complex128)
    e0[N // 2] = 2.5 - 1.0j
    assert np.abs(fc[0] - e0).max() < 1e-12

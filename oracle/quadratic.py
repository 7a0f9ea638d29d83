"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The quadratic case M = N of the paper (Section "The quadratic case", and the
adjoint Remark P:576-584), written from the paper with plain direct
sums in float64:

  a_l = prod_n sin(pi (x_l - y_n)),  b_j = prod_{n != j} 1 / sin(pi (y_j - y_n))   (eq. coeff_ab)
  g_l = a_l sum_j f_j b_j (cot(pi (x_l - y_j)) - i)                                (eq. lagrange_formula)
  fcheck_k = (1/N) sum_l g_l e^{-2 pi i k x_l},  k = -N/2..N/2-1                  (Alg. step 6)
  adjoint: v = (1/N) E h, f_j = b_j sum_l a_l v_l (cot(pi (x_l - y_j)) + i)        (eq. lagrange_formula_adjoint)

with the log-domain magnitudes atilde = ln|a|, btilde = ln|b|, a stabilisation
shift s (Remark P:431-449: the rule there names undefined symbols; reading A22 = SPEC's
max-balancing shift s = (max btilde - max atilde) / 2) and the signs counted directly.  The
equispaced targets are x_l = -1/2 + l/N + delta (P:374-376 leaves the offset free; reading
A23: delta = 1/(2N), the midpoints).  Everything is O(N^2) direct summation -- the paper's
fast summation is an acceleration of exactly these sums.
"""
import numpy as np


def targets(N, delta=None):
    """Equispaced x_l = -1/2 + l/N + delta, l = 0..N-1 (reading A23: delta = 1/(2N))."""
    if delta is None:
        delta = 0.5 / N
    return -0.5 + np.arange(N) / N + delta


def log_coeffs(y, x):
    """(atilde, sign_a, btilde, sign_b): atilde_l = sum_n ln|sin(pi(x_l - y_n))|,
    btilde_j = -sum_{n != j} ln|sin(pi(y_j - y_n))|, and the signs of the
    products, each factor's sign taken directly."""
    y = np.asarray(y, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    sa = np.sin(np.pi * (x[:, None] - y[None, :]))
    atil = np.log(np.abs(sa)).sum(axis=1)
    sign_a = np.prod(np.sign(sa), axis=1)
    sb = np.sin(np.pi * (y[:, None] - y[None, :]))
    np.fill_diagonal(sb, 1.0)
    btil = -np.log(np.abs(sb)).sum(axis=1)
    sign_b = np.prod(np.sign(sb), axis=1)
    return atil, sign_a, btil, sign_b


def stabilization_shift(atil, btil):
    """Reading A22: s = (max_j btilde_j - max_l atilde_l) / 2, so that the largest exponents
    of e^{atilde + s} and e^{btilde - s} are equal (Remark P:431-449)."""
    return 0.5 * (np.max(btil) - np.max(atil))


def coeffs(y, delta=None):
    """Signed, stabilised a_l = sign_a e^{atilde_l + s}, b_j = sign_b e^{btilde_j - s}
    (Alg. steps 1-3); returns (x, a, b, s)."""
    y = np.asarray(y, dtype=np.float64)
    x = targets(y.size, delta)
    atil, sa, btil, sb = log_coeffs(y, x)
    s = stabilization_shift(atil, btil)
    return x, sa * np.exp(atil + s), sb * np.exp(btil - s), s


def inverse(y, f, delta=None):
    """Alg. "Fast inverse NFFT - quadratic case" by direct sums: f [R][N] samples
    at the nodes y -> fcheck [R][N], k = -N/2..N/2-1."""
    y = np.asarray(y, dtype=np.float64)
    f = np.atleast_2d(np.asarray(f, dtype=np.complex128))
    N = y.size
    x, a, b, _ = coeffs(y, delta)
    C = 1.0 / np.tan(np.pi * (x[:, None] - y[None, :]))  # cot(pi (x_l - y_j))
    fb = f * b[None, :]
    gt = fb @ C.T                                        # eq. coeff_g_tilde
    g = a[None, :] * (gt - 1j * fb.sum(axis=1, keepdims=True))  # eq. coeff_g
    k = np.arange(-N // 2, N // 2)
    E = np.exp(-2j * np.pi * np.outer(x, k))             # e^{-2 pi i k x_l}
    return (g @ E) / N                                   # Alg. step 6


def adjoint(y, h, delta=None):
    """Inverse adjoint (Remark P:576-584) by direct sums: h [R][N] (k = -N/2..N/2-1) ->
    f [R][N] with v = (1/N) sum_k h_k e^{2 pi i k x_l} (the adjoint of step 6)."""
    y = np.asarray(y, dtype=np.float64)
    h = np.atleast_2d(np.asarray(h, dtype=np.complex128))
    N = y.size
    x, a, b, _ = coeffs(y, delta)
    k = np.arange(-N // 2, N // 2)
    v = (h @ np.exp(2j * np.pi * np.outer(k, x))) / N
    C = 1.0 / np.tan(np.pi * (x[:, None] - y[None, :]))
    av = v * a[None, :]
    return b[None, :] * (av @ C + 1j * av.sum(axis=1, keepdims=True))

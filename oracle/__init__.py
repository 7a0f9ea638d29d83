"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what Kircheis & Potts'
direct inverse NFFT (arXiv:1811.05335) computes, written from the paper.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It shares no code with the CUDA path
(``paper_1811_05335_b200/csrc``) and never imports it; neither side calls the
other.  Citations: ``P:<n>`` = /root/reference/PAPER.md line n.

Parts (each pinned by tests/test_oracle_*.py against something other than
itself):

* window pair (Kaiser-Bessel, reading A7), deconvolution D (eq. matrix_D)
* index sets I(x_j) (eq. set_xj) and I(l) (eq. set_l),
  slot layout l0_j = ceil(M_sigma x_j) - m, node bins / stable permutation
* dense matrices A, D, F, B (eqs. matrix_A, matrix_D, matrix_F, matrix_B) and
  the dense-literal inversions  s D^* F^* B^* f  and  s B F D h
* NDFT  f = A fhat, h = A^* f  (eqs. nfft, nfft*)
* Alg. "Fast optimization of the matrix B" and
  Alg. "Fast optimization of the matrix B*" as per-column least
  squares solved by SVD / eigendecomposition with the min-norm cutoff
  (reading A6)
* the fast apply (spread -> DFT -> truncate/deconvolve and its dual) in plain
  C (oracle/inft_oracle.c) for speed; pinned against the dense-literal path.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

TAU_DEFAULT = 1e-6  # relative singular-value cutoff (reading A6)


# =============================================================== window (A7)
def i0(x):
    """Modified Bessel function I_0 by its power series sum_k (x/2)^{2k}/(k!)^2
    (all terms positive: no cancellation).  Pinned against scipy.special.i0."""
    x = np.asarray(x, dtype=np.float64)
    q = (x * 0.5) ** 2
    term = np.ones_like(x)
    total = np.ones_like(x)
    k = 1
    while True:
        term = term * q / (k * k)
        total = total + term
        if np.all(term <= 1e-18 * total):
            break
        k += 1
    return total


def kb_b(sigma):
    """Kaiser-Bessel shape parameter b = pi (2 - 1/sigma) (reading A7)."""
    return np.pi * (2.0 - 1.0 / sigma)


def kb_what(k, Msig, m, sigma):
    """KB Fourier coefficients what(k) = (1/M_sigma) I0(m sqrt(b^2 - (2 pi k/M_sigma)^2))
    for |2 pi k / M_sigma| <= b (always true for |k| <= M/2, sigma >= 1).
    This is c_k(w~) of eq. (fourier_transform) P:158-167 for the KB window."""
    k = np.asarray(k, dtype=np.float64)
    b = kb_b(sigma)
    arg = b * b - (2.0 * np.pi * k / Msig) ** 2
    if np.any(arg < 0):
        raise ValueError("KB what(k) requested outside |2 pi k/M_sigma| <= b")
    return i0(m * np.sqrt(arg)) / Msig


def kb_w(x, Msig, m, sigma):
    """Truncated KB window w_m(x) = chi_[-m/Msig, m/Msig] w(x) with
    w(x) = (1/pi) sinh(b sqrt(m^2 - Msig^2 x^2)) / sqrt(m^2 - Msig^2 x^2)
    (limit b/pi where the root vanishes)."""
    x = np.asarray(x, dtype=np.float64)
    b = kb_b(sigma)
    r2 = m * m - (Msig * x) ** 2
    out = np.zeros_like(x)
    inside = np.abs(x) <= m / Msig
    root = np.sqrt(np.where(inside & (r2 > 0), r2, 1.0))
    val = np.where(r2 > 0, np.sinh(b * root) / root, b) / np.pi
    out[inside] = val[inside]
    return out


def kb_w_periodic(x, Msig, m, sigma):
    """1-periodic w~_m(x) = sum_z w_m(x + z); |x| < 1 suffices z in {-1,0,1}."""
    x = np.asarray(x, dtype=np.float64)
    return kb_w(x - 1.0, Msig, m, sigma) + kb_w(x, Msig, m, sigma) + kb_w(x + 1.0, Msig, m, sigma)


def msigma(M, sigma):
    """M_sigma = sigma M; must be an even integer (DESIGN.md plan validation)."""
    v = sigma * M
    iv = int(round(v))
    if abs(v - iv) > 1e-9 or iv % 2:
        raise ValueError("sigma*M must be an even integer")
    return iv


def bspline_centred(v, n):
    """Centred cardinal B-spline M_n (support [-n/2, n/2], integral 1) by the recursion
    M_1 = chi_[-1/2, 1/2),  M_n(v) = ((n/2 + v) M_{n-1}(v + 1/2) + (n/2 - v) M_{n-1}(v - 1/2)) / (n - 1)."""
    v = np.asarray(v, dtype=np.float64)
    # level k holds M_k at the offsets v + j - (n - k)/2, j = 0..n-k (the ones M_n(v) needs)
    off = [v + (j - 0.5 * (n - 1)) for j in range(n)]
    cur = [((o >= -0.5) & (o < 0.5)).astype(np.float64) for o in off]
    for k in range(2, n + 1):
        off = [v + (j - 0.5 * (n - k)) for j in range(n - k + 1)]
        cur = [((0.5 * k + off[j]) * cur[j + 1] + (0.5 * k - off[j]) * cur[j]) / (k - 1) for j in range(n - k + 1)]
    return cur[0]


def bspline_w(x, Msig, m):
    """B-spline window of the paper's experiments (reading A24):
    w(x) = M_2m(M_sigma x), support [-m/M_sigma, m/M_sigma] (no truncation)."""
    return bspline_centred(Msig * np.asarray(x, dtype=np.float64), 2 * m)


def bspline_what(k, Msig, m):
    """what(k) = int w(x) e^{-2 pi i k x} dx = (1/M_sigma) sinc(pi k/M_sigma)^{2m} (the B-spline's
    Fourier transform; pinned by quadrature in tests/test_oracle_bspline.py)."""
    k = np.asarray(k, dtype=np.float64)
    return np.sinc(k / Msig) ** (2 * m) / Msig


def window_hat_vector(M, sigma, m, window="kb"):
    """what(k) for k = -M/2..M/2-1 (centered): Kaiser-Bessel (A7) or B-spline (A24)."""
    Ms = msigma(M, sigma)
    k = np.arange(-M // 2, M // 2)
    if window == "bspline":
        return bspline_what(k, Ms, m)
    return kb_what(k, Ms, m, sigma)


def inv_what_vector(M, sigma, m, window="kb"):
    """1/what(k) for k = -M/2..M/2-1 (centered).
    window='kb': the Kaiser-Bessel window (reading A7).
    window='dirichlet': the Dirichlet-kernel variant of Remarks P:934-957 and P:1343-1358:
    what(k) = 1 for k = -M/2+1..M/2-1 and the entry of D^* at the unpaired frequency set to
    zero (the text names it 1/what(M/2); in the centred range -M/2..M/2-1 it is k = -M/2,
    reading A21)."""
    if window in ("kb", "bspline"):
        return 1.0 / window_hat_vector(M, sigma, m, window)
    if window == "dirichlet":
        v = np.ones(M)
        v[0] = 0.0
        return v
    raise ValueError(f"unknown window {window!r}")


def dirichlet_kernel(x, M):
    """D_{M/2-1}(x) = sin((M-1) pi x) / sin(pi x), eq. kernel_Dirichlet P:937-944 (closed form;
    the limit M-1 at integer x)."""
    x = np.asarray(x, dtype=np.float64)
    sx = np.sin(np.pi * x)
    with np.errstate(divide="ignore", invalid="ignore"):
        v = np.sin((M - 1) * np.pi * x) / sx
    return np.where(np.abs(sx) < 1e-300, float(M - 1), v)


def deconv_vector(M, sigma, m, s=1.0, window="kb"):
    """d_k = s / (M_sigma what(k)) -- the diagonal of D (eq. matrix_D)
    with the apply scale s folded in (reading A2)."""
    Ms = msigma(M, sigma)
    if window in ("kb", "bspline"):
        return s / (Ms * window_hat_vector(M, sigma, m, window))
    return s * inv_what_vector(M, sigma, m, window) / Ms


# ============================================================= index sets
def node_base(x, Msig, m):
    """l0_j = ceil(M_sigma x_j) - m: lowest grid index of the sum in P:195.
    M_sigma * x_j is one correctly rounded multiply (reading A20)."""
    x = np.asarray(x, dtype=np.float64)
    return (np.ceil(np.float64(Msig) * x) - m).astype(np.int64)


def index_set_node_bruteforce(x, Msig, m):
    """I_{Msig,m}(x) of eq. (set_xj) P:768-774 by enumeration of every
    l in {-Msig/2..Msig/2-1} and z in {-1, 0, 1}."""
    out = []
    for l in range(-Msig // 2, Msig // 2):
        for z in (-1, 0, 1):
            v = Msig * x - l + Msig * z
            if -m <= v <= m:
                out.append(l)
                break
    return out


def slot_live(x, Msig, m):
    """Boolean [N][2m+1]: slot t of node j (grid l0_j + t) is a distinct member
    of I(x_j).  Slot t is in the support iff |M_sigma x_j - (l0_j + t)| <= m
    (P:765); an aliased repeat of an earlier live slot (only possible when
    2m+1 > M_sigma) is not live (reading A5)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    P = 2 * m + 1
    l0 = node_base(x, Msig, m)
    t = np.arange(P)
    v = np.float64(Msig) * x[:, None] - (l0[:, None] + t[None, :])
    live = (v >= -m) & (v <= m)
    if P > Msig:
        for j in range(x.size):
            seen = set()
            for tt in range(P):
                if live[j, tt]:
                    n = (l0[j] + tt) % Msig
                    if n in seen:
                        live[j, tt] = False
                    else:
                        seen.add(n)
    return live


def bins_1d(x, Msig, m, T):
    """Plan integers: l0, n0 = l0 mod M_sigma, bin = n0 // T and
    perm = stable sort of j by (n0_j, j) (reading A19; sorting by n0 also sorts
    by bin, and keeps increasing node sets a cyclic shift of the caller order)."""
    l0 = node_base(x, Msig, m)
    n0 = np.mod(l0, Msig)
    b = n0 // T
    perm = np.argsort(n0, kind="stable")
    return l0, n0, b, perm


def grid_node_sets(x, Msig, m):
    """I_{Msig,m}(l) of eq. (set_l) P:1212-1218 for every grid point n = l mod Msig:
    list of (j, t) with live slot t of node j on n."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    l0 = node_base(x, Msig, m)
    live = slot_live(x, Msig, m)
    sets = [[] for _ in range(Msig)]
    for j in range(x.size):
        for t in np.nonzero(live[j])[0]:
            sets[(l0[j] + t) % Msig].append((j, int(t)))
    return sets


# ========================================================= dense matrices
def matrix_A(x, M):
    """A = (e^{2 pi i k x_j})_{j, k=-M/2..M/2-1} (eq. matrix_A).
    2-D (reading A12): x [N][2], M = (M1, M2), k flattened row-major."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        k = np.arange(-M // 2, M // 2)
        return np.exp(2j * np.pi * np.outer(x, k))
    M1, M2 = M
    k1 = np.arange(-M1 // 2, M1 // 2)
    k2 = np.arange(-M2 // 2, M2 // 2)
    A1 = np.exp(2j * np.pi * np.outer(x[:, 0], k1))
    A2 = np.exp(2j * np.pi * np.outer(x[:, 1], k2))
    return (A1[:, :, None] * A2[:, None, :]).reshape(x.shape[0], M1 * M2)


def matrix_F(M, Msig):
    """F = (e^{2 pi i k l / M_sigma})_{l=-Msig/2..Msig/2-1, k=-M/2..M/2-1} (eq. matrix_F)."""
    l = np.arange(-Msig // 2, Msig // 2)
    k = np.arange(-M // 2, M // 2)
    return np.exp(2j * np.pi * np.outer(l, k) / Msig)


def _w_periodic(x, Ms, m, sigma, window):
    if window == "bspline":
        x = np.asarray(x, dtype=np.float64)
        return bspline_w(x - 1.0, Ms, m) + bspline_w(x, Ms, m) + bspline_w(x + 1.0, Ms, m)
    return kb_w_periodic(x, Ms, m, sigma)


def matrix_B_window(x, M, sigma, m, window="kb"):
    """Window matrix B = (w~_m(x_j - l/M_sigma))_{j, l} (eq. matrix_B)."""
    Ms = msigma(M, sigma)
    l = np.arange(-Ms // 2, Ms // 2)
    return _w_periodic(np.asarray(x)[:, None] - l[None, :] / Ms, Ms, m, sigma, window)


def window_slot_weights(x, M, sigma, m, window="kb"):
    """Slot weights of the window matrix B: w[j][t] = w~_m(x_j - (l0_j+t)/M_sigma)
    on live slots (ordinary NFFT, the INFT_PLAIN_NFFT method)."""
    Ms = msigma(M, sigma)
    x = np.asarray(x, dtype=np.float64)
    l0 = node_base(x, Ms, m)
    t = np.arange(2 * m + 1)
    w = _w_periodic(x[:, None] - (l0[:, None] + t[None, :]) / Ms, Ms, m, sigma, window)
    return np.where(slot_live(x, Ms, m), w, 0.0)


def window_slot_weights_2d(x, M, sigma, m):
    """Tensor-product window slot weights (reading A12): w[j][t1*P+t2] =
    w~_m(x_j1 - l1/Msig1) w~_m(x_j2 - l2/Msig2) on live slot pairs."""
    x = np.asarray(x, dtype=np.float64)
    w1 = window_slot_weights(x[:, 0], M[0], sigma, m)
    w2 = window_slot_weights(x[:, 1], M[1], sigma, m)
    return (w1[:, :, None] * w2[:, None, :]).reshape(x.shape[0], -1)


def dense_from_slots(w, l0, Msig):
    """Dense N x M_sigma matrix with columns l = -Msig/2..Msig/2-1 from slot
    weights: B[j, l] = sum_{t: l0_j + t = l mod Msig} w[j][t]."""
    w = np.asarray(w)
    N, P = w.shape
    B = np.zeros((N, Msig), dtype=w.dtype)
    for t in range(P):
        col = np.mod(l0 + t + Msig // 2, Msig)
        np.add.at(B, (np.arange(N), col), w[:, t])
    return B


def dense_from_slots_2d(w, l0, Msig, P):
    """2-D: B[j, (l1, l2)] row-major over l_i = -Msig_i/2..Msig_i/2-1."""
    w = np.asarray(w)
    N = w.shape[0]
    S1, S2 = Msig
    P1, P2 = P
    B = np.zeros((N, S1 * S2), dtype=w.dtype)
    for t1 in range(P1):
        c1 = np.mod(l0[:, 0] + t1 + S1 // 2, S1)
        for t2 in range(P2):
            c2 = np.mod(l0[:, 1] + t2 + S2 // 2, S2)
            np.add.at(B, (np.arange(N), c1 * S2 + c2), w[:, t1 * P2 + t2])
    return B


def dense_inverse(x, M, sigma, m, w, s, f, window="kb"):
    """Dense-literal inverse NFFT  s D^* F^* B_opt^* f  (P:631 / P:1279), f [R][N]."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        Ms = msigma(M, sigma)
        B = dense_from_slots(w, node_base(x, Ms, m), Ms)
        D = np.diag(deconv_vector(M, sigma, m, 1.0, window))
        F = matrix_F(M, Ms)
    else:
        B, D, F = _dense_2d_factors(x, M, sigma, m, w, window)
    return (s * D.conj() @ F.conj().T @ B.conj().T @ np.asarray(f).T).T


def dense_adjoint(x, M, sigma, m, w, s, h, window="kb"):
    """Dense-literal inverse adjoint NFFT  s B_opt F D h  (P:1116 / P:1522), h [R][M]."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        Ms = msigma(M, sigma)
        B = dense_from_slots(w, node_base(x, Ms, m), Ms)
        D = np.diag(deconv_vector(M, sigma, m, 1.0, window))
        F = matrix_F(M, Ms)
    else:
        B, D, F = _dense_2d_factors(x, M, sigma, m, w, window)
    return (s * B @ F @ D @ np.asarray(h).T).T


def _dense_2d_factors(x, M, sigma, m, w, window="kb"):
    M1, M2 = M
    S = (msigma(M1, sigma), msigma(M2, sigma))
    l0 = np.stack([node_base(x[:, 0], S[0], m), node_base(x[:, 1], S[1], m)], axis=1)
    B = dense_from_slots_2d(w, l0, S, (2 * m + 1, 2 * m + 1))
    D = np.diag(np.kron(deconv_vector(M1, sigma, m, 1.0, window), deconv_vector(M2, sigma, m, 1.0, window)))
    F = np.kron(matrix_F(M1, S[0]), matrix_F(M2, S[1]))
    return B, D, F


# ================================================================= NDFT
def ndft(x, fhat, M):
    """f = A fhat by direct sums (eq. nfft); fhat [R][prod M]."""
    A = matrix_A(x, M)
    return (A @ np.asarray(fhat).T).T


def ndft_adjoint(x, f, M):
    """h = A^* f by direct sums (eq. nfft* P:42-45); f [R][N]."""
    A = matrix_A(x, M)
    return (A.conj().T @ np.asarray(f).T).T


# ===================================================== least squares (A6)
def lstsq_minnorm_svd(Lmat, e, tau=TAU_DEFAULT, real=True):
    """min ||L b - e||_2, minimum norm, singular values below tau*s_max dropped.
    real=True constrains b to R^n (P:1248 'b in R^{2m+1}') by stacking
    [Re L; Im L] b = [Re e; Im e]."""
    if real:
        A = np.vstack([Lmat.real, Lmat.imag])
        rhs = np.concatenate([np.real(e), np.imag(e)])
    else:
        A = Lmat
        rhs = e
    if A.shape[1] == 0:
        return np.zeros(0, dtype=A.dtype), 0
    U, sv, Vh = np.linalg.svd(A, full_matrices=False)
    keep = sv > tau * sv[0] if sv[0] > 0 else np.zeros_like(sv, dtype=bool)
    coef = (U[:, keep].conj().T @ rhs) / sv[keep]
    b = Vh[keep].conj().T @ coef
    return b, int(A.shape[1] - keep.sum())


def solve_minnorm_gram(G, y, tau=TAU_DEFAULT):
    """Same minimiser from the normal equations G b = y (G = Re(L^*L) PSD):
    eigendecomposition, eigenvalues below tau^2 * lambda_max dropped (the Gram
    form squares the singular values)."""
    n = G.shape[0]
    if n == 0:
        return np.zeros(0), 0
    lam, V = np.linalg.eigh(G)
    lmax = lam[-1]
    keep = lam > (tau * tau) * lmax if lmax > 0 else np.zeros(n, dtype=bool)
    b = V[:, keep] @ ((V[:, keep].T @ y) / lam[keep])
    return b, int(n - keep.sum())


# ------------------------------------------------ Alg. 2 ingredients
def L_explicit(l, xs, M, sigma, m, window="kb"):
    """L_l = F D H_l (eq. matrix_Ll) for the nodes xs = {x_j : j in I(l)}:
    H_l = (e^{-2 pi i k x_j})_{k, j}; returns [M_sigma][|I(l)|]; row s <-> s - Msig/2."""
    Ms = msigma(M, sigma)
    k = np.arange(-M // 2, M // 2)
    H = np.exp(-2j * np.pi * np.outer(k, np.asarray(xs)))
    D = deconv_vector(M, sigma, m, 1.0, window)
    return matrix_F(M, Ms) @ (D[:, None] * H)


def G_kernel(dx, M, sigma, m, window="kb"):
    """G(x) = (1/M_sigma) sum_k e^{2 pi i k x} / what(k)^2 (complex), direct sum.
    (L_l^* L_l)_{jj'} = G(x_j - x_j') by F^*F = M_sigma I_M (Gram form)."""
    Ms = msigma(M, sigma)
    k = np.arange(-M // 2, M // 2)
    c = (1.0 / window_hat_vector(M, sigma, m) ** 2 / Ms if window == "kb"
         else inv_what_vector(M, sigma, m, window) ** 2 / Ms)
    dx = np.asarray(dx, dtype=np.float64)
    return np.exp(2j * np.pi * dx[..., None] * k) @ c


def Kplus_kernel(dx, M, sigma, m, window="kb"):
    """K+(x) = (1/M_sigma) sum_k e^{2 pi i k x} / what(k): (L_l^* e_l)_j = K+(x_j - l/M_sigma)."""
    Ms = msigma(M, sigma)
    k = np.arange(-M // 2, M // 2)
    c = (1.0 / window_hat_vector(M, sigma, m) / Ms if window == "kb"
         else inv_what_vector(M, sigma, m, window) / Ms)
    dx = np.asarray(dx, dtype=np.float64)
    return np.exp(2j * np.pi * dx[..., None] * k) @ c


def wrap_diff(a):
    """Reduce a real difference to [-1/2, 1/2) (kernels are 1-periodic)."""
    a = np.asarray(a, dtype=np.float64)
    return a - np.floor(a + 0.5)


def alg2_setup(x, M, sigma, m, tau=TAU_DEFAULT, form="explicit", columns=None, weights="real", window="kb"):
    """Alg. "Fast optimization of the matrix B", per grid point l:
    J = I_{Msig,m}(l) (eq. set_l), minimise ||L_l b - e_l|| with the
    minimum-norm cutoff (A6); store B_opt[j, l] = b_j as slot weight.

    form='explicit': L_l formed densely from its definition (small sizes).
    form='gram': normal equations from G, K+ (no M_sigma-row matrix; large sizes).
    Returns (w [N][2m+1], info dict)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 2:
        return _alg2_setup_2d(x, M, sigma, m, tau, form, columns, weights, window)
    Ms = msigma(M, sigma)
    N = x.size
    P = 2 * m + 1
    sets = grid_node_sets(x, Ms, m)
    cplx = weights == "complex"
    w = np.zeros((N, P), dtype=np.complex128 if cplx else np.float64)
    cols = range(Ms) if columns is None else columns
    rank_def = 0
    max_col = 0
    resid = {}
    for n in cols:
        js = [j for (j, t) in sets[n]]
        ts = [t for (j, t) in sets[n]]
        max_col = max(max_col, len(js))
        if not js:
            resid[n] = 1.0
            continue
        l = n - Ms if n >= Ms // 2 else n  # grid index in [-Msig/2, Msig/2)
        if form == "explicit":
            Lm = L_explicit(l, x[js], M, sigma, m, window)
            e = np.zeros(Ms, dtype=np.complex128)
            e[l + Ms // 2] = 1.0
            b, nd = lstsq_minnorm_svd(Lm, e, tau, real=not cplx)
            resid[n] = float(np.linalg.norm(Lm @ b - e))
        else:
            if cplx:
                raise NotImplementedError("complex weights use the explicit form in the oracle")
            dx = wrap_diff(x[js][:, None] - x[js][None, :])
            G = np.real(G_kernel(dx, M, sigma, m, window))
            y = np.real(Kplus_kernel(wrap_diff(x[js] - l / Ms), M, sigma, m, window))
            b, nd = solve_minnorm_gram(G, y, tau)
            # ||L b - e||^2 = b^T G b - 2 b^T y + 1 for real b
            resid[n] = float(np.sqrt(max(b @ G @ b - 2 * b @ y + 1.0, 0.0)))
        rank_def += nd > 0
        w[js, ts] = b
    return w, dict(n_rank_deficient=rank_def, max_col_size=max_col, resid=resid)


def _alg2_setup_2d(x, M, sigma, m, tau, form, columns, weights, window="kb"):
    """Tensor-product reading A12 of Alg. 2: I(x_j) = I1 x I2, grid l = (l1, l2)."""
    M1, M2 = M
    S1, S2 = msigma(M1, sigma), msigma(M2, sigma)
    N = x.shape[0]
    P1 = 2 * m + 1
    l0 = np.stack([node_base(x[:, 0], S1, m), node_base(x[:, 1], S2, m)], axis=1)
    live1 = slot_live(x[:, 0], S1, m)
    live2 = slot_live(x[:, 1], S2, m)
    sets = {}
    for j in range(N):
        for t1 in np.nonzero(live1[j])[0]:
            n1 = (l0[j, 0] + t1) % S1
            for t2 in np.nonzero(live2[j])[0]:
                n2 = (l0[j, 1] + t2) % S2
                sets.setdefault(n1 * S2 + n2, []).append((j, int(t1) * P1 + int(t2)))
    w = np.zeros((N, P1 * P1))
    cols = range(S1 * S2) if columns is None else columns
    k1 = np.arange(-M1 // 2, M1 // 2)
    k2 = np.arange(-M2 // 2, M2 // 2)
    D1 = deconv_vector(M1, sigma, m, 1.0, window)
    D2 = deconv_vector(M2, sigma, m, 1.0, window)
    rank_def = 0
    max_col = 0
    resid = {}
    for n in cols:
        lst = sets.get(n, [])
        max_col = max(max_col, len(lst))
        if not lst:
            resid[n] = 1.0
            continue
        js = [j for (j, t) in lst]
        ts = [t for (j, t) in lst]
        n1, n2 = divmod(n, S2)
        l1 = n1 - S1 if n1 >= S1 // 2 else n1
        l2 = n2 - S2 if n2 >= S2 // 2 else n2
        if form == "explicit":
            H = (np.exp(-2j * np.pi * np.outer(k1, x[js, 0]))[:, None, :] *
                 np.exp(-2j * np.pi * np.outer(k2, x[js, 1]))[None, :, :]).reshape(M1 * M2, len(js))
            Dk = np.kron(D1, D2)
            Lm = np.kron(matrix_F(M1, S1), matrix_F(M2, S2)) @ (Dk[:, None] * H)
            e = np.zeros(S1 * S2, dtype=np.complex128)
            e[(l1 + S1 // 2) * S2 + (l2 + S2 // 2)] = 1.0
            b, nd = lstsq_minnorm_svd(Lm, e, tau, real=True)
            resid[n] = float(np.linalg.norm(Lm @ b - e))
        else:
            xs = x[js]
            g1 = G_kernel(wrap_diff(xs[:, None, 0] - xs[None, :, 0]), M1, sigma, m, window)
            g2 = G_kernel(wrap_diff(xs[:, None, 1] - xs[None, :, 1]), M2, sigma, m, window)
            G = np.real(g1 * g2)
            y = np.real(Kplus_kernel(wrap_diff(xs[:, 0] - l1 / S1), M1, sigma, m, window) *
                        Kplus_kernel(wrap_diff(xs[:, 1] - l2 / S2), M2, sigma, m, window))
            b, nd = solve_minnorm_gram(G, y, tau)
            resid[n] = float(np.sqrt(max(b @ G @ b - 2 * b @ y + 1.0, 0.0)))
        rank_def += nd > 0
        w[js, ts] = b
    return w, dict(n_rank_deficient=rank_def, max_col_size=max_col, resid=resid)


# ------------------------------------------------ Alg. 1 ingredients
def K_kernel_matrix(x, M, sigma, m, window="kb"):
    """K = A D^* F^* = (K(x_h - l/M_sigma))_{h, l} with K(x) = (1/M_sigma)
    sum_k e^{2 pi i k x}/what(-k) (eqs. matrix_K, kernel P:734-757), formed as
    the literal matrix product."""
    Ms = msigma(M, sigma)
    A = matrix_A(x, M)
    D = deconv_vector(M, sigma, m, 1.0, window)
    return A @ (D.conj()[:, None] * matrix_F(M, Ms).conj().T)


def alg1_setup(x, M, sigma, m, tau=TAU_DEFAULT, weights="real", window="kb"):
    """Alg. "Fast optimization of the matrix B*": per node j minimise
    ||K_j b - M e_j|| (eq. opt_ansatz1), K_j = columns l in I(x_j) of
    K (eq. matrix_Kj); b~_j is column j of B_opt^* (P:858), stored conjugated as
    slot weights of B_opt (reading A4).  Returns (w [N][2m+1], info)."""
    x = np.asarray(x, dtype=np.float64)
    Ms = msigma(M, sigma)
    N = x.size
    P = 2 * m + 1
    K = K_kernel_matrix(x, M, sigma, m, window)
    l0 = node_base(x, Ms, m)
    live = slot_live(x, Ms, m)
    cplx = weights == "complex"
    w = np.zeros((N, P), dtype=np.complex128 if cplx else np.float64)
    rank_def = 0
    resid = {}
    for j in range(N):
        ts = np.nonzero(live[j])[0]
        cols = np.mod(l0[j] + ts + Ms // 2, Ms)  # column index of l in [-Msig/2, Msig/2)
        Kj = K[:, cols]
        e = np.zeros(N, dtype=np.complex128)
        e[j] = M
        b, nd = lstsq_minnorm_svd(Kj, e, tau, real=not cplx)
        resid[j] = float(np.linalg.norm(Kj @ b - e))
        rank_def += nd > 0
        w[j, ts] = np.conj(b)
    return w, dict(n_rank_deficient=rank_def, max_col_size=P, resid=resid)


# ------------------------------------------------ objectives
def objective_alg2(x, M, sigma, m, w, window="kb"):
    """||F D A^* B - I_{M_sigma}||_F (eq. matrixnorm_opt_ansatz2)."""
    Ms = msigma(M, sigma)
    B = dense_from_slots(w, node_base(x, Ms, m), Ms)
    D = np.diag(deconv_vector(M, sigma, m, 1.0, window))
    X = matrix_F(M, Ms) @ D @ matrix_A(x, M).conj().T @ B
    return float(np.linalg.norm(X - np.eye(Ms)))


def objective_alg1(x, M, sigma, m, w, window="kb"):
    """||A D^* F^* B^* - M I_N||_F (eq. matrixnorm_opt_ansatz1)."""
    Ms = msigma(M, sigma)
    B = dense_from_slots(w, node_base(x, Ms, m), Ms)
    X = K_kernel_matrix(x, M, sigma, m, window) @ B.conj().T
    return float(np.linalg.norm(X - M * np.eye(len(x))))


# ===================================================== C apply (fast oracle)
def build_c(force=False):
    """Compile oracle/inft_oracle.c -> oracle/liboracle.so (gcc -O2 -fopenmp)."""
    src = os.path.join(_HERE, "inft_oracle.c")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(src)):
        return _LIB_PATH
    cmd = ["gcc", "-O2", "-std=c99", "-fopenmp", "-fPIC", "-shared", "-o", _LIB_PATH, src, "-lm"]
    subprocess.check_call(cmd)
    return _LIB_PATH


_lib = None


def _clib():
    global _lib
    if _lib is None:
        build_c()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        for name in ("oracle_inverse_1d", "oracle_adjoint_1d"):
            fn = getattr(lib, name)
            fn.argtypes = [I64, I64, I64, ctypes.c_int, P, P, P, P, P, P, I64, ctypes.c_int]
            fn.restype = ctypes.c_int
        for name in ("oracle_inverse_2d", "oracle_adjoint_2d"):
            fn = getattr(lib, name)
            fn.argtypes = [I64, P, P, P, P, P, P, P, P, P, P, I64, ctypes.c_int]
            fn.restype = ctypes.c_int
        lib.oracle_dft.argtypes = [P, I64, ctypes.c_int]
        lib.oracle_trig_sum.argtypes = [I64, I64, P, I64, P, P, ctypes.c_int]
        lib.oracle_trig_sum.restype = ctypes.c_int
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def num_threads():
    return int(_clib().oracle_num_threads())


def dft(x, sign):
    """The oracle's DFT (pinned against the definition)."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.complex128).copy())
    _clib().oracle_dft(_ptr(a), a.size, int(sign))
    return a


def trig_sum(c, x, nthreads=0):
    """out[r][i] = sum_{k=-M/2}^{M/2-1} c[r][k + M/2] e^{2 pi i k x_i}: the plain direct sum in C
    (oracle_trig_sum; angle-addition steps restarted from an exactly reduced phase every 32
    terms).  c [M] or [R][M] complex; returns [n] or [R][n]."""
    c = np.asarray(c, dtype=np.complex128)
    one = c.ndim == 1
    c = np.ascontiguousarray(np.atleast_2d(c))
    R, M = c.shape
    xs = np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel())
    out = np.zeros((R, xs.size), dtype=np.complex128)
    if xs.size and R:
        _clib().oracle_trig_sum(M, R, _ptr(c), xs.size, _ptr(xs), _ptr(out), nthreads)
    shape = np.asarray(x).shape
    return out[0].reshape(shape) if one else out.reshape((R,) + shape)


_COEF_CACHE = {}


def _kernel_coefs(M, sigma, m, window, power):
    """1/(M_sigma what(k)^power), k = -M/2..M/2-1 (cached: the I0 series over 2^20 k is slow)."""
    key = (M, sigma, m, window, power)
    if key not in _COEF_CACHE:
        Ms = msigma(M, sigma)
        c = (1.0 / window_hat_vector(M, sigma, m) ** power / Ms if window == "kb"
             else inv_what_vector(M, sigma, m, window) ** power / Ms)
        if len(_COEF_CACHE) > 16:
            _COEF_CACHE.clear()
        _COEF_CACHE[key] = np.ascontiguousarray(c, dtype=np.complex128)
    return _COEF_CACHE[key]


def G_kernel_c(dx, M, sigma, m, window="kb"):
    """G(x) of G_kernel by the C direct sum (same sum, for large test samples)."""
    return trig_sum(_kernel_coefs(M, sigma, m, window, 2), dx)


def Kplus_kernel_c(dx, M, sigma, m, window="kb"):
    """K+(x) of Kplus_kernel by the C direct sum."""
    return trig_sum(_kernel_coefs(M, sigma, m, window, 1), dx)


def ndft_c(x, fhat, M):
    """f = A fhat (eq. nfft) by the C direct sum; 1-D, fhat [R][M] centered."""
    return trig_sum(np.atleast_2d(fhat), x)


def _split_w(w):
    w = np.asarray(w)
    if np.iscomplexobj(w):
        return np.ascontiguousarray(w.real), np.ascontiguousarray(w.imag)
    return np.ascontiguousarray(w, dtype=np.float64), None


def apply_inverse(x, M, sigma, m, w, s, f, nthreads=0, window="kb"):
    """Fast oracle inverse NFFT  s D^* F^* B_opt^* f  (C loops), f [R][N] complex."""
    x = np.asarray(x, dtype=np.float64)
    f = np.ascontiguousarray(np.asarray(f, dtype=np.complex128))
    R = f.shape[0]
    wre, wim = _split_w(w)
    if x.ndim == 1:
        Ms = msigma(M, sigma)
        l0 = np.ascontiguousarray(node_base(x, Ms, m))
        d = np.ascontiguousarray(deconv_vector(M, sigma, m, s, window))
        out = np.zeros((R, M), dtype=np.complex128)
        rc = _clib().oracle_inverse_1d(x.size, M, Ms, 2 * m + 1, _ptr(l0), _ptr(wre), _ptr(wim),
                                       _ptr(d), _ptr(f), _ptr(out), R, nthreads)
    else:
        M1, M2 = M
        S = np.array([msigma(M1, sigma), msigma(M2, sigma)], dtype=np.int64)
        Mv = np.array([M1, M2], dtype=np.int64)
        Pv = np.array([2 * m + 1, 2 * m + 1], dtype=np.int32)
        l0 = np.ascontiguousarray(np.stack([node_base(x[:, 0], S[0], m), node_base(x[:, 1], S[1], m)], 1))
        d1 = np.ascontiguousarray(deconv_vector(M1, sigma, m, s, window))
        d2 = np.ascontiguousarray(deconv_vector(M2, sigma, m, 1.0, window))
        out = np.zeros((R, M1 * M2), dtype=np.complex128)
        rc = _clib().oracle_inverse_2d(x.shape[0], _ptr(Mv), _ptr(S), _ptr(Pv), _ptr(l0), _ptr(wre),
                                       _ptr(wim), _ptr(d1), _ptr(d2), _ptr(f), _ptr(out), R, nthreads)
    if rc:
        raise RuntimeError("oracle inverse failed")
    return out


def apply_adjoint(x, M, sigma, m, w, s, h, nthreads=0, window="kb"):
    """Fast oracle inverse adjoint NFFT  s B_opt F D h  (C loops), h [R][prod M] complex."""
    x = np.asarray(x, dtype=np.float64)
    h = np.ascontiguousarray(np.asarray(h, dtype=np.complex128))
    R = h.shape[0]
    wre, wim = _split_w(w)
    N = x.shape[0]
    out = np.zeros((R, N), dtype=np.complex128)
    if x.ndim == 1:
        Ms = msigma(M, sigma)
        l0 = np.ascontiguousarray(node_base(x, Ms, m))
        d = np.ascontiguousarray(deconv_vector(M, sigma, m, s, window))
        rc = _clib().oracle_adjoint_1d(N, M, Ms, 2 * m + 1, _ptr(l0), _ptr(wre), _ptr(wim),
                                       _ptr(d), _ptr(h), _ptr(out), R, nthreads)
    else:
        M1, M2 = M
        S = np.array([msigma(M1, sigma), msigma(M2, sigma)], dtype=np.int64)
        Mv = np.array([M1, M2], dtype=np.int64)
        Pv = np.array([2 * m + 1, 2 * m + 1], dtype=np.int32)
        l0 = np.ascontiguousarray(np.stack([node_base(x[:, 0], S[0], m), node_base(x[:, 1], S[1], m)], 1))
        d1 = np.ascontiguousarray(deconv_vector(M1, sigma, m, s, window))
        d2 = np.ascontiguousarray(deconv_vector(M2, sigma, m, 1.0, window))
        rc = _clib().oracle_adjoint_2d(N, _ptr(Mv), _ptr(S), _ptr(Pv), _ptr(l0), _ptr(wre),
                                       _ptr(wim), _ptr(d1), _ptr(d2), _ptr(h), _ptr(out), R, nthreads)
    if rc:
        raise RuntimeError("oracle adjoint failed")
    return out


def apply_scale(alg, M):
    """Reading A2: s = 1/M for Alg. 1, 1 for Alg. 2 and the plain NFFT."""
    return 1.0 / float(np.prod(M)) if alg == 1 else 1.0


def rel_l2(y, yref):
    """Reading A15: per-RHS ||y - y_ref||_2 / ||y_ref||_2, max over RHS."""
    y = np.atleast_2d(y)
    yref = np.atleast_2d(yref)
    num = np.linalg.norm(y - yref, axis=1)
    den = np.linalg.norm(yref, axis=1)
    return float(np.max(num / np.where(den > 0, den, 1.0)))

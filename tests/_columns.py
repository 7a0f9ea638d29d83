"""Test helpers (not a test module): the grid columns I(l) of Alg. "Fast optimization of the
matrix B" (eq. set_l) for a seeded SAMPLE of columns, and the oracle's per-column
optimum of ||L_l b - e_l|| in the Gram form (reading A6), so that the GPU's B_opt can
be checked column by column at full config size.

Everything here is built from oracle functions (index sets, kernels G and K+, the min-norm
solve); nothing comes from the CUDA path except the weights under test."""
import numpy as np

import oracle as O


def column_sizes_1d(x, Ms, m):
    """|I(l)| for every grid point n = l mod Ms (live slots only, reading A5)."""
    l0 = O.node_base(x, Ms, m)
    live = O.slot_live(x, Ms, m)
    size = np.zeros(Ms, dtype=np.int64)
    for t in range(2 * m + 1):
        size += np.bincount(np.mod(l0 + t, Ms), weights=live[:, t], minlength=Ms).astype(np.int64)
    return size


def column_members_1d(x, Ms, m, cols):
    """{n: [(j, t), ...]} for the sampled grid columns n (live slot t of node j lands on n)."""
    l0 = O.node_base(x, Ms, m)
    n0 = np.mod(l0, Ms)
    live = O.slot_live(x, Ms, m)
    order = np.argsort(n0, kind="stable")
    n0s = n0[order]
    out = {}
    for n in cols:
        mem = []
        for t in range(2 * m + 1):
            target = (n - t) % Ms
            a, b = np.searchsorted(n0s, target, "left"), np.searchsorted(n0s, target, "right")
            for j in order[a:b]:
                if live[j, t]:
                    mem.append((int(j), t))
        out[int(n)] = mem
    return out


def column_sizes_2d(x, M, sigma, m):
    S1, S2 = O.msigma(M[0], sigma), O.msigma(M[1], sigma)
    l1, l2 = O.node_base(x[:, 0], S1, m), O.node_base(x[:, 1], S2, m)
    v1, v2 = O.slot_live(x[:, 0], S1, m), O.slot_live(x[:, 1], S2, m)
    size = np.zeros(S1 * S2, dtype=np.int64)
    for t1 in range(2 * m + 1):
        for t2 in range(2 * m + 1):
            keep = v1[:, t1] & v2[:, t2]
            n = np.mod(l1 + t1, S1) * S2 + np.mod(l2 + t2, S2)
            size += np.bincount(n[keep], minlength=S1 * S2)
    return size


def column_members_2d(x, M, sigma, m, cols):
    S1, S2 = O.msigma(M[0], sigma), O.msigma(M[1], sigma)
    P1 = 2 * m + 1
    l1, l2 = O.node_base(x[:, 0], S1, m), O.node_base(x[:, 1], S2, m)
    v1, v2 = O.slot_live(x[:, 0], S1, m), O.slot_live(x[:, 1], S2, m)
    out = {}
    for n in cols:
        n1, n2 = divmod(int(n), S2)
        t1 = np.mod(n1 - l1, S1)
        t2 = np.mod(n2 - l2, S2)
        ok = (t1 <= 2 * m) & (t2 <= 2 * m)
        js = np.nonzero(ok)[0]
        js = js[v1[js, t1[js]] & v2[js, t2[js]]]
        out[int(n)] = [(int(j), int(t1[j]) * P1 + int(t2[j])) for j in js]
    return out


def sample_columns(size, n_total=512, n_largest=32, seed=0):
    """The n_largest largest columns (ties: lowest index) plus seeded non-empty others."""
    order = np.argsort(-size, kind="stable")
    largest = [int(n) for n in order[:n_largest]]
    rest = np.setdiff1d(np.nonzero(size > 0)[0], largest)
    rng = np.random.default_rng(seed)
    k = min(n_total - len(largest), rest.size)
    return largest, largest + [int(n) for n in rng.choice(rest, k, replace=False)]


def _sym_kernel(fn, xs, M, sigma, m, window):
    """Symmetric matrix fn(xs_i - xs_j) (wrapped differences), upper triangle evaluated."""
    n = xs.size
    iu = np.triu_indices(n)
    vals = fn(O.wrap_diff(xs[iu[0]] - xs[iu[1]]), M, sigma, m, window)
    A = np.zeros((n, n), dtype=np.complex128)
    A[iu] = vals
    A[(iu[1], iu[0])] = np.conj(vals)  # G(-x) = conj G(x) (real coefficients)
    return A


def gram_1d(x, js, n, M, sigma, m, window="kb"):
    """Re(L_l^* L_l) = Re G(x_j - x_j') and Re(L_l^* e_l) = Re K+(x_j - l/Ms) (Gram form)."""
    Ms = O.msigma(M, sigma)
    l = n - Ms if n >= Ms // 2 else n
    xs = x[np.asarray(js, dtype=np.int64)]
    G = np.real(_sym_kernel(O.G_kernel_c, xs, M, sigma, m, window))
    y = np.real(O.Kplus_kernel_c(O.wrap_diff(xs - l / Ms), M, sigma, m, window))
    return G, y


def gram_2d(x, js, n, M, sigma, m, window="kb"):
    """Tensor-product reading A12: G = G1 G2, K+ = K+1 K+2 (real parts of the products)."""
    S1, S2 = O.msigma(M[0], sigma), O.msigma(M[1], sigma)
    n1, n2 = divmod(int(n), S2)
    l1 = n1 - S1 if n1 >= S1 // 2 else n1
    l2 = n2 - S2 if n2 >= S2 // 2 else n2
    xs = x[np.asarray(js, dtype=np.int64)]
    g1 = _sym_kernel(O.G_kernel_c, xs[:, 0], M[0], sigma, m, window)
    g2 = _sym_kernel(O.G_kernel_c, xs[:, 1], M[1], sigma, m, window)
    y = np.real(O.Kplus_kernel_c(O.wrap_diff(xs[:, 0] - l1 / S1), M[0], sigma, m, window) *
                O.Kplus_kernel_c(O.wrap_diff(xs[:, 1] - l2 / S2), M[1], sigma, m, window))
    return np.real(g1 * g2), y


def residual(G, y, b):
    """||L_l b - e_l||_2 from the Gram form: b^T G b - 2 b^T y + ||e_l||^2, ||e_l|| = 1."""
    return float(np.sqrt(max(b @ G @ b - 2.0 * b @ y + 1.0, 0.0)))

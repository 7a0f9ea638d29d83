"""GPU Alg. 2 setup at the sizes whose columns are large (config 3: Chebyshev nodes, |I(l)| up
to 652; config 4: polar grid, |I(l)| up to 3528): the GPU's B_opt must reach the oracle's
per-column optimum of ||L_l b - e_l|| (Alg. "Fast optimization of the matrix B", P:1298-1333,
Gram form of reading A6) on a seeded sample of columns that includes the largest ones.

The columns are numerically rank deficient (reading A6's cutoff drops most directions of the
big ones), so b itself is only determined up to the rounding of near-null directions; the
residual -- what the algorithm minimises -- is the compared quantity."""
import time

import numpy as np
import pytest

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1811_05335_b200 as P
    return P


def _columns_1d(x, Ms, m):
    sets = O.grid_node_sets(x, Ms, m)
    return {n: s for n, s in enumerate(sets)}


def _columns_2d(x, M, sigma, m):
    S1, S2 = O.msigma(M[0], sigma), O.msigma(M[1], sigma)
    P1 = 2 * m + 1
    l0 = np.stack([O.node_base(x[:, 0], S1, m), O.node_base(x[:, 1], S2, m)], axis=1)
    live1, live2 = O.slot_live(x[:, 0], S1, m), O.slot_live(x[:, 1], S2, m)
    sets = {}
    for j in range(x.shape[0]):
        for t1 in np.nonzero(live1[j])[0]:
            n1 = (l0[j, 0] + t1) % S1
            for t2 in np.nonzero(live2[j])[0]:
                n2 = (l0[j, 1] + t2) % S2
                sets.setdefault(int(n1 * S2 + n2), []).append((j, int(t1) * P1 + int(t2)))
    return sets


def _kernel_rows(fn, dx, M, sigma, m):
    """fn (the oracle's G / K+ direct sum) over the rows of dx in chunks of <= 2^24 terms."""
    dx = np.atleast_2d(dx)
    rows = max(1, (1 << 24) // max(1, dx.shape[1] * M))
    return np.concatenate([fn(dx[i:i + rows], M, sigma, m) for i in range(0, dx.shape[0], rows)])


def _gram(x, js, n, M, sigma, m):
    xs = x[js]
    if x.ndim == 1:
        Ms = O.msigma(M, sigma)
        l = n - Ms if n >= Ms // 2 else n
        G = np.real(_kernel_rows(O.G_kernel, O.wrap_diff(xs[:, None] - xs[None, :]), M, sigma, m))
        y = np.real(O.Kplus_kernel(O.wrap_diff(xs - l / Ms), M, sigma, m))
        return G, y
    S1, S2 = O.msigma(M[0], sigma), O.msigma(M[1], sigma)
    n1, n2 = divmod(n, S2)
    l1 = n1 - S1 if n1 >= S1 // 2 else n1
    l2 = n2 - S2 if n2 >= S2 // 2 else n2
    g1 = _kernel_rows(O.G_kernel, O.wrap_diff(xs[:, None, 0] - xs[None, :, 0]), M[0], sigma, m)
    g2 = _kernel_rows(O.G_kernel, O.wrap_diff(xs[:, None, 1] - xs[None, :, 1]), M[1], sigma, m)
    y = np.real(O.Kplus_kernel(O.wrap_diff(xs[:, 0] - l1 / S1), M[0], sigma, m) *
                O.Kplus_kernel(O.wrap_diff(xs[:, 1] - l2 / S2), M[1], sigma, m))
    return np.real(g1 * g2), y


def _resid(G, y, b):
    return float(np.sqrt(max(b @ G @ b - 2 * b @ y + 1.0, 0.0)))


@pytest.mark.parametrize("cid", [3, 4])
def test_alg2_gpu_setup_large_columns(P, cid):
    c = S.config(cid)
    x = S.make_nodes(c)
    M = c["M"][0] if c["d"] == 1 else c["M"]
    sigma, m = c["sigma"], c["m"]
    t0 = time.perf_counter()
    plan = P.Plan(x, M, sigma, m).precompute("alg2")
    dt = time.perf_counter() - t0
    info = plan.info()
    w = plan.get_bopt()
    assert np.all(np.isfinite(w))
    sets = _columns_1d(x, O.msigma(M, sigma), m) if c["d"] == 1 else _columns_2d(x, M, sigma, m)
    assert info["max_col_size"] == max(len(s) for s in sets.values())
    big = [n for n in sets if len(sets[n]) > 64]
    assert info["n_rank_deficient"] > 0 and 0 < info["max_lowrank_rank"] <= 512
    # seeded sample: the largest column (config 4; config 3's largest 1-D columns cost the
    # oracle's direct sums M = 16384 terms per entry, so its sample stops at 200 unknowns),
    # large columns of several sizes, and small ones
    rng = np.random.default_rng(cid)
    cap = 4000 if c["d"] == 2 else 200
    by_size = sorted((n for n in sets if len(sets[n]) <= cap), key=lambda n: -len(sets[n]))
    mid = [n for n in big if len(sets[n]) <= min(cap, 600)]
    sample = by_size[:1] + list(rng.choice(mid, 5, replace=False)) + \
        list(rng.choice([n for n in sets if 0 < len(sets[n]) <= 64], 6, replace=False))
    for n in sample:
        js = [j for j, _ in sets[n]]
        ts = [t for _, t in sets[n]]
        G, y = _gram(x, js, n, M, sigma, m)
        bo, _ = O.solve_minnorm_gram(G, y)
        bg = w[js, ts]
        ro, rg = _resid(G, y, bo), _resid(G, y, bg)
        assert abs(rg - ro) <= 1e-6, (n, len(js), ro, rg)
    print(f"config {cid}: GPU Alg. 2 setup {dt:.2f} s, {len(big)} large columns, "
          f"max |I(l)| {info['max_col_size']}, max rank {info['max_lowrank_rank']}")


@pytest.mark.parametrize("seed", range(6))
def test_alg2_random_large_columns(P, seed):
    """Seeded random 1-D node clusters whose grid columns hold more than 64 unknowns (the
    pivoted-Cholesky low-rank solver) next to ordinary ones: sampled columns, including the
    largest, reach the oracle's per-column optimum."""
    rng = np.random.default_rng(4000 + seed)
    M = int(rng.choice([512, 1024, 2048]))
    sigma = float(rng.choice([1.5, 2.0]))
    if (sigma * M) % 2:
        sigma = 2.0
    m = int(rng.integers(2, 9))
    N = int(rng.choice([8192, 16384]))
    width = float(rng.choice([0.002, 0.01, 0.03]))
    x = np.sort(np.clip(np.concatenate([rng.normal(rng.uniform(-0.4, 0.4), width, N // 2),
                                        rng.random(N - N // 2) - 0.5]), -0.5, 0.5 - 1e-12))
    window = "dirichlet" if seed % 3 == 2 else "kb"
    plan = P.Plan(x, M, sigma, m, window=window).precompute("alg2")
    w = plan.get_bopt()
    assert np.all(np.isfinite(w))
    Ms = O.msigma(M, sigma)
    sets = _columns_1d(x, Ms, m)
    big = [n for n in sets if len(sets[n]) > 64]
    assert big, "the cluster should produce low-rank columns"
    by_size = sorted((n for n in sets if 0 < len(sets[n]) <= 400), key=lambda n: -len(sets[n]))
    small = [n for n in sets if 0 < len(sets[n]) <= 64]
    sample = by_size[:2] + list(rng.choice(big, min(3, len(big)), replace=False)) + \
        list(rng.choice(small, 4, replace=False))
    for n in sample:
        if len(sets[n]) > 400:
            continue
        js = [j for j, _ in sets[n]]
        ts = [t for _, t in sets[n]]
        xs = x[js]
        l = n - Ms if n >= Ms // 2 else n
        G = np.real(_kernel_rows(lambda d, M_, s_, m_: O.G_kernel(d, M_, s_, m_, window),
                                 O.wrap_diff(xs[:, None] - xs[None, :]), M, sigma, m))
        y = np.real(O.Kplus_kernel(O.wrap_diff(xs - l / Ms), M, sigma, m, window))
        bo, _ = O.solve_minnorm_gram(G, y)
        ro, rg = _resid(G, y, bo), _resid(G, y, w[js, ts])
        assert abs(rg - ro) <= 1e-6, (seed, n, len(js), ro, rg)

"""GPU: the ring kernels' node-balanced chunk tables on clustered nodes -- heavy segments split
into node ranges (spread: side slots + fixed-order fix-up; gather: independent outputs), heavy
segments at the periodic wrap, runs of consecutive heavy segments, all nodes in a few
segments -- element-wise against the oracle (inverse = spread path, adjoint = gather path)."""
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


def _nodes(kind, N, Ms, m, seed):
    rng = np.random.default_rng(seed)
    if kind == "wrap":  # half uniform, half within 3 grid cells of the wrap point
        a = rng.random(N // 2) - 0.5
        b = (rng.random(N - N // 2) - 0.5) * 6.0 / Ms
        x = np.concatenate([a, np.where(b < 0, b + 0.5, b - 0.5)])
    elif kind == "block":  # every node inside 3 consecutive segments (m = 8: 48 cells)
        x = 0.1 + rng.random(N) * 40.0 / Ms
    else:  # two clusters plus a sparse background
        x = np.concatenate([rng.normal(-0.2, 2e-3, N // 3), rng.normal(0.3, 1e-3, N // 3),
                            rng.random(N - 2 * (N // 3)) - 0.5])
    # the ring kernels need the caller order to be a cyclic shift of the plan's sort order
    # (by n0 = l0 mod M_sigma, reading A19; their f tiles are contiguous node runs): sorted by
    # n0, then rotated by about a third at a change of n0
    x = np.clip(x, -0.5, 0.5 - 1e-12)
    n0 = np.mod(O.node_base(x, Ms, m), Ms)
    o = np.lexsort((x, n0))
    x, n0 = x[o], n0[o]
    k = N // 3
    while k < N and n0[k] == n0[k - 1]:
        k += 1
    return np.roll(x, -k)


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("m", [4, 8, 16])
@pytest.mark.parametrize("kind", ["wrap", "block", "clusters"])
def test_ring_split_parity(P, torch, kind, m, prec):
    M, sigma, N = 2048, 2.0, 4096
    Ms = O.msigma(M, sigma)
    x = _nodes(kind, N, Ms, m, m)
    live = O.slot_live(x, Ms, m)
    rng = np.random.default_rng(m)
    w = rng.standard_normal(live.shape) * live
    plan = P.Plan(x, M, sigma, m, precision=prec).set_bopt(w, "alg2")
    info = plan.info()
    dt = torch.complex128 if prec == "c128" else torch.complex64
    tol = 1e-12 if prec == "c128" else 1e-5
    c = lambda t: t.cpu().numpy().astype(np.complex128)  # noqa: E731
    for R in (1, 40, 64):
        f = torch.from_numpy(S.normal_complex(R, N, R)).to("cuda", dt)
        h = torch.from_numpy(S.normal_complex(R, M, R + 1)).to("cuda", dt)
        for _ in range(2):  # plain call, then graph capture
            assert O.rel_l2(c(plan.apply(f)), O.apply_inverse(x, M, sigma, m, w, 1.0, c(f))) <= tol, (kind, m, R)
            assert O.rel_l2(c(plan.adjoint_apply(h)), O.apply_adjoint(x, M, sigma, m, w, 1.0, c(h))) <= tol, (kind, m, R)
    assert info["fast_path"] == 2 or (prec == "c64" and m == 4)  # the ring kernels ran

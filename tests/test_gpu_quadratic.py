"""GPU: the quadratic case M = N (inft_quad_*)
against the oracle (oracle/quadratic.py, direct sums) element by element, and -- at sizes the
oracle's dense sums cannot reach -- against the exactness of the Lagrange relation (the inverse
returns fhat from f = A fhat, the adjoint returns f from h = A^* f), with sparse inputs whose
NDFTs are cheap in numpy."""
import time

import numpy as np
import pytest

import oracle as O
from oracle import quadratic as Q
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


def _nodes(kind, N, seed):
    if kind == "jittered":
        return S.jittered(N, seed)
    return np.sort(np.random.default_rng(seed).random(N) - 0.5)


@pytest.mark.parametrize("N,kind,R", [(2, "jittered", 1), (8, "jittered", 5), (64, "iid", 3), (1000, "jittered", 33),
                                      (4096, "jittered", 17)])
def test_quadratic_parity(P, torch, N, kind, R):
    y = _nodes(kind, N, N)
    q = P.QuadPlan(y)
    x, a, b, s = q.coeffs()
    xo, ao, bo, so = Q.coeffs(y)
    np.testing.assert_array_equal(x, xo)
    tol_c = 1e-9 if N > 1000 else 1e-11
    assert np.abs(a / ao - 1).max() < tol_c and np.abs(b / bo - 1).max() < tol_c
    assert abs(s - so) <= 1e-11 * max(1.0, abs(so))
    f = S.normal_complex(R, N, 1)
    h = S.normal_complex(R, N, 2)
    tol = 1e-9 if N > 1000 else 1e-11
    got = q.apply(torch.from_numpy(f).cuda()).cpu().numpy()
    assert O.rel_l2(got, Q.inverse(y, f)) < tol
    got = q.adjoint_apply(torch.from_numpy(h).cuda()).cpu().numpy()
    assert O.rel_l2(got, Q.adjoint(y, h)) < tol
    # host buffers through the same entry points
    assert O.rel_l2(q.apply(f), Q.inverse(y, f)) < tol
    assert q.kernel_launches() > 0


@pytest.mark.parametrize("N", [1 << 14, 1 << 16])
def test_quadratic_exact_large(P, torch, N):
    """Sparse fhat (8 frequencies) -> f = A fhat by 8 exponentials per node; the GPU inverse
    must return fhat.  Sparse f (8 nodes) -> h = A^* f; the GPU adjoint must return f."""
    y = S.jittered(N, 3)
    rng = np.random.default_rng(N)
    R = 4
    ks = rng.choice(N, 8, replace=False)
    fhat = np.zeros((R, N), dtype=np.complex128)
    fhat[:, ks] = S.normal_complex(R, 8, 4)
    f = fhat[:, ks] @ np.exp(2j * np.pi * np.outer(ks - N // 2, y))
    q = P.QuadPlan(y)
    ft = torch.from_numpy(f).cuda()
    q.apply(ft)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    got = q.apply(ft)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"quadratic inverse N = {N}, R = {R}: {dt * 1e3:.1f} ms")
    assert O.rel_l2(got.cpu().numpy(), fhat) < 1e-9
    js = rng.choice(N, 8, replace=False)
    fs = np.zeros((R, N), dtype=np.complex128)
    fs[:, js] = S.normal_complex(R, 8, 5)
    h = fs[:, js] @ np.exp(-2j * np.pi * np.outer(y[js], np.arange(-N // 2, N // 2)))
    got = q.adjoint_apply(torch.from_numpy(np.ascontiguousarray(h)).cuda()).cpu().numpy()
    assert O.rel_l2(got, fs) < 1e-9


def test_quadratic_errors(P):
    with pytest.raises(P.InftError):
        P.QuadPlan(S.jittered(7, 1))  # N odd
    N = 16
    y = S.jittered(N, 2)
    y[3] = -0.5 + 5 / N + 0.5 / N  # a node on the target x_5
    with pytest.raises(P.InftError):
        P.QuadPlan(np.sort(y))
    with pytest.raises(P.InftError):
        P.QuadPlan(np.array([0.1, 0.1, 0.2, 0.3]))  # repeated node


@pytest.mark.parametrize("N,kind", [(512, "jittered"), (4096, "jittered"), (1500, "iid"), (1 << 15, "jittered")])
def test_fast_summation_equals_direct(P, torch, N, kind):
    """The fast summation (default for N >= 512) against the direct GPU sums (INFT_QUAD_DIRECT=1)
    on the same nodes: coefficients a, b and both applies."""
    import os
    y = _nodes(kind, N, 7)
    qf = P.QuadPlan(y)
    os.environ["INFT_QUAD_DIRECT"] = "1"
    try:
        qd = P.QuadPlan(y)
    finally:
        del os.environ["INFT_QUAD_DIRECT"]
    _, af, bf, _ = qf.coeffs()
    _, ad, bd, _ = qd.coeffs()
    assert np.abs(af / ad - 1).max() < 1e-9 and np.abs(bf / bd - 1).max() < 1e-9
    R = 3
    f = torch.from_numpy(S.normal_complex(R, N, 8)).cuda()
    h = torch.from_numpy(S.normal_complex(R, N, 9)).cuda()
    tol = 1e-9 if kind == "jittered" else 1e-7
    assert O.rel_l2(qf.apply(f).cpu().numpy(), qd.apply(f).cpu().numpy()) < tol
    assert O.rel_l2(qf.adjoint_apply(h).cpu().numpy(), qd.adjoint_apply(h).cpu().numpy()) < tol


@pytest.mark.parametrize("seed", range(8))
def test_fast_summation_random(P, torch, seed):
    """Random even N (not powers of two) and jitter levels: fast summation = direct sums."""
    import os
    rng = np.random.default_rng(900 + seed)
    N = 2 * int(rng.integers(256, 15000))
    y = S.jittered(N, seed, jitter=float(rng.choice([0.05, 0.25, 0.45])))
    delta = float(rng.choice([0.0, 0.3 / N, 0.7 / N]))
    qf = P.QuadPlan(y, delta=delta)
    os.environ["INFT_QUAD_DIRECT"] = "1"
    try:
        qd = P.QuadPlan(y, delta=delta)
    finally:
        del os.environ["INFT_QUAD_DIRECT"]
    np.testing.assert_array_equal(qf.coeffs()[0], qd.coeffs()[0])
    R = int(rng.choice([1, 5, 20]))
    f = torch.from_numpy(S.normal_complex(R, N, seed)).cuda()
    h = torch.from_numpy(S.normal_complex(R, N, seed + 1)).cuda()
    assert O.rel_l2(qf.apply(f).cpu().numpy(), qd.apply(f).cpu().numpy()) < 1e-9, (N, seed)
    assert O.rel_l2(qf.adjoint_apply(h).cpu().numpy(), qd.adjoint_apply(h).cpu().numpy()) < 1e-9, (N, seed)

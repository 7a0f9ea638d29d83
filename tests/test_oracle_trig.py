"""Pins of the oracle's C direct trigonometric sum (oracle_trig_sum) and of the test helpers
built on it: it must equal the numpy direct sums (G_kernel, Kplus_kernel: pinned through the
Gram identity against the explicit L_l in test_oracle_pins; ndft: pinned by the equispaced
identities A A^* = M I), the column sampler must reproduce the brute-force index sets I(l)
(eq. set_l), and the wide-window plain NFFT that forms the real-workload inputs
must equal the direct NDFT."""
import numpy as np

import oracle as O
import synth as S

from _columns import (column_sizes_1d, column_members_1d, column_sizes_2d, column_members_2d,
                      sample_columns, gram_1d, residual)


def test_trig_sum_equals_numpy_direct_sums():
    rng = np.random.default_rng(0)
    for M, sigma, m in [(64, 2.0, 4), (512, 2.0, 6), (1000, 1.5, 5)]:
        dx = rng.random(257) - 0.5
        for fn, ref in ((O.G_kernel_c, O.G_kernel), (O.Kplus_kernel_c, O.Kplus_kernel)):
            a, b = fn(dx, M, sigma, m), ref(dx, M, sigma, m)
            assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()
        x = rng.random(101) - 0.5
        fh = rng.standard_normal((3, M)) + 1j * rng.standard_normal((3, M))
        assert O.rel_l2(O.ndft_c(x, fh, M), O.ndft(x, fh, M)) <= 1e-13


def test_trig_sum_large_frequency_phase():
    """|k| up to 2^20: the restarted recurrence keeps the phase exact (vs a few direct terms)."""
    M = 1 << 21
    x = np.array([0.123456789012345, -0.3999999999, 0.5 - 2.0 ** -30])
    c = np.zeros(M, dtype=np.complex128)
    ks = np.array([-M // 2, -12345, 7, M // 2 - 1])
    c[ks + M // 2] = [1.0, 2.0 - 1j, 0.5j, -3.0]
    got = O.trig_sum(c, x)
    from fractions import Fraction
    # exact rational phase frac(k x) (x is a binary fraction), rounded once to double
    ref = np.array([sum(c[k + M // 2] * np.exp(2j * np.pi * float((Fraction(int(k)) * Fraction(xi)) % 1))
                        for k in ks) for xi in x])
    assert np.abs(got - ref).max() <= 1e-12


def test_column_sampler_equals_index_sets():
    for x, M, sigma, m in [(S.jittered(300, 1), 128, 2.0, 4), (S.chebyshev(512), 256, 2.0, 6),
                           (np.concatenate([S.iid_sorted(200, 3), [0.0, 5 / 256]]), 128, 2.0, 3)]:
        Ms = O.msigma(M, sigma)
        sets = O.grid_node_sets(x, Ms, m)
        size = column_sizes_1d(x, Ms, m)
        np.testing.assert_array_equal(size, [len(s) for s in sets])
        cols = list(range(Ms))
        mem = column_members_1d(x, Ms, m, cols)
        for n in cols:
            assert sorted(mem[n]) == sorted(sets[n])
        largest, sample = sample_columns(size, n_total=64, n_largest=8, seed=1)
        assert len(set(sample)) == len(sample) and all(size[n] > 0 for n in sample)
        assert min(size[largest]) >= max(np.delete(size, largest))


def test_column_sampler_2d_equals_brute_force():
    x = S.polar(16, 16)
    M, sigma, m = (16, 16), 2.0, 2
    S1 = O.msigma(16, sigma)
    P1 = 2 * m + 1
    l1, l2 = O.node_base(x[:, 0], S1, m), O.node_base(x[:, 1], S1, m)
    v1, v2 = O.slot_live(x[:, 0], S1, m), O.slot_live(x[:, 1], S1, m)
    brute = {}
    for j in range(x.shape[0]):
        for t1 in range(P1):
            for t2 in range(P1):
                if v1[j, t1] and v2[j, t2]:
                    n = ((l1[j] + t1) % S1) * S1 + (l2[j] + t2) % S1
                    brute.setdefault(n, []).append((j, t1 * P1 + t2))
    size = column_sizes_2d(x, M, sigma, m)
    assert all(size[n] == len(brute.get(n, [])) for n in range(S1 * S1))
    mem = column_members_2d(x, M, sigma, m, list(range(S1 * S1)))
    for n in range(S1 * S1):
        assert sorted(mem[n]) == sorted(brute.get(n, []))


def test_gram_residual_equals_explicit_residual():
    """residual() from the Gram form = ||L_l b - e_l|| with the explicit L_l (eq. matrix_Ll)."""
    x = S.jittered(96, 2)
    M, sigma, m = 64, 2.0, 4
    Ms = O.msigma(M, sigma)
    mem = column_members_1d(x, Ms, m, [3, 70, 127])
    rng = np.random.default_rng(3)
    for n, ms in mem.items():
        js = [j for j, _ in ms]
        G, y = gram_1d(x, js, n, M, sigma, m)
        b = rng.standard_normal(len(js))
        l = n - Ms if n >= Ms // 2 else n
        L = O.L_explicit(l, x[js], M, sigma, m)
        e = np.zeros(Ms)
        e[l + Ms // 2] = 1.0
        assert abs(residual(G, y, b) - np.linalg.norm(L @ b - e)) <= 1e-10 * np.linalg.norm(L @ b - e)


def test_wide_nfft_inputs_match_direct_sum():
    """The real-workload input generator (oracle plain NFFT, KB m = 16, sigma = 2) equals the
    direct NDFT f = A fhat on sampled nodes of configs 3 and 5."""
    for cid in (3, 5):
        c = S.config(cid)
        x = S.make_nodes(c)
        M = c["M"][0]
        fh = S.uniform_complex(1, M, 77)
        xs = x[np.random.default_rng(cid).choice(x.size, 48, replace=False)]
        wB = O.window_slot_weights(xs, M, 2.0, 16)
        f = O.apply_adjoint(xs, M, 2.0, 16, wB, 1.0, fh)
        assert O.rel_l2(f, O.ndft_c(xs, fh, M)) < 1e-12, cid

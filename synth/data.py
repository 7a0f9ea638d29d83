"""Seeded right-hand sides and the five BASELINE configurations (shapes only).

Reading A14: numpy PCG64 ``default_rng(seed)``; for a batch of R
right-hand sides of length L the draw order is, per RHS, one Re block of L
values then one Im block of L values.
"""
import numpy as np

from .nodes import jittered, chebyshev, iid_sorted, polar


def uniform_complex(R, L, seed, lo=-1.0, hi=1.0):
    """[R][L] complex128 with Re, Im ~ U[lo, hi)."""
    rng = np.random.default_rng(seed)
    out = np.empty((R, L), dtype=np.complex128)
    for r in range(R):
        re = rng.uniform(lo, hi, L)
        im = rng.uniform(lo, hi, L)
        out[r] = re + 1j * im
    return out


def normal_complex(R, L, seed):
    """[R][L] complex128 with Re, Im ~ N(0, 1)."""
    rng = np.random.default_rng(seed)
    out = np.empty((R, L), dtype=np.complex128)
    for r in range(R):
        re = rng.standard_normal(L)
        im = rng.standard_normal(L)
        out[r] = re + 1j * im
    return out


def blob_image(R, M1, M2, seed, n_blobs=8, noise_var=0.01):
    """Config-4 coefficients (reading A13): per RHS, 8 Gaussian blobs
    (amplitude U[0.5,1], centre U[-40,40)^2 in k-index units, width U[3,12])
    plus N(0, noise_var) noise; real image stored as complex128, [R][M1][M2]
    centered (index k + M/2)."""
    rng = np.random.default_rng(seed)
    k1 = np.arange(-M1 // 2, M1 // 2, dtype=np.float64)[:, None]
    k2 = np.arange(-M2 // 2, M2 // 2, dtype=np.float64)[None, :]
    out = np.empty((R, M1, M2), dtype=np.complex128)
    for r in range(R):
        img = np.zeros((M1, M2))
        for _ in range(n_blobs):
            a = rng.uniform(0.5, 1.0)
            c1, c2 = rng.uniform(-40.0, 40.0, 2)
            wdt = rng.uniform(3.0, 12.0)
            img += a * np.exp(-((k1 - c1) ** 2 + (k2 - c2) ** 2) / (2.0 * wdt * wdt))
        img += rng.normal(0.0, np.sqrt(noise_var), (M1, M2))
        out[r] = img
    return out


# The five BASELINE.json configs.  "alg": 1 = node-wise (Alg. "Fast optimization
# of the matrix B*"), 2 = grid-wise (Alg. "Fast optimization of the
# matrix B") -- SURVEY D1.  "dirs": which apply directions the
# config times.
CONFIGS = {
    1: dict(d=1, M=(256,), N=512, nodes="jittered", seed=0, sigma=2.0, m=4, R=1,
            alg=2, dirs=("inverse",), data="uniform_fhat"),
    2: dict(d=1, M=(1024,), N=512, nodes="iid_sorted", seed=1, sigma=2.0, m=6, R=16,
            alg=1, dirs=("adjoint",), data="normal_f"),
    3: dict(d=1, M=(16384,), N=32768, nodes="chebyshev", seed=2, sigma=2.0, m=8, R=256,
            alg=2, dirs=("inverse",), data="uniform_fhat"),
    4: dict(d=2, M=(128, 128), N=65536, nodes="polar", seed=3, sigma=2.0, m=6, R=64,
            alg=2, dirs=("inverse",), data="blob_fhat"),
    5: dict(d=1, M=(1 << 20,), N=1 << 21, nodes="jittered", seed=4, sigma=2.0, m=8, R=512,
            alg=2, dirs=("inverse", "adjoint"), data="uniform_fhat"),
}


def config(i):
    c = dict(CONFIGS[i])
    c["id"] = i
    return c


def make_nodes(cfg):
    """Nodes of a config: float64 [N] (1-D) or [N][2] (2-D)."""
    kind = cfg["nodes"]
    N = cfg["N"]
    if kind == "jittered":
        return jittered(N, cfg["seed"])
    if kind == "chebyshev":
        return chebyshev(N)
    if kind == "iid_sorted":
        return iid_sorted(N, cfg["seed"])
    if kind == "polar":
        return polar(256, 256)
    raise ValueError(kind)


def make_rhs(cfg, R=None, kind="inverse", seed_offset=0):
    """Random right-hand-side material of the config's distribution.

    kind == "inverse": returns the spectral coefficients fhat [R][prod M]
    (uniform or blob) -- the sample vector f = A fhat is formed by the oracle's
    NDFT where that is affordable; parity tests of the linear apply may use
    samples drawn directly with ``normal_complex`` instead (inputs).
    kind == "adjoint": returns sample values f [R][N] ~ N(0,1) complex.
    """
    R = cfg["R"] if R is None else R
    seed = cfg["seed"] + 1000 * (1 + seed_offset)
    Mtot = int(np.prod(cfg["M"]))
    if kind == "inverse":
        if cfg["data"] == "blob_fhat":
            M1, M2 = cfg["M"]
            return blob_image(R, M1, M2, seed).reshape(R, Mtot)
        return uniform_complex(R, Mtot, seed)
    if kind == "adjoint":
        return normal_complex(R, cfg["N"], seed)
    raise ValueError(kind)

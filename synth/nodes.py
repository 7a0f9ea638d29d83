"""Node distributions of the paper's experiments (no method arithmetic)."""
import numpy as np


def wrap_half_open(x):
    """Map reals into [-1/2, 1/2) by a periodic shift (reading A10).

    A is 1-periodic in x_j (eq. matrix_A), so wrapping does not change
    the problem.  Only exact representatives are shifted (x >= 1/2 -> x - 1,
    x < -1/2 -> x + 1); everything already in range is returned bit-identical.
    """
    x = np.array(x, dtype=np.float64, copy=True)
    x[x >= 0.5] -= 1.0
    x[x < -0.5] += 1.0
    return x


def jittered(N, seed, jitter=0.25):
    """Jittered equispaced nodes, eq. (jittered_nodes) P:506-509:
    y_j = -1/2 + (j-1)/N + (jitter/N)*theta_j, theta_j ~ U(0,1), j = 1..N.
    The paper's perturbation parameter is 1/4."""
    if not (0.0 <= jitter < 0.5):
        raise ValueError("jitter must be in [0, 1/2) (P:510)")
    rng = np.random.default_rng(seed)
    theta = rng.random(N)
    j = np.arange(N, dtype=np.float64)
    return -0.5 + j / N + (jitter / N) * theta


def chebyshev(N):
    """Chebyshev nodes, eq. (tschebyscheff_nodes) P:553-556:
    y_j = 1/2 cos((2(N-j)+1)/(2N) pi), j = 1..N (increasing in j, all in (-1/2,1/2))."""
    j = np.arange(1, N + 1, dtype=np.float64)
    return 0.5 * np.cos((2.0 * (N - j) + 1.0) / (2.0 * N) * np.pi)


def iid_sorted(N, seed):
    """i.i.d. U[-1/2, 1/2) nodes, sorted increasingly (BASELINE config 2)."""
    rng = np.random.default_rng(seed)
    return np.sort(rng.random(N) - 0.5)


def equispaced(N):
    """x_j = j/N, j = -N/2..N/2-1."""
    return np.arange(-(N // 2), N - N // 2, dtype=np.float64) / N


def polar(n_angles=256, n_radii=256):
    """Polar grid (BASELINE config 4; reading A12):
    theta_t = pi (t - n_angles/2) / n_angles, r_s = -1/2 + s/n_radii,
    x = r (cos theta, sin theta); row-major N x 2, angle-major.
    Coordinates equal to +1/2 are wrapped to -1/2 (reading A10); the origin
    appears once per radial line (duplicates are kept)."""
    t = np.arange(n_angles, dtype=np.float64)
    s = np.arange(n_radii, dtype=np.float64)
    th = np.pi * (t - n_angles / 2) / n_angles
    r = -0.5 + s / n_radii
    x1 = (r[None, :] * np.cos(th)[:, None]).ravel()
    x2 = (r[None, :] * np.sin(th)[:, None]).ravel()
    return wrap_half_open(np.stack([x1, x2], axis=1))

"""Weight schedules (host side).  Mirrors schedules.py:8-82 of the reference
so the GPU package runs without it; any object with `omega`, `alpha`,
`alpha_tilde`, `variant`, `m` (e.g. a richlab.WeightSchedule) is accepted by
the solvers.  Adds the Leja ordering and stencil-symbol spectral bounds used
to build the config-3 schedules.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

VARIANTS = ("plain", "mom", "nag", "nagex")  # schedules.py:8


@dataclass(frozen=True)
class WeightSchedule:
    """omega (step weights), alpha (momentum), alpha_tilde (look-ahead).

    Validation follows schedules.py:24-50: plain forbids momentum, nag ties
    alpha_tilde to alpha, missing arrays default to zeros.
    """

    omega: np.ndarray
    alpha: np.ndarray = None
    alpha_tilde: np.ndarray = None
    variant: str = "plain"

    def __post_init__(self):
        w = np.atleast_1d(np.asarray(self.omega, dtype=float))
        m = w.size
        if m < 1:
            raise ValueError("schedule needs at least one weight")
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}")
        a = np.zeros(m) if self.alpha is None else np.atleast_1d(np.asarray(self.alpha, dtype=float))
        at = self.alpha_tilde
        if self.variant == "plain":
            at_chk = np.zeros(m) if at is None else np.atleast_1d(at)
            if np.any(a != 0.0) or np.any(at_chk != 0.0):
                raise ValueError("plain variant requires zero momentum coefficients")
        if self.variant == "nag":
            if at is not None and not np.array_equal(np.atleast_1d(at), a):
                raise ValueError("nag requires alpha_tilde == alpha")
            at = a
        at = np.zeros(m) if at is None else np.atleast_1d(np.asarray(at, dtype=float))
        if a.size != m or at.size != m:
            raise ValueError("omega, alpha, alpha_tilde must share length m")
        object.__setattr__(self, "omega", w)
        object.__setattr__(self, "alpha", a)
        object.__setattr__(self, "alpha_tilde", at)

    @property
    def m(self):
        return int(self.omega.size)


def chebyshev_weights(lambda_max, lambda_min, m):
    """omega_i = 1/lambda_i at the m Chebyshev points of [lambda_min,
    lambda_max], in the reference's order i = 1..m (schedules.py:57-67)."""
    if not lambda_max > lambda_min > 0:
        raise ValueError(
            f"need lambda_max > lambda_min > 0, got ({lambda_max}, {lambda_min})")
    if m < 1:
        raise ValueError("m must be >= 1")
    x = np.cos((2 * np.arange(1, m + 1) - 1) * np.pi / (2 * m))
    return 2.0 / (lambda_max + lambda_min + (lambda_max - lambda_min) * x)


def chebyshev_semi_weights(lambda_max, m, alpha=1.0 / 30.0):
    """schedules.py:70-74."""
    if not 0.0 < alpha < 1.0:
        raise ValueError("alpha must lie in (0, 1)")
    return chebyshev_weights(lambda_max, alpha * lambda_max, m)


def chebyshev_schedule(lambda_max, lambda_min, m):
    """schedules.py:77-78."""
    return WeightSchedule(omega=chebyshev_weights(lambda_max, lambda_min, m))


def chebyshev_semi_schedule(lambda_max, m, alpha=1.0 / 30.0):
    """schedules.py:81-82."""
    return WeightSchedule(omega=chebyshev_semi_weights(lambda_max, m, alpha))


def leja_order(omega):
    """Reorder weights so their roots 1/omega form a Leja sequence: start
    from the largest root, then repeatedly take the remaining root that
    maximises the product of distances to the chosen ones (log-sum to avoid
    overflow).  A permutation of the same weights, applied in array order by
    the solver; it tames the rounding amplification of long cyclic Chebyshev
    sweeps (SURVEY.md §8(d) cfg 3)."""
    w = np.asarray(omega, dtype=float)
    roots = 1.0 / w
    left = list(range(w.size))
    first = int(np.argmax(roots))
    chosen = [first]
    left.remove(first)
    while left:
        score = [np.sum(np.log(np.abs(roots[j] - roots[chosen]))) for j in left]
        nxt = left[int(np.argmax(score))]
        chosen.append(nxt)
        left.remove(nxt)
    return w[chosen]


def stencil_symbol_bounds(coeffs, n, grid=721):
    """Spectral bounds of a constant 9-point stencil from its symbol
    sigma(xi, eta) = sum_{a,b} c[a,b] cos(a xi + b eta): lambda_max = max of
    sigma on a grid x grid sampling of [-pi, pi]^2; lambda_min = the smaller
    of sigma(pi/n, pi/n) and sigma(pi/n, -pi/n), the two lowest Dirichlet
    frequencies (the rotated operator's cross term makes them differ; the
    smaller one is a lower estimate of the true lambda_min, which keeps the
    Chebyshev interval covering the spectrum).  coeffs in CSR order (3x3)."""
    c = np.asarray(coeffs, dtype=float).reshape(3, 3)
    t = np.linspace(-np.pi, np.pi, grid)
    xi, eta = np.meshgrid(t, t, indexing="ij")

    def sigma(x, y):
        s = 0.0
        for a in (-1, 0, 1):
            for b in (-1, 0, 1):
                s = s + c[a + 1, b + 1] * np.cos(a * x + b * y)
        return s

    lmax = float(np.max(sigma(xi, eta)))
    lmin = float(min(sigma(np.pi / n, np.pi / n), sigma(np.pi / n, -np.pi / n)))
    return lmax, lmin


def stencil_matrix(coeffs, side):
    """Host CSR of a constant 9-point stencil on a side x side interior
    (CSR column order, zero-padded at the Dirichlet boundary)."""
    import scipy.sparse as sp
    c = np.asarray(coeffs, dtype=float).reshape(3, 3)
    idx = np.arange(side * side).reshape(side, side)
    rows, cols, vals = [], [], []
    for a in (-1, 0, 1):
        for b in (-1, 0, 1):
            if c[a + 1, b + 1] == 0.0:
                continue
            i0, i1 = max(0, -a), min(side, side - a)
            j0, j1 = max(0, -b), min(side, side - b)
            r = idx[i0:i1, j0:j1]
            rows.append(r.reshape(-1))
            cols.append((r + a * side + b).reshape(-1))
            vals.append(np.full(r.size, c[a + 1, b + 1]))
    n = side * side
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(n, n))


def stencil_lambda_min(coeffs, n, grids=(64, 128), safety=0.9):
    """lambda_min of the stencil on the n-cell grid, extrapolated from exact
    small-grid eigenvalues: the unscaled FEM stiffness has lambda_min(n) ~
    mu / n^2 with an O(h^2) error, so mu is Richardson-extrapolated from
    n = grids[0], grids[1] and a safety factor keeps the estimate below the
    true value.  (The symbol value at the lowest Dirichlet frequency can
    miss the rotated operator's lambda_min by 10x or more.)"""
    import scipy.sparse.linalg as sla
    mu = []
    for g in grids:
        if g >= n:
            g = n
        A = stencil_matrix(coeffs, g - 1)
        lam = sla.eigsh(A, k=1, sigma=0, which="LM", return_eigenvectors=False)[0]
        mu.append(lam * g * g)
    if grids[1] >= n:
        return safety * mu[1] / (n * n)
    r = (grids[1] / grids[0]) ** 2
    ext = (r * mu[1] - mu[0]) / (r - 1)
    return safety * min(ext, mu[1]) / (n * n)

"""Model problems -> stencil data for the GPU operators (host side).

The reference assembles CSR matrices (problems.py:121-200) that the solver
then streams from memory on every matvec.  The GPU path never materialises
the CSR: it needs only the 9 stencil coefficients of the anisotropic
operator, or the off-diagonal constant plus the per-node complex diagonal of
the Helmholtz operator.  This module computes exactly those numbers with the
same floating-point operations the reference's assembly performs, so the
GPU operator is bitwise the reference's matrix:

* the element matrix Ke is the same NumPy expression as
  bilinear_element_stiffness (problems.py:102-118);
* each assembled stencil entry is the left-to-right sum of the element
  contributions in the order SciPy's COO->CSR duplicate summation sees
  them (triplets emitted in (a, b) order, problems.py:143-149; stable sort
  of the 16 row entries by column, then consecutive duplicates summed);
* entries with |value| <= 1e-14 * max|Ke| are dropped (problems.py:153).

tests/test_problems.py pins this against the CSR assembly of the oracle
(and the reference itself when it is importable).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ShannonViolation

# local node order of a bilinear element: (0,0), (1,0), (1,1), (0,1) in (x, y)
_LOCAL = ((0, 0), (1, 0), (1, 1), (0, 1))
# CSR column order of the 3x3 neighbourhood (lexicographic (dx, dy))
OFFSETS9 = tuple((dx, dy) for dx in (-1, 0, 1) for dy in (-1, 0, 1))
OFFSETS5 = ((-1, 0), (0, -1), (0, 0), (0, 1), (1, 0))


@dataclass(frozen=True)
class AnisotropicProblem:
    """-div(C grad u) = f, C = Q(theta) diag(1, eps) Q(theta)^T
    (problems.py:30-55)."""

    epsilon: float
    theta: float
    n: int
    kind = "anisotropic"

    def __post_init__(self):
        if not 0.0 < self.epsilon <= 1.0:
            raise ValueError(f"epsilon must be in (0, 1], got {self.epsilon}")
        if not 0.0 <= self.theta <= np.pi:
            raise ValueError(f"theta must be in [0, pi], got {self.theta}")
        if self.n < 2:
            raise ValueError(f"n must be >= 2, got {self.n}")

    @property
    def ndof(self):
        return (self.n - 1) ** 2

    @property
    def mu(self):
        return np.array([np.log10(self.epsilon), self.theta])


@dataclass(frozen=True)
class HelmholtzProblem:
    """-Lap u - k^2 u + i gamma (omega/c^2) u = f with a sponge layer
    (problems.py:58-89)."""

    angular_frequency: float
    n: int
    wave_speed: float = 1.0
    sponge_width: int | None = None
    shannon_check: bool = True
    kind = "helmholtz"

    def __post_init__(self):
        if self.angular_frequency <= 0.0:
            raise ValueError("angular_frequency must be positive")
        if self.wave_speed <= 0.0:
            raise ValueError("wave_speed must be positive")
        if self.n < 2:
            raise ValueError(f"n must be >= 2, got {self.n}")

    @property
    def ndof(self):
        return (self.n - 1) ** 2

    @property
    def wavelength_cells(self):
        return 2.0 * np.pi * self.wave_speed / (self.angular_frequency * (1.0 / self.n))

    @property
    def mu(self):
        return np.array([self.angular_frequency])


def diffusion_tensor(epsilon, theta):
    """problems.py:95-99 (same NumPy ops)."""
    c, s = np.cos(theta), np.sin(theta)
    rot = np.array([[c, -s], [s, c]])
    return rot @ np.diag([1.0, epsilon]) @ rot.T


def element_stiffness(C):
    """4x4 bilinear element matrix, 2x2 Gauss rule, symmetrised
    (problems.py:17-23,102-118; same NumPy ops so the bits agree)."""
    g = 0.5 / np.sqrt(3.0)
    pts = [(0.5 - g, 0.5 - g), (0.5 + g, 0.5 - g), (0.5 + g, 0.5 + g), (0.5 - g, 0.5 + g)]
    Ke = np.zeros((4, 4))
    for xi, eta in pts:
        G = np.array([[-(1 - eta), (1 - eta), eta, -eta],
                      [-(1 - xi), -xi, xi, (1 - xi)]])
        Ke += 0.25 * G.T @ C @ G
    return 0.5 * (Ke + Ke.T)


def anisotropic_stencil(p: AnisotropicProblem) -> np.ndarray:
    """The 9 assembled coefficients of an interior row, CSR order."""
    Ke = element_stiffness(diffusion_tensor(p.epsilon, p.theta))
    drop = 1e-14 * np.abs(Ke).max()
    # contributions to offset (dx, dy), in the order COO->CSR summation adds them
    parts = {off: [] for off in OFFSETS9}
    for a, (ax, ay) in enumerate(_LOCAL):
        for b, (bx, by) in enumerate(_LOCAL):
            parts[(bx - ax, by - ay)].append(Ke[a, b])
    out = np.zeros(9)
    for q, off in enumerate(OFFSETS9):
        terms = parts[off]
        acc = terms[0]
        for t in terms[1:]:
            acc = acc + t
        out[q] = 0.0 if abs(acc) <= drop else acc
    return out


def sponge(p: HelmholtzProblem) -> np.ndarray:
    """Damping gamma on the interior, flattened (problems.py:157-171)."""
    n = p.n
    width = p.sponge_width
    if width is None:
        width = max(1, int(round(p.wavelength_cells)))
    i = np.arange(1, n)
    edge = np.minimum(i, n - i)
    dist = np.minimum(edge[:, None], edge[None, :])
    depth = np.clip(width - dist, 0, width) / width
    return (p.angular_frequency * depth ** 2).reshape(-1)


def helmholtz_stencil(p: HelmholtzProblem):
    """(off-diagonals [4] complex in CSR order, diagonal [(n-1)^2] complex)
    of the 5-point damped operator (problems.py:174-200)."""
    if p.shannon_check and p.wavelength_cells < 10.0:
        raise ShannonViolation(
            f"only {p.wavelength_cells:.2f} grid points per wavelength (need >= 10)")
    h = 1.0 / p.n
    k = p.angular_frequency / p.wave_speed
    gamma = sponge(p)
    diag = (4.0 - k ** 2 * h ** 2) / h ** 2 + 1j * gamma * (
        p.angular_frequency / p.wave_speed ** 2)
    off = np.full(4, -1.0 / h ** 2, dtype=np.complex128)
    return off, np.asarray(diag, dtype=np.complex128)

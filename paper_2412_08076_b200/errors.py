"""Result and error types of the solve loop, mirroring the reference.

If the reference package `richlab` is importable (a user migrating from it),
its own classes are re-exported so existing `except richlab.DivergenceError`
handlers keep working; otherwise identical local definitions are used.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DIVERGENCE_FACTOR = 1e12  # richardson.py:17

try:  # pragma: no cover - depends on the user's environment
    from richlab.richardson import DivergenceError, IterationState, SolveReport  # type: ignore
    from richlab.sparse import DimensionMismatch  # type: ignore
    from richlab.precond import ZeroDiagonalError  # type: ignore
    from richlab.problems import ShannonViolation  # type: ignore
    REFERENCE_TYPES = True
except Exception:  # noqa: BLE001
    REFERENCE_TYPES = False

    class DivergenceError(RuntimeError):
        """richardson.py:20-23: raised with the 1-based inner iteration index."""

        def __init__(self, message, inner_iteration):
            super().__init__(message)
            self.inner_iteration = inner_iteration

    class DimensionMismatch(ValueError):
        """sparse.py:9-10."""

    class ZeroDiagonalError(ValueError):
        """precond.py:23-27."""

        def __init__(self, row):
            super().__init__(f"zero diagonal entry in row {row}")
            self.row = row

    class ShannonViolation(ValueError):
        """problems.py:26-27."""

    @dataclass
    class IterationState:
        """richardson.py:26-35 (u, v may be numpy arrays or CUDA tensors)."""
        u: object
        v: object
        outer_count: int = 0
        residual_history: list = field(default_factory=list)

        @classmethod
        def start(cls, n, dtype=np.float64):
            return cls(u=np.zeros(n, dtype=dtype), v=np.zeros(n, dtype=dtype))

    @dataclass
    class SolveReport:
        """richardson.py:38-46."""
        iterations: int
        inner_iterations: int
        converged: bool
        final_relative_residual: float
        wall_time: float
        trace: np.ndarray
        stagnated: bool = False


class UnsupportedOperator(ValueError):
    """The matrix is not a structured-grid operator this library handles
    (pattern outside the 3x3 neighbourhood, non-square grid, ...)."""

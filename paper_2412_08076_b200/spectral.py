"""GPU drop-in for the spectral-bound estimators (spectral.py:10-98),
SURVEY.md §8(f) item 4.

    estimate_lambda_max(A, tol=1e-8, max_iter=10_000, seed=0) -> SpectralBounds
    estimate_lambda_min(A, lambda_max, tol=1e-8, max_iter=50_000, seed=0,
                        shift_factor=1.01)                    -> SpectralBounds
    power_iterations(A, steps, seed=0, shift=None)             -> (lam, x)

The start vector is the reference's (`default_rng(seed).standard_normal(n)`,
drawn on the host), the matvec is the bitwise-CSR-order stencil kernel, and
the Rayleigh quotients / norms are device reductions (not BLAS-bitwise, so
the estimates agree with the reference to ~1e-14 and the iteration count to
the tolerance test).  Iterations run in device batches; the per-step
estimates are copied back once per batch and the reference's stopping rule
(spectral.py:45-53) is applied to them in order, so the returned estimate
and count are those of the first converged step.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .operator import GpuStencilOperator, as_operator


class PowerIterationError(RuntimeError):
    """spectral.py:10-16."""

    def __init__(self, message, last_estimate, iterations):
        super().__init__(message)
        self.last_estimate = last_estimate
        self.iterations = iterations


@dataclass(frozen=True)
class SpectralBounds:
    """spectral.py:19-28."""
    lambda_max: float
    lambda_min: float
    method: str
    residual_tolerance: float

    def __post_init__(self):
        if not self.lambda_max >= self.lambda_min:
            raise ValueError(f"lambda_max={self.lambda_max} < lambda_min={self.lambda_min}")


def _matvec_dev(op, x):
    y = torch.empty_like(x)
    L.check(op._lib.rg_matvec(op.handle, L.ptr(x), L.ptr(y), L.stream_ptr()))
    return y


def _power(op: GpuStencilOperator, tol, max_iter, seed, sigma=None, monotone_check=False,
           batch=32):
    """spectral.py:31-57 on the device.  sigma: iterate on sigma*I - A."""
    n = op.P
    x0 = np.random.default_rng(seed).standard_normal(n)
    x = torch.as_tensor(x0 / np.linalg.norm(x0)).to(op.device, op.torch_dtype).reshape(1, n)
    lam_prev = 0.0
    k = 0
    change = np.inf
    while k < max_iter:
        nb = min(batch, max_iter - k)
        lams = torch.empty(nb, dtype=torch.float64, device=op.device)
        nys = torch.empty(nb, dtype=torch.float64, device=op.device)
        for q in range(nb):
            y = _matvec_dev(op, x)
            if sigma is not None:
                y = sigma * x - y
            lams[q] = torch.real(torch.vdot(x.reshape(-1), y.reshape(-1)))
            ny = torch.linalg.vector_norm(y)
            nys[q] = ny
            x = y / ny
        lam_h, ny_h = lams.cpu().numpy(), nys.cpu().numpy()
        for q in range(nb):
            k += 1
            if ny_h[q] == 0.0:
                return 0.0, 0.0
            lam_new = float(lam_h[q])
            change = abs(lam_new - lam_prev) / max(abs(lam_new), np.finfo(float).tiny)
            if monotone_check and k > 1 and lam_new < lam_prev - 1e-12 * abs(lam_prev):
                raise AssertionError("Rayleigh quotient decreased on an SPD operator")
            lam_prev = lam_new
            if k > 1 and change <= tol:
                return lam_prev, change
    raise PowerIterationError(
        f"power iteration did not converge in {max_iter} steps "
        f"(last estimate {lam_prev:.6g}, last change {change:.3g})",
        last_estimate=lam_prev, iterations=max_iter)


def estimate_lambda_max(A, tol=1e-8, max_iter=10_000, seed=0):
    """spectral.py:60-66."""
    op = as_operator(A)
    lam, change = _power(op, tol, max_iter, seed, monotone_check=True)
    return SpectralBounds(lambda_max=lam, lambda_min=lam, method="power",
                          residual_tolerance=change)


def estimate_lambda_min(A, lambda_max, tol=1e-8, max_iter=50_000, seed=0, shift_factor=1.01):
    """spectral.py:69-82: power iteration on sigma*I - A, sigma = shift_factor*lambda_max."""
    op = as_operator(A)
    sigma = shift_factor * lambda_max
    lam_s, change = _power(op, tol, max_iter, seed, sigma=sigma)
    return SpectralBounds(lambda_max=lambda_max, lambda_min=sigma - lam_s,
                          method="shifted-power", residual_tolerance=change)


def power_iterations(A, steps, seed=0, shift=None):
    """Fixed-step variant (the cfg1 '50 power iterations' recipe): the
    Rayleigh quotient after `steps` steps (of sigma*I - A when shift=sigma)."""
    op = as_operator(A)
    n = op.P
    x0 = np.random.default_rng(seed).standard_normal(n)
    x = torch.as_tensor(x0 / np.linalg.norm(x0)).to(op.device, op.torch_dtype).reshape(1, n)
    lam_t = None
    for _ in range(steps):
        y = _matvec_dev(op, x)
        if shift is not None:
            y = shift * x - y
        lam_t = torch.real(torch.vdot(x.reshape(-1), y.reshape(-1)))
        x = y / torch.linalg.vector_norm(y)
    return float(lam_t.item()), x.reshape(-1)

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
the tolerance test).  On a float64 grid operator every power step is ONE
fused launch (rg_power_steps: x = y/||y|| on load, stencil, <x,y> and
||y||^2 partials, last-CTA fixed-order finalisation), chained on the device
with no host round trip inside a batch; other square matrices take a generic
device CSR SpMV.  Iterations run in device batches; the per-step
estimates are copied back once per batch and the reference's stopping rule
(spectral.py:45-53) is applied to them in order, so the returned estimate
and count are those of the first converged step.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .errors import UnsupportedOperator
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


class _CsrDevice:
    """Device SpMV for matrices that are not a structured-grid stencil (any
    square CSR: e.g. the reference's diag(1, 2, 3) examples).  The product is
    a cuSPARSE CSR matvec through torch; the fused stencil path below is the
    one the solvers' grid operators take."""

    def __init__(self, A):
        from .operator import _csr_arrays
        nrows, ncols, indptr, indices, data = _csr_arrays(A)
        if nrows != ncols:
            raise ValueError(f"matrix is {nrows}x{ncols}, not square")
        dev = torch.device("cuda", torch.cuda.current_device())
        self.P = ncols
        self.M = torch.sparse_csr_tensor(torch.as_tensor(np.asarray(indptr, dtype=np.int64)),
                                         torch.as_tensor(np.asarray(indices, dtype=np.int64)),
                                         torch.as_tensor(np.asarray(data)), size=(nrows, ncols),
                                         device=dev)
        self.device = dev
        self.torch_dtype = self.M.dtype

    def matvec(self, x):
        return (self.M @ x.reshape(-1, 1)).reshape(x.shape)


def _operator(A):
    try:
        op = as_operator(A)
    except UnsupportedOperator:
        return _CsrDevice(A)
    if op.batch != 1:
        raise ValueError("spectral estimates take one system (spectral.py:60-82)")
    return op


def _fused(op):
    return isinstance(op, GpuStencilOperator) and op.rg_dtype == L.RG_F64


class _PowerChain:
    """Device state of a power iteration: the current (unnormalised) y and
    its norm; x = y / ny is formed inside the next fused step."""

    def __init__(self, op, seed):
        n = op.P
        x0 = np.random.default_rng(seed).standard_normal(n)
        x0 /= np.linalg.norm(x0)                      # spectral.py:40-41, on the host
        self.op = op
        self.y = torch.as_tensor(x0).to(op.device, op.torch_dtype).reshape(1, n).contiguous()
        self.ny = None                                # None: y already is x
        if _fused(op):
            self.bufs = [torch.empty_like(self.y), torch.empty_like(self.y)]

    def run(self, nb, sigma=None, want_x=False):
        """nb steps; returns (lam[nb], ny[nb]) device arrays (and x of the last step)."""
        op = self.op
        dev = op.device
        if _fused(op):
            lam = torch.empty(nb, dtype=torch.float64, device=dev)
            ny = torch.empty(nb, dtype=torch.float64, device=dev)
            y0 = self.bufs[0] if self.bufs[0].data_ptr() != self.y.data_ptr() else self.bufs[1]
            y1 = self.bufs[1] if y0 is self.bufs[0] else self.bufs[0]
            x_last = torch.empty_like(self.y) if want_x else None
            L.check(op._lib.rg_power_steps(op.handle, int(nb), L.ptr(self.y), L.ptr(self.ny),
                                           L.ptr(y0), L.ptr(y1),
                                           float(sigma if sigma is not None else 0.0),
                                           int(sigma is not None), L.ptr(lam), L.ptr(ny),
                                           L.ptr(x_last), L.stream_ptr()))
            self.y = y0 if (nb - 1) % 2 == 0 else y1
            self.ny = ny[nb - 1:nb]
            return lam, ny, x_last
        # generic device SpMV (eager torch ops)
        lams = torch.empty(nb, dtype=torch.float64, device=dev)
        nys = torch.empty(nb, dtype=torch.float64, device=dev)
        x = self.y if self.ny is None else self.y / self.ny
        for q in range(nb):
            y = op.matvec(x) if not isinstance(op, GpuStencilOperator) else _matvec_dev(op, x)
            if sigma is not None:
                y = sigma * x - y
            lams[q] = torch.real(torch.vdot(x.reshape(-1), y.reshape(-1)))
            ny = torch.linalg.vector_norm(y)
            nys[q] = ny
            self.y, self.ny = y, ny
            if q < nb - 1:
                x = y / ny
        return lams, nys, x


def _power(op, tol, max_iter, seed, sigma=None, monotone_check=False, batch=32):
    """spectral.py:31-57 on the device.  sigma: iterate on sigma*I - A."""
    chain = _PowerChain(op, seed)
    lam_prev = 0.0
    k = 0
    change = np.inf
    while k < max_iter:
        nb = min(batch, max_iter - k)
        lams, nys, _ = chain.run(nb, sigma)
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
    op = _operator(A)
    lam, change = _power(op, tol, max_iter, seed, monotone_check=True)
    return SpectralBounds(lambda_max=lam, lambda_min=lam, method="power",
                          residual_tolerance=change)


def estimate_lambda_min(A, lambda_max, tol=1e-8, max_iter=50_000, seed=0, shift_factor=1.01):
    """spectral.py:69-82: power iteration on sigma*I - A, sigma = shift_factor*lambda_max."""
    op = _operator(A)
    sigma = shift_factor * lambda_max
    lam_s, change = _power(op, tol, max_iter, seed, sigma=sigma)
    return SpectralBounds(lambda_max=lambda_max, lambda_min=sigma - lam_s,
                          method="shifted-power", residual_tolerance=change)


def power_iterations(A, steps, seed=0, shift=None):
    """Fixed-step variant (the cfg1 '50 power iterations' recipe): the
    Rayleigh quotient after `steps` steps (of sigma*I - A when shift=sigma)
    and the normalised iterate x = y / ||y|| of the last step."""
    op = _operator(A)
    if steps <= 0:
        raise ValueError("steps must be positive")
    chain = _PowerChain(op, seed)
    lams, _, _ = chain.run(int(steps), shift)
    x = (chain.y / chain.ny).reshape(-1)
    return float(lams[-1].item()), x

"""GPU drop-in for the FNS-lite hybrid iteration (fns.py:30-105) and the
orthonormal 2D DST-I (transforms.py:24-35).

    dst2(x) / dst2_inv(x)                          -> like x
    SpectralCorrection(lambda_tilde, n)            (.apply(r))
    fns_lite_step(A, f, u, schedule, M, corr)      -> u
    solve_fns(A, f, schedule, corr, M, tol, max_iters) -> (u, SolveReport)

The M smoothing steps run as one temporally blocked sweep (plain Richardson,
weights cycled mod m, no preconditioner); the correction is one residual
kernel plus three shared-memory DST line passes (rows; columns with the
symbol multiply between two transforms; rows accumulated into u).  The DST
is not bitwise pocketfft: agreement ~1e-15 relative.
"""
from __future__ import annotations

import ctypes as C
import math
import time

import numpy as np
import torch

from . import _lib as L
from .errors import DivergenceError, SolveReport
from .operator import GpuStencilOperator, as_operator
from .richardson import DeviceSchedule, _is_host, _op_for

_PLANS = {}


def dst_plan(batch, side):
    """Cached rg_dst plan (twiddles + workspace) for (batch, side)."""
    key = (batch, side, torch.cuda.current_device())
    plan = _PLANS.get(key)
    if plan is None:
        plan = _DstPlan(batch, side)
        _PLANS[key] = plan
    return plan


class _DstPlan:
    def __init__(self, batch, side):
        self.lib = L.load()
        h = C.c_void_p()
        L.check(self.lib.rg_dst_create(C.byref(h), int(batch), int(side)))
        self.h, self.batch, self.side = h, batch, side

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.rg_dst_destroy(self.h)
            self.h = None


def _as_grid_batch(x):
    """(device float64 tensor [B, s*s], batch, side, host?)"""
    host = _is_host(x)
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, dtype=np.float64))
    t = t.to(device="cuda", dtype=torch.float64)
    n = t.shape[-1] if t.ndim >= 1 else t.numel()
    side = math.isqrt(n)
    if side * side != n:
        raise ValueError(f"vector length {n} is not a perfect square")
    return t.reshape(-1, n).contiguous(), t.numel() // n, side, host


def dst2(x):
    """Orthonormal 2D DST-I of flattened interior vector(s) (transforms.py:24-30)."""
    t, B, side, host = _as_grid_batch(x)
    out = torch.empty_like(t)
    L.check(dst_plan(B, side).lib.rg_dst2(dst_plan(B, side).h, L.ptr(t), L.ptr(out),
                                          L.stream_ptr()))
    out = out.reshape(np.shape(x) if host else x.shape)
    return out.cpu().numpy() if host else out


def dst2_inv(x):
    """transforms.py:33-35 (the transform is involutory)."""
    return dst2(x)


def sine_mode(n, p, q):
    """transforms.py:38-43: the (p, q) discrete sine mode on the (n-1)^2
    interior, flattened (x the first axis)."""
    i = np.arange(1, n)
    return np.outer(np.sin(p * np.pi * i / n), np.sin(q * np.pi * i / n)).reshape(-1)


def sine_basis_eigenvalues(A, n, chunk=256):
    """fns.py:60-73: diagonal of A in the orthonormal sine basis (its exact
    eigenvalues when the basis diagonalises A).

    The reference transforms one unit vector per entry on the host.  Here a
    constant 9-point operator takes the closed form: with v_p the orthonormal
    DST-I vectors, <v_p, shift_{+-1} v_p> = cos(pi p / n), so entry (p, q) is
    sum_{a,b} c[a,b] g_a(p) g_b(q), g_0 = 1, g_{+-1} = cos(pi p / n).  Other
    operators are transformed on the device, `chunk` sine modes per batch
    (dst2(A dst2(e_k)))."""
    op = as_operator(A) if not isinstance(A, GpuStencilOperator) else A
    if op.side != n - 1:
        raise ValueError("operator and grid size differ")
    N = n - 1
    if op.kind == L.RG_CONST9:
        c = np.asarray(op._host_stencil[0], dtype=np.float64).reshape(3, 3)
        cp = np.cos(np.pi * np.arange(1, n) / n)
        g = np.stack([cp, np.ones(N), cp])           # g_a for a = -1, 0, 1
        lam = np.zeros((N, N))
        for a in range(3):
            for b in range(3):
                lam = lam + c[a, b] * np.outer(g[a], g[b])
        return lam.reshape(-1)
    if op.np_dtype != np.float64 or op.nsets != 1:
        raise ValueError("sine_basis_eigenvalues needs one real float64 operator (fns.py:60-73)")
    size = N * N
    lam = np.empty(size)
    ops = {}
    for k0 in range(0, size, chunk):
        k1 = min(size, k0 + chunk)
        kb = k1 - k0
        if kb not in ops:
            ops[kb] = op.broadcast(kb)
        idx = torch.arange(kb, device="cuda")
        E = torch.zeros((kb, size), dtype=torch.float64, device="cuda")
        E[idx, idx + k0] = 1.0
        AV = ops[kb].matvec(dst2(E))
        lam[k0:k1] = dst2(AV)[idx, idx + k0].cpu().numpy()
    return lam


class SpectralCorrection:
    """Diagonal operator in the sine basis (fns.py:30-44); the symbol lives
    on the device.  lambda_tilde: [(n-1)^2] or a batch [B, (n-1)^2]."""

    def __init__(self, lambda_tilde, n):
        lam = lambda_tilde if isinstance(lambda_tilde, torch.Tensor) else torch.as_tensor(
            np.asarray(lambda_tilde, dtype=np.float64))
        lam = lam.to(device="cuda", dtype=torch.float64)
        if lam.shape[-1] != (n - 1) ** 2:
            raise ValueError("correction length does not match the grid")
        if not bool(torch.isfinite(lam).all()):
            raise ValueError("correction entries must be finite")
        self.lam = lam.reshape(-1, (n - 1) ** 2).contiguous()
        self.n = n
        self.lambda_tilde = lambda_tilde

    def apply(self, r):
        return dst2_inv(self._times(dst2(r)))

    def _times(self, x):
        host = not isinstance(x, torch.Tensor)
        t = torch.as_tensor(x).to("cuda", torch.float64).reshape(self.lam.shape)
        y = (t * self.lam).reshape(np.shape(x) if host else x.shape)
        return y.cpu().numpy() if host else y


class FnsEngine:
    """Device state of the hybrid iteration for a batch of systems."""

    def __init__(self, op: GpuStencilOperator, schedule, corr: SpectralCorrection, M):
        if op.np_dtype != np.float64:
            raise ValueError("FNS runs in float64 (fns.py:36)")
        self.op, self.M = op, int(M)
        self.sched = DeviceSchedule(op, schedule, None)
        if self.sched.variant != "plain":
            # fns_lite_step uses omega only (fns.py:78-79)
            from .schedules import WeightSchedule
            self.sched = DeviceSchedule(op, WeightSchedule(omega=np.asarray(schedule.omega)), None)
        lam = corr.lam
        if lam.shape[0] == 1 and op.batch > 1:
            lam = lam.expand(op.batch, -1).contiguous()
        if lam.shape[0] != op.batch:
            raise ValueError("one symbol per system (or one shared) expected")
        self.lam = lam
        self.plan = dst_plan(op.batch, op.side)
        self.u = [torch.empty((op.batch, op.P), dtype=torch.float64, device=op.device)
                  for _ in range(2)]
        self.cur = 0

    def step(self, f):
        """fns_lite_step on the device iterate self.u[self.cur] (no host sync)."""
        lib = self.op._lib
        outb = C.c_int()
        if self.M > 0:
            L.check(lib.rg_sweep(self.op.handle, C.byref(self.sched.struct), 0, self.M, 0,
                                 L.ptr(self.u[self.cur]), L.ptr(self.u[self.cur ^ 1]), None, None,
                                 L.ptr(f), C.byref(outb), L.stream_ptr()))
            self.cur = self.cur ^ outb.value
        L.check(lib.rg_fns_correct(self.op.handle, self.plan.h, L.ptr(self.lam),
                                   L.ptr(self.u[self.cur]), L.ptr(f), L.stream_ptr()))
        return self.u[self.cur]


def fns_lite_step(A, f, u, schedule, M, corr: SpectralCorrection):
    """fns.py:76-84: M plain smoothing steps (omega[k % m]), one correction,
    non-finite check.  Returns u like the input."""
    op = _op_for(A, f)
    eng = FnsEngine(op, schedule, corr, M)
    host = _is_host(u)
    ft = op.to_device(f)
    eng.u[0].copy_(op.to_device(u))
    out = eng.step(ft)
    if not bool(torch.isfinite(out).all()):
        raise DivergenceError("hybrid step produced a non-finite iterate", inner_iteration=M)
    shp = np.shape(u) if host else u.shape
    out = out.reshape(shp)
    return out.cpu().numpy() if host else out.clone()


def solve_fns(A, f, schedule, corr, M, tol=1e-6, max_iters=10_000):
    """fns.py:87-105 on the device: hybrid steps from zero until the relative
    residual (one fused residual-norm per step, host-polled) reaches tol."""
    t0 = time.perf_counter()
    op = _op_for(A, f)
    host = _is_host(f)
    ft = op.to_device(f)
    eng = FnsEngine(op, schedule, corr, M)
    eng.u[0].zero_()
    fn2 = torch.linalg.vector_norm(ft, dim=1)
    fnorm = float(fn2[0].item()) if op.batch == 1 else fn2.cpu().numpy()
    if op.batch != 1:
        raise ValueError("solve_fns drives one system; use FnsEngine for batches")
    rel, trace, it = 1.0, [1.0], 0
    converged = fnorm == 0.0
    while not converged and it < max_iters:
        u = eng.step(ft)
        it += 1
        _, n2 = op.residual(u, ft, want_r=False)
        r2 = float(n2[0].item())
        if not math.isfinite(r2):
            raise DivergenceError("hybrid step produced a non-finite iterate", inner_iteration=M)
        rel = math.sqrt(r2) / fnorm
        trace.append(rel)
        converged = rel <= tol
    u = eng.u[eng.cur].reshape(-1)
    return (u.cpu().numpy() if host else u.clone()), SolveReport(
        iterations=it, inner_iterations=it * M, converged=converged,
        final_relative_residual=rel, wall_time=time.perf_counter() - t0, trace=np.array(trace))


def solve_fns_batched(A, F, schedule, corr, M, tol=1e-6, max_iters=10_000):
    """fns.py:87-105 for B independent systems at once: A a batched operator,
    F [B, P], corr one symbol per system (or one shared).  Every system stops
    on its own (its iterate is frozen at the step that reaches tol, as the
    reference's loop would leave it) while the rest of the batch goes on.
    Returns [(u_b, SolveReport_b)]."""
    t0 = time.perf_counter()
    op = _op_for(A, F)
    host = _is_host(F)
    Ft = op.to_device(F)
    B = op.batch
    eng = FnsEngine(op, schedule, corr, M)
    eng.u[0].zero_()
    fnorm = torch.linalg.vector_norm(Ft, dim=1).cpu().numpy()
    rel = np.ones(B)
    traces = [[1.0] for _ in range(B)]
    iters = np.zeros(B, dtype=np.int64)
    done = fnorm == 0.0
    final = [None] * B
    for b in np.flatnonzero(done):
        final[b] = eng.u[0][b].clone()
    it = 0
    while not done.all() and it < max_iters:
        u = eng.step(Ft)
        it += 1
        _, n2 = op.residual(u, Ft, want_r=False)
        r2 = n2.cpu().numpy()
        for b in np.flatnonzero(~done):
            if not math.isfinite(r2[b]):
                raise DivergenceError("hybrid step produced a non-finite iterate", inner_iteration=M)
            rel[b] = math.sqrt(r2[b]) / fnorm[b]
            traces[b].append(rel[b])
            iters[b] = it
            if rel[b] <= tol:
                done[b] = True
                final[b] = u[b].clone()
    out = []
    for b in range(B):
        ub = final[b] if final[b] is not None else eng.u[eng.cur][b]
        out.append(((ub.cpu().numpy() if host else ub.clone()), SolveReport(
            iterations=int(iters[b]), inner_iterations=int(iters[b]) * M,
            converged=bool(done[b]), final_relative_residual=float(rel[b]),
            wall_time=time.perf_counter() - t0, trace=np.array(traces[b]))))
    return out


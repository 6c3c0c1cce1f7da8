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
        self.norm2 = torch.empty(op.batch, dtype=torch.float64, device=op.device)

    def _third(self):
        if len(self.u) < 3:
            self.u.append(torch.empty_like(self.u[0]))

    def step(self, f, want_norm=False, keep_input=False):
        """fns_lite_step on the device iterate self.u[self.cur] (no host sync).

        want_norm: self.norm2[b] = ||f - A u_b||^2 of the INPUT iterate -- the
        residual the first smoothing step computes anyway, reduced in that
        sweep's epilogue (rg_sweep_norm): the relative residual fns.py:99
        takes after a correction costs no pass of its own, it arrives with
        the next alternation.  keep_input: the input iterate survives in its
        buffer (a third buffer takes the ping-pong), so a caller that finds
        it converged can still return it; self.prev is its index."""
        lib = self.op._lib
        outb = C.c_int()
        h, sched, s = self.op.handle, C.byref(self.sched.struct), L.stream_ptr()
        M, cur = self.M, self.cur
        self.prev = cur
        def sweep(i0, n, src, dst, norm):
            """n smoothing steps from weight index i0, ping-pong src <-> dst;
            returns the index holding the result."""
            if norm:
                L.check(lib.rg_sweep_norm(h, sched, i0, n, 0, L.ptr(self.u[src]), L.ptr(self.u[dst]),
                                          None, None, L.ptr(f), L.ptr(self.norm2), C.byref(outb), s))
            else:
                L.check(lib.rg_sweep(h, sched, i0, n, 0, L.ptr(self.u[src]), L.ptr(self.u[dst]), None,
                                     None, L.ptr(f), C.byref(outb), s))
            return src if outb.value == 0 else dst

        if M > 0 and keep_input:
            self._third()
            a, b = [i for i in range(3) if i != cur]
            # constant real stencils on grids of side >= 128 take blocked sweeps:
            # 4 steps are exactly one launch (cur -> a), the rest runs a <-> b
            if self.op.kind == L.RG_CONST9 and self.op.side >= 128:
                first = min(4, M)
                got = sweep(0, first, cur, a, want_norm)
                if got != a:
                    raise RuntimeError("blocked sweep expected to take one launch")
                cur = a if M == first else sweep(first, M - first, a, b, False)
            else:        # any other path: work on a copy
                self.u[a].copy_(self.u[cur])
                cur = sweep(0, M, a, b, want_norm)
        elif M > 0:
            cur = sweep(0, M, cur, (cur + 1) % len(self.u), want_norm)
        else:
            if want_norm:
                L.check(lib.rg_residual(h, L.ptr(self.u[cur]), L.ptr(f), None, L.ptr(self.norm2), s))
            if keep_input:
                self._third()
                a = (cur + 1) % 3
                self.u[a].copy_(self.u[cur])
                cur = a
        self.cur = cur
        L.check(lib.rg_fns_correct(h, self.plan.h, L.ptr(self.lam), L.ptr(self.u[cur]), L.ptr(f), s))
        return self.u[cur]

    def residual_norm2(self, f):
        """||f - A u||^2 of the current iterate (one residual pass)."""
        L.check(self.op._lib.rg_residual(self.op.handle, L.ptr(self.u[self.cur]), L.ptr(f), None,
                                         L.ptr(self.norm2), L.stream_ptr()))
        return self.norm2


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


def _fns_drive(eng, Ft, fnorm, tol, max_iters, M):
    """The loop of fns.py:87-105 for the engine's batch, every system stopping
    on its own.  The relative residual after alternation j is the first
    residual of alternation j + 1, so it is taken from that sweep's fused
    reduction (FnsEngine.step(want_norm=True)): alternation j + 1 runs
    speculatively, on a buffer of its own, and is discarded for a system
    that turns out to have converged at j; only the last iterate of a run
    that exhausts max_iters needs a residual pass of its own.
    Returns (final [B] of tensors or None, iters, rel, traces, done)."""
    B = eng.op.batch
    rel = np.ones(B)
    traces = [[1.0] for _ in range(B)]
    iters = np.zeros(B, dtype=np.int64)
    done = np.asarray(fnorm) == 0.0
    final = [eng.u[eng.cur][b].clone() if done[b] else None for b in range(B)]

    def record(j, r2, src):
        for b in np.flatnonzero(~done):
            if not math.isfinite(r2[b]):
                raise DivergenceError("hybrid step produced a non-finite iterate", inner_iteration=M)
            rel[b] = math.sqrt(r2[b]) / fnorm[b]
            traces[b].append(rel[b])
            iters[b] = j
            if rel[b] <= tol:
                done[b] = True
                final[b] = src[b].clone()

    it = 0
    while not done.all() and it < max_iters:
        eng.step(Ft, want_norm=it >= 1, keep_input=it >= 1)
        if it >= 1:
            record(it, eng.norm2.cpu().numpy(), eng.u[eng.prev])
            if done.all():
                break
        it += 1
    if not done.all() and it >= 1:
        record(it, eng.residual_norm2(Ft).cpu().numpy(), eng.u[eng.cur])
    return final, iters, rel, traces, done


def solve_fns(A, f, schedule, corr, M, tol=1e-6, max_iters=10_000):
    """fns.py:87-105 on the device: hybrid steps from zero until the relative
    residual (fused into the next alternation's first sweep, host-polled)
    reaches tol."""
    t0 = time.perf_counter()
    op = _op_for(A, f)
    if op.batch != 1:
        raise ValueError("solve_fns drives one system; use solve_fns_batched for batches")
    host = _is_host(f)
    ft = op.to_device(f)
    eng = FnsEngine(op, schedule, corr, M)
    eng.u[0].zero_()
    fnorm = torch.linalg.vector_norm(ft, dim=1).cpu().numpy()
    final, iters, rel, traces, done = _fns_drive(eng, ft, fnorm, tol, max_iters, M)
    u = (final[0] if final[0] is not None else eng.u[eng.cur][0]).reshape(-1)
    return (u.cpu().numpy() if host else u.clone()), SolveReport(
        iterations=int(iters[0]), inner_iterations=int(iters[0]) * M, converged=bool(done[0]),
        final_relative_residual=float(rel[0]), wall_time=time.perf_counter() - t0,
        trace=np.array(traces[0]))


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
    eng = FnsEngine(op, schedule, corr, M)
    eng.u[0].zero_()
    fnorm = torch.linalg.vector_norm(Ft, dim=1).cpu().numpy()
    final, iters, rel, traces, done = _fns_drive(eng, Ft, fnorm, tol, max_iters, M)
    out = []
    for b in range(op.batch):
        ub = final[b] if final[b] is not None else eng.u[eng.cur][b]
        out.append(((ub.cpu().numpy() if host else ub.clone()), SolveReport(
            iterations=int(iters[b]), inner_iterations=int(iters[b]) * M,
            converged=bool(done[b]), final_relative_residual=float(rel[b]),
            wall_time=time.perf_counter() - t0, trace=np.array(traces[b]))))
    return out

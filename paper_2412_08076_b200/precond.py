"""GPU drop-in for the reference preconditioners (precond.py:47-129) and the
solve loop preconditioned by Gauss-Seidel / SOR / SSOR (SURVEY.md §8(f)
item 1).

    Preconditioner.identity() / .weighted_jacobi(A, relax=2/3)
                  / .gauss_seidel(A) / .sor(A, relax) / .ssor(A, relax=1.0)
    P.apply(r), P(r)                            -> B^{-1} r on the device
    solve_stationary(..., P=<GS/SOR/SSOR>)      -> routed here by richardson.py

The triangular maps are hand-written wavefront substitutions
(csrc/tri.cuh, `rg_tri_apply`).  They agree with the reference's SuperLU
substitutions to rounding (~1e-15); the reference holds these maps to 1e-13
against dense solves (test_precond.py:33-62), and that is the parity bar
(solve traces then agree to ~1e-12, not bitwise).  Reference Preconditioner
objects of these kinds are accepted too: their kind and relax select the
GPU map, built from the operator the solve is given (the reference builds P
from that same A).
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np
import torch

from . import _lib as L
from .errors import DivergenceError, SolveReport, UnsupportedOperator
from .operator import GpuStencilOperator, JacobiScale, ZeroDiagonalError, as_operator

DIVERGENCE_FACTOR = 1e12  # richardson.py:17

_TRI_KINDS = {"gauss-seidel": L.RG_TRI_SOR, "sor": L.RG_TRI_SOR, "ssor": L.RG_TRI_SSOR}


class TriangularPreconditioner:
    """Gauss-Seidel / SOR / SSOR map of one (batched) operator."""

    def __init__(self, op: GpuStencilOperator, kind: str, relax: float):
        if kind not in _TRI_KINDS:
            raise ValueError(f"unknown triangular preconditioner {kind!r}")
        if kind == "gauss-seidel":
            relax = 1.0
        name = "SSOR" if kind == "ssor" else "SOR"
        if not 0.0 < relax < 2.0:
            raise ValueError(f"{name} relaxation must be in (0, 2), got {relax}")
        # any operator the reference builds these maps for (precond.py:86-118):
        # constant real stencils take the cluster wavefront (csrc/tri.cuh),
        # per-node / complex coefficients the general one (csrc/trigen.cuh)
        for b in range(op.nsets):
            d = op.diagonal(b)
            if np.any(d == 0):
                raise ZeroDiagonalError(int(np.flatnonzero(d == 0)[0]))
        self.op = op
        self.kind = kind
        self.relax = None if kind == "gauss-seidel" else float(relax)
        self._relax = float(relax)
        self.mode = _TRI_KINDS[kind]

    def apply_device(self, r, z=None, work=None, transpose=False):
        """z = B^{-1} r (or B^{-T} r) for device tensors [B, P]."""
        op = self.op
        z = torch.empty_like(r) if z is None else z
        mode = self.mode
        if transpose:
            mode = L.RG_TRI_SSOR_T if mode == L.RG_TRI_SSOR else L.RG_TRI_SOR_T
        if mode in (L.RG_TRI_SSOR, L.RG_TRI_SSOR_T) and work is None:
            work = torch.empty_like(r)
        L.check(op._lib.rg_tri_apply(op.handle, mode, self._relax, L.ptr(r), L.ptr(z),
                                     L.ptr(work), L.stream_ptr()))
        return z

    def _host_apply(self, r, transpose):
        host = not (isinstance(r, torch.Tensor) and r.is_cuda)
        rd = self.op.to_device(r)
        z = self.apply_device(rd.reshape(self.op.batch, self.op.P), transpose=transpose)
        z = z.reshape(rd.shape)
        return z.cpu().numpy().reshape(np.shape(r)) if host else z

    def apply(self, r):
        """B^{-1} r (precond.py:56-57)."""
        return self._host_apply(r, False)

    def apply_transpose(self, r):
        """B^{-T} r (precond.py:59-61, used by reverse-mode differentiation)."""
        return self._host_apply(r, True)

    __call__ = apply


class Preconditioner:
    """Constructors with the reference's names (precond.py:59-118)."""

    @staticmethod
    def identity():
        return None

    @staticmethod
    def weighted_jacobi(A, relax=2.0 / 3.0):
        return JacobiScale.weighted_jacobi(A, relax)

    @staticmethod
    def gauss_seidel(A):
        return TriangularPreconditioner(as_operator(A), "gauss-seidel", 1.0)

    @staticmethod
    def sor(A, relax):
        return TriangularPreconditioner(as_operator(A), "sor", relax)

    @staticmethod
    def ssor(A, relax=1.0):
        return TriangularPreconditioner(as_operator(A), "ssor", relax)


def apply_preconditioner(P, r):
    """precond.py:125-129: B^{-1} r for a built preconditioner (identity for
    None).  Device tensors stay on the device."""
    if P is None:
        return r if isinstance(r, torch.Tensor) else np.asarray(r)
    return P.apply(r)


def tri_spec(P):
    """(kind, relax) when P is a GS / SOR / SSOR map (ours or richlab's), else None."""
    if isinstance(P, TriangularPreconditioner):
        return P.kind, P._relax
    kind = getattr(P, "kind", None)
    if kind in _TRI_KINDS and hasattr(P, "apply"):
        relax = getattr(P, "relax", None)
        return kind, 1.0 if relax is None else float(relax)
    return None


def solve_tri(op: GpuStencilOperator, F, schedules, kind, relax, tol=1e-6, max_outer=100_000,
              u0=None, check="outer"):
    """solve_stationary (richardson.py:77-141) for every system of `op`
    with z = B^{-1} r from the triangular map.  Per inner step:
    rg_tri_apply (z), rg_precond_update (v, u and the next look-ahead), and
    the residual/norm kernel wherever the reference computes one; one host
    sync per outer sweep (per inner step for check="inner").  Returns
    [(u_b, SolveReport) | (None, DivergenceError)]."""
    from .richardson import DeviceSchedule, _is_host
    t0 = time.perf_counter()
    lib, s = op._lib, L.stream_ptr
    B, P = op.batch, op.P
    pre = TriangularPreconditioner(op, kind, relax)
    ds = DeviceSchedule(op, schedules)
    m = ds.m
    nag = ds.variant in ("nag", "nagex")
    reuse = not nag                       # richardson.py:101-103
    like_numpy = _is_host(F)
    mk = lambda: torch.empty((B, P), dtype=op.torch_dtype, device=op.device)  # noqa: E731
    f = op.to_device(F).reshape(B, P).contiguous()
    u = mk()
    if u0 is None:
        u.zero_()
    else:
        u.copy_(op.to_device(u0).reshape(B, P))
    v = torch.zeros_like(u)
    r, z = mk(), mk()
    work = mk() if pre.mode == L.RG_TRI_SSOR else None
    y = mk() if nag else None
    sched = C.byref(ds.struct)
    n2 = torch.empty((m + 2, B), dtype=torch.float64, device=op.device)
    L.check(lib.rg_residual(op.handle, L.ptr(torch.zeros_like(u)), L.ptr(f), None,
                            L.ptr(n2[m]), s()))                          # ||f||
    L.check(lib.rg_residual(op.handle, L.ptr(u), L.ptr(f), L.ptr(r), L.ptr(n2[m + 1]), s()))
    h0 = np.sqrt(n2[m:].cpu().numpy())
    fnorm = h0[0]

    done = [None] * B            # (u_b or None, SolveReport | DivergenceError)
    trace = [[] for _ in range(B)]
    inner = [0] * B
    rel = np.zeros(B)
    thr = np.zeros(B)
    for b in range(B):
        if fnorm[b] == 0.0:      # richardson.py:95-99
            done[b] = (u[b].clone(), SolveReport(0, 0, True, 0.0, 0.0, np.array([0.0])))
            continue
        rel[b] = h0[1, b] / fnorm[b]
        trace[b].append(rel[b])
        thr[b] = DIVERGENCE_FACTOR * max(trace[b][0], 1.0)
        if rel[b] <= tol:
            done[b] = (u[b].clone(), SolveReport(0, 0, True, float(rel[b]), 0.0,
                                                 np.array(trace[b])))
    norm_at = [reuse or check == "inner" or i == m - 1 for i in range(m)]
    outer = 0

    def step(b, hb):
        """One inner step of system b with squared norm hb (None: no check);
        True when b finished (richardson.py:122-131)."""
        inner[b] += 1
        if hb is None:
            return False
        rel[b] = np.sqrt(hb) / fnorm[b]
        if not np.isfinite(rel[b]) or rel[b] > thr[b]:
            done[b] = (None, DivergenceError(
                f"residual blew up to {rel[b]:.3g} at inner iteration {inner[b]}",
                inner_iteration=inner[b]))
            return True
        if check == "inner" and rel[b] <= tol:
            trace[b].append(rel[b])
            done[b] = (u[b].clone(), SolveReport(outer + 1, inner[b], True, float(rel[b]), 0.0,
                                                 np.array(trace[b])))
            return True
        return False

    if nag and any(d is None for d in done):
        L.check(lib.rg_precond_update(op.handle, sched, 0, None, L.ptr(u), L.ptr(v), L.ptr(y), s()))
    while outer < max_outer and any(d is None for d in done):
        live = [b for b in range(B) if done[b] is None]
        for i in range(m):
            if nag:   # residual at the look-ahead point (richardson.py:118-119)
                L.check(lib.rg_residual(op.handle, L.ptr(y), L.ptr(f), L.ptr(r), None, s()))
            pre.apply_device(r, z, work)
            L.check(lib.rg_precond_update(op.handle, sched, i, L.ptr(z), L.ptr(u), L.ptr(v),
                                          L.ptr(y) if nag else None, s()))
            if norm_at[i]:
                L.check(lib.rg_residual(op.handle, L.ptr(u), L.ptr(f),
                                        L.ptr(r) if reuse else None, L.ptr(n2[i]), s()))
            if check == "inner":
                hi = n2[i].cpu().numpy()
                live = [b for b in live if not step(b, hi[b])]
                if not live:
                    break
        if check == "outer":
            hs = n2[:m].cpu().numpy()
            nxt = []
            for b in live:
                if not any(step(b, hs[i, b] if norm_at[i] else None) for i in range(m)):
                    nxt.append(b)
            live = nxt
        for b in live:       # sweep end (richardson.py:133-135)
            trace[b].append(rel[b])
            if rel[b] <= tol:
                done[b] = (u[b].clone(), SolveReport(outer + 1, inner[b], True, float(rel[b]),
                                                     0.0, np.array(trace[b])))
        outer += 1
    wall = time.perf_counter() - t0
    out = []
    for b in range(B):
        if done[b] is None:      # max_outer sweeps without convergence
            done[b] = (u[b].clone(), SolveReport(outer, inner[b], False, float(rel[b]), 0.0,
                                                 np.array(trace[b])))
        ub, rep = done[b]
        if isinstance(rep, DivergenceError):
            out.append((None, rep))
            continue
        rep.wall_time = wall
        out.append((ub.cpu().numpy() if like_numpy else ub, rep))
    return out


def tri_inner_update(op, f, u, v, i, schedule, spec):
    """_inner_update (richardson.py:49-59) with a GS / SOR / SSOR map."""
    from .richardson import DeviceSchedule, _is_host, _out
    host = _is_host(u)
    shp = np.shape(u) if host else u.shape
    B, P = op.batch, op.P
    ds = DeviceSchedule(op, schedule)
    pre = TriangularPreconditioner(op, *spec)
    ut = op.to_device(u).reshape(B, P).clone()
    vt = op.to_device(v).reshape(B, P).clone()
    ft = op.to_device(f).reshape(B, P)
    sched = C.byref(ds.struct)
    lib, s = op._lib, L.stream_ptr
    x = ut
    if ds.variant in ("nag", "nagex"):
        x = torch.empty_like(ut)
        L.check(lib.rg_precond_update(op.handle, sched, int(i), None, L.ptr(ut), L.ptr(vt),
                                      L.ptr(x), s()))
    r = torch.empty_like(ut)
    L.check(lib.rg_residual(op.handle, L.ptr(x), L.ptr(ft), L.ptr(r), None, s()))
    z = pre.apply_device(r)
    L.check(lib.rg_precond_update(op.handle, sched, int(i), L.ptr(z), L.ptr(ut), L.ptr(vt),
                                  None, s()))
    return _out(ut.reshape(shp), host), _out(vt.reshape(shp), host)

"""GPU drop-in for the V-cycle (multigrid.py:71-163).

    build_hierarchy(A, n, coarsest=8, schedules=None, batch=1) -> GpuHierarchy
    GpuHierarchy.from_reference(h, batch=1)    (a richlab Hierarchy)
    v_cycle(h, f, u=None, pre=1, post=1)       -> u like f

Host setup (Galerkin R A P products, coarsest LU) is one-time host work,
as in the reference (out of the hot path); it uses SciPy
exactly like multigrid.py so the coarse operators are the reference's bit
for bit.  Per cycle everything runs on the device:

  smoother      rg_sweep, NAG/plain with fresh v and no preconditioner
                (multigrid.py:126-138); 5-point Helmholtz fine level, 9-point
                variable-coefficient Galerkin levels
  residual      rg_residual (CSR-order stencil)
  transfers     rg_restrict / rg_prolong_add (bitwise = R.matvec / P.matvec)
  coarsest      rg_dense_apply with the precomputed inverse of the coarsest
                operator (replaces lu_solve; ~1e-15 relative)

A hierarchy serves `batch` right-hand sides of the same operator at once
(the coefficient planes are shared, not replicated).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import torch

from . import _lib as L
from .errors import DivergenceError
from .operator import GpuStencilOperator, default_device, extract_planes, classify
from .richardson import DeviceSchedule, _is_host


class CoarseSolveError(RuntimeError):
    """multigrid.py:20-21."""


def _fw1d(n):
    if n % 2 != 0:   # multigrid.py:26-27
        raise ValueError(f"grid side {n} must be even to coarsen")
    nc = n // 2
    r = np.repeat(np.arange(nc - 1), 3)
    c = (2 * np.arange(nc - 1)[:, None] + np.arange(3)[None, :]).reshape(-1)
    return sp.csr_matrix((np.tile([0.25, 0.5, 0.25], nc - 1), (r, c)), shape=(nc - 1, n - 1))


def _canonical(M):
    M = sp.csr_matrix(M)
    M.sum_duplicates()
    M.sort_indices()
    M.eliminate_zeros()
    return M


def restriction_matrix(n):
    """multigrid.py:39-42 (host, for setup and checks)."""
    r1 = _fw1d(n)
    return _canonical(sp.kron(r1, r1, format="csr"))


def prolongation_matrix(n):
    """multigrid.py:45-49."""
    p1 = (2.0 * _fw1d(n).T).tocsr()
    return _canonical(sp.kron(p1, p1, format="csr"))


def _transfer(x, n, coarse_side, fn):
    """Shared body of restrict / prolong: flat vector(s) -> device kernel."""
    if n % 2 != 0:
        raise ValueError(f"grid side {n} must be even to coarsen")
    host = _is_host(x)
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
    cplx = t.is_complex()
    t = t.to(device=default_device(), dtype=torch.complex128 if cplx else torch.float64)
    fine_p, coarse_p = (n - 1) ** 2, (n // 2 - 1) ** 2
    src_p, dst_p = (fine_p, coarse_p) if coarse_side else (coarse_p, fine_p)
    if t.shape[-1] != src_p:
        raise ValueError(f"vector length {t.shape[-1]} does not match the n={n} grid")
    lead = t.shape[:-1]
    src = t.reshape(-1, src_p).contiguous()
    dst = torch.zeros((src.shape[0], dst_p), dtype=src.dtype, device=src.device)
    dt = L.RG_C128 if cplx else L.RG_F64
    L.check(fn(dt, src.shape[0], n, L.ptr(src), L.ptr(dst), L.stream_ptr()))
    out = dst.reshape(*lead, dst_p)
    return out.cpu().numpy() if host else out


def restrict(fine, n):
    """multigrid.py:52-54: full-weighting restriction of a flat (n-1)^2
    interior vector (or a batch [..., (n-1)^2]) to the n/2 grid, on the
    device (bitwise R.matvec)."""
    return _transfer(fine, n, True, L.load().rg_restrict)


def prolong(coarse, n):
    """multigrid.py:57-59: bilinear interpolation of a flat (n/2-1)^2 vector
    up to the n grid, on the device (bitwise P.matvec)."""
    return _transfer(coarse, n, False, L.load().rg_prolong_add)


def _csr(A):
    if hasattr(A, "to_scipy"):
        return _canonical(A.to_scipy())
    return _canonical(A)


class GpuLevel:
    def __init__(self, n, op, sched):
        self.n, self.op, self.sched = n, op, sched


class GpuHierarchy:
    """Device hierarchy for `batch` right-hand sides (multigrid.py:80-87)."""

    def __init__(self, levels_csr, ns, coarsest_lu, schedules, batch=1, device=None):
        self.device = torch.device(device) if device is not None else default_device()
        self.batch = int(batch)
        if schedules is not None and not isinstance(schedules, (list, tuple)):
            schedules = [schedules] * (len(levels_csr) - 1)
        self.levels = []
        for k, (Ak, nk) in enumerate(zip(levels_csr, ns)):
            s, planes, present = extract_planes(Ak)
            kind, data = classify(s, planes, present)
            dt = planes.dtype if np.iscomplexobj(planes) else np.dtype(np.float64)
            if kind == "const9":
                op = GpuStencilOperator("const9", s, data[None], None, dt, self.device, batch=batch)
            elif kind == "diag5":
                off, dg = data
                op = GpuStencilOperator("diag5", s, off[None], dg[None], dt, self.device, batch=batch)
            else:
                op = GpuStencilOperator("var9", s, planes[None], None, dt, self.device, batch=batch)
            sched = None
            if schedules is not None and k < len(levels_csr) - 1 and k < len(schedules) \
                    and schedules[k] is not None:
                sched = DeviceSchedule(op, schedules[k], None)
            self.levels.append(GpuLevel(nk, op, sched))
        self.dtype = self.levels[0].op.np_dtype
        self.tdtype = self.levels[0].op.torch_dtype
        nc = self.levels[-1].op.P
        inv = scipy.linalg.lu_solve(coarsest_lu, np.eye(nc, dtype=self.dtype))
        if not np.all(np.isfinite(inv)):
            raise CoarseSolveError("coarsest solve failed: non-finite inverse")
        self.coarse_inv = torch.as_tensor(np.ascontiguousarray(inv)).to(self.device)
        self.lib = L.load()
        self._ws = {}

    @property
    def depth(self):
        return len(self.levels)

    @classmethod
    def from_reference(cls, h, batch=1, device=None):
        """Device copy of a richlab Hierarchy (levels' A, n, schedule; coarsest_lu)."""
        return cls([lvl.A for lvl in h.levels], [lvl.n for lvl in h.levels], h.coarsest_lu,
                   [lvl.schedule for lvl in h.levels[:-1]], batch=batch, device=device)

    # ---- device V-cycle ---------------------------------------------------
    def _buf(self, key, k):
        t = self._ws.get((key, k))
        if t is None:
            t = torch.empty((self.batch, self.levels[k].op.P), dtype=self.tdtype,
                            device=self.device)
            self._ws[(key, k)] = t
        return t

    def _smooth(self, k, f, u, count, u_zero=False):
        """multigrid.py:126-138 on the device; returns the tensor holding u.
        The momentum starts at zero (:128) and, with u_zero, so does the
        iterate: rg_sweep_from_zero is told instead of clearing the buffers
        (the fine-level vectors are 67 MB each at 4 x 1023^2 c128)."""
        lvl = self.levels[k]
        if count == 0 or lvl.sched is None:
            if u_zero:
                u.zero_()
            return u
        m = lvl.sched.m
        v0, v1 = self._buf("v0", k), self._buf("v1", k)
        other = self._buf("ua", k) if u.data_ptr() != self._buf("ua", k).data_ptr() else self._buf("ub", k)
        outb = C.c_int()
        L.check(self.lib.rg_sweep_from_zero(lvl.op.handle, C.byref(lvl.sched.struct), 0, count * m, 0,
                                            L.ptr(u), L.ptr(other), L.ptr(v0), L.ptr(v1), L.ptr(f),
                                            1 | (2 if u_zero else 0), C.byref(outb), L.stream_ptr()))
        return u if outb.value == 0 else other

    def _level(self, k, f, u, pre, post, u_zero=False):
        lib, s = self.lib, L.stream_ptr()
        if k == self.depth - 1:
            y = self._buf("y", k)
            L.check(lib.rg_dense_apply(self.levels[k].op.rg_dtype, self.batch, self.levels[k].op.P,
                                       L.ptr(self.coarse_inv), 1, L.ptr(f), L.ptr(y), s))
            return y
        lvl = self.levels[k]
        u = self._smooth(k, f, u, pre, u_zero=u_zero)
        r = self._buf("r", k)
        L.check(lib.rg_residual(lvl.op.handle, L.ptr(u), L.ptr(f), L.ptr(r), None, s))
        fc = self._buf("f", k + 1)
        L.check(lib.rg_restrict(lvl.op.rg_dtype, self.batch, lvl.n, L.ptr(r), L.ptr(fc), s))
        uc = self._buf("ua", k + 1)            # zero coarse guess (multigrid.py:154)
        ec = self._level(k + 1, fc, uc, pre, post, u_zero=True)
        L.check(lib.rg_prolong_add(lvl.op.rg_dtype, self.batch, lvl.n, L.ptr(ec), L.ptr(u), s))
        return self._smooth(k, f, u, post)

    use_graphs = True

    def _cycle(self, zero_u, pre, post):
        ud = self._buf("ua", 0)
        return self._level(0, self._buf("f", 0), ud, pre, post, u_zero=zero_u)

    def apply(self, f, u=None, pre=1, post=1, check=True, clone=True):
        """One V-cycle on device tensors f, u [batch, P0]; returns a new tensor.
        check=False skips the host-synchronising non-finite test of
        multigrid.py:135-137 (callers that test later, e.g. the pipelined
        FGMRES, which checks whenever a Hessenberg column is not finite).

        The ~200 launches of a cycle (smoother steps, residuals, transfers on
        7 levels) are captured once into a CUDA graph per (u given, pre,
        post) and replayed: the inputs are copied into the hierarchy's fixed
        buffers first, so every replay sees the same pointers."""
        fd = self._buf("f", 0)
        fd.copy_(f.reshape(fd.shape))
        if u is not None:
            self._buf("ua", 0).copy_(u.reshape(fd.shape))
        key = (u is None, pre, post)
        graphs = self.__dict__.setdefault("_graphs", {})
        if self.use_graphs and key not in graphs:
            self._cycle(u is None, pre, post)            # eager warm-up: buffers, attributes
            if u is not None:
                self._buf("ua", 0).copy_(u.reshape(fd.shape))
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    out_g = self._cycle(u is None, pre, post)
                graphs[key] = (g, out_g)
            except Exception:  # noqa: BLE001  capture unsupported here: stay eager
                self.use_graphs = False
        if self.use_graphs and key in graphs:
            g, out = graphs[key]
            g.replay()
        else:
            out = self._cycle(u is None, pre, post)
        # clone=False hands out the hierarchy's own buffer, valid until the next
        # apply (the FGMRES driver consumes it at once: matvec, store into Z)
        res = out.clone() if clone else out
        if check and not bool(torch.isfinite(res).all()):
            m = self.levels[0].sched.m if self.levels[0].sched is not None else 0
            raise DivergenceError("smoother produced a non-finite iterate",
                                  inner_iteration=pre * m)
        return res


def build_hierarchy(A, n, coarsest=8, schedules=None, batch=1, device=None):
    """multigrid.py:90-123: Galerkin-coarsen by 2 down to `coarsest` on the
    host (SciPy, as the reference), then move every level to the device."""
    if n < 2 * coarsest:
        raise ValueError(f"n={n} leaves no room to coarsen to {coarsest}")
    levels, ns, side, Al = [], [], n, _csr(A)
    while side > coarsest:
        R, P = restriction_matrix(side), prolongation_matrix(side)
        levels.append(Al)
        ns.append(side)
        Al = _canonical((R @ Al @ P).tocsr())
        side //= 2
    levels.append(Al)
    ns.append(side)
    if (side - 1) ** 2 > 1024:
        raise ValueError("coarsest level exceeds the direct-solve budget")
    try:
        lu = scipy.linalg.lu_factor(Al.toarray())
    except (ValueError, scipy.linalg.LinAlgError) as exc:
        raise CoarseSolveError(f"coarsest factorization failed: {exc}")
    if not np.all(np.isfinite(lu[0])):
        raise CoarseSolveError("coarsest factorization produced non-finite factors "
                               "(singular coarse operator)")
    return GpuHierarchy(levels, ns, lu, schedules, batch=batch, device=device)


def v_cycle(h: GpuHierarchy, f, u=None, pre=1, post=1):
    """multigrid.py:141-148: one V-cycle; numpy in -> numpy out."""
    host = _is_host(f)
    ft = torch.as_tensor(np.asarray(f) if host else f)
    ut = None if u is None else torch.as_tensor(np.asarray(u) if _is_host(u) else u)
    cplx = ft.is_complex() or (ut is not None and ut.is_complex())
    if cplx and not h.tdtype.is_complex:
        # the reference promotes to complex (multigrid.py:144) and runs the
        # real hierarchy on complex vectors.  Every operation of the cycle is
        # real-linear with real coefficients, and (a + 0j) * x equals the
        # component-wise real products, so the real and imaginary parts are
        # two independent real V-cycles (same values as the promoted run).
        ft = ft.to(torch.complex128)
        ut = None if ut is None else ut.to(torch.complex128)
        re = h.apply(ft.real.to(h.device, h.tdtype),
                     None if ut is None else ut.real.to(h.device, h.tdtype), pre, post)
        im = h.apply(ft.imag.to(h.device, h.tdtype),
                     None if ut is None else ut.imag.to(h.device, h.tdtype), pre, post)
        out = torch.complex(re, im)
    else:
        ft = ft.to(h.device, h.tdtype)
        ut = None if ut is None else ut.to(h.device, h.tdtype)
        out = h.apply(ft, ut, pre, post)
    shp = np.shape(f) if host else f.shape
    out = out.reshape(shp)
    return out.cpu().numpy() if host else out

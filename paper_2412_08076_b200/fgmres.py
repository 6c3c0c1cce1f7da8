"""GPU FGMRES driver (fgmres.py:18-131) for the multilevel solves.

    fgmres(A, f, precond_apply=None, cfg=None, u0=None) -> (u, SolveReport)
    fgmres_batched(A, F, precond_apply=None, cfg=None)   -> [(u, SolveReport)]

The driver stays host Python as in the reference (FGMRES is
not on the hot path); vectors, the operator, modified Gram-Schmidt and the
preconditioner (e.g. the device V-cycle) live on the GPU, while the small
Hessenberg / Givens recurrences run on the host exactly as fgmres.py:81-97
writes them (one device->host copy of the new Hessenberg column per Arnoldi
step).  The batched form runs B independent FGMRES state machines in
lockstep so that one batched preconditioner application serves all of them
per step; each system keeps its own restart position and stops on its own.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .errors import SolveReport
from .operator import GpuStencilOperator
from .richardson import _is_host, _op_for


@dataclass
class FgmresConfig:
    """fgmres.py:18-28."""
    restart: int = 20
    tol: float = 1e-6
    max_outer: int = 100

    def __post_init__(self):
        if self.restart < 1:
            raise ValueError("restart must be >= 1")
        if self.tol <= 0:
            raise ValueError("tol must be positive")


class _Sys:
    """Per-system FGMRES state (the locals of fgmres.py:31-131).  The Krylov
    bases live in the batched tensors V [B, mr+1, n], Z [B, mr, n]."""

    def __init__(self, b, V, Z, mr, npdt):
        self.b, self.V, self.Z, self.mr, self.npdt = b, V, Z, mr, npdt
        self.trace = []
        self.total = 0
        self.outer = 0
        self.converged = False
        self.stagnated = False
        self.done = False

    def start_cycle(self, r, beta):
        mr, dt = self.mr, self.npdt
        self.cycle_start_rel = self.rel
        self.H = np.zeros((mr + 1, mr), dtype=dt)
        self.cs = np.zeros(mr, dtype=dt)
        self.sn = np.zeros(mr, dtype=dt)
        self.g = np.zeros(mr + 1, dtype=dt)
        self.V[self.b].zero_()
        self.Z[self.b].zero_()
        self.V[self.b, 0] = r / beta
        self.g[0] = beta
        self.k = 0


def fgmres_batched(A, F, precond_apply=None, cfg: FgmresConfig = None, U0=None):
    """B independent FGMRES solves sharing batched operator/preconditioner
    calls.  Modified Gram-Schmidt is vectorised across the systems that sit
    at the same Arnoldi index (the common case): per orthogonalisation index
    one batched dot and one batched update for all of them, each system
    still orthogonalised in the reference's order (fgmres.py:76-78)."""
    cfg = cfg or FgmresConfig()
    op = A if isinstance(A, GpuStencilOperator) else _op_for(A, F)
    host = _is_host(F)
    t0 = time.perf_counter()
    B, n = op.batch, op.P
    Fd = op.to_device(F)
    npdt = op.np_dtype
    mr = cfg.restart
    precond = precond_apply if precond_apply is not None else (lambda r: r)
    U = torch.zeros_like(Fd) if U0 is None else op.to_device(U0).clone()
    V = torch.zeros((B, mr + 1, n), dtype=op.torch_dtype, device=op.device)
    Z = torch.zeros((B, mr, n), dtype=op.torch_dtype, device=op.device)
    fn = torch.linalg.vector_norm(Fd, dim=1).cpu().numpy()
    systems = [_Sys(b, V, Z, mr, npdt) for b in range(B)]
    Rr = Fd - _matvec(op, U)
    beta = torch.linalg.vector_norm(Rr, dim=1).cpu().numpy()
    for b, s in enumerate(systems):
        if fn[b] == 0.0:
            s.done, s.converged, s.rel, s.trace = True, True, 0.0, [0.0]
            continue
        s.fnorm = float(fn[b])
        s.rel = float(beta[b]) / s.fnorm
        s.trace = [s.rel]
        s.converged = s.rel <= cfg.tol
        s.done = s.converged or cfg.max_outer <= 0
        if not s.done:
            s.start_cycle(Rr[b], float(beta[b]))
    while not all(s.done for s in systems):
        # ---- one Arnoldi step for every running system (fgmres.py:349-385)
        run = [s for s in systems if not s.done]
        ks = torch.tensor([s.k if not s.done else 0 for s in systems], device=op.device)
        Vk = V[torch.arange(B, device=op.device), ks]
        for s in systems:
            if s.done:
                Vk[s.b].zero_()
        Zk = precond(Vk)
        Zk = (Zk if isinstance(Zk, torch.Tensor) else torch.as_tensor(np.asarray(Zk))).to(
            op.device, op.torch_dtype).reshape(B, n)
        W = _matvec(op, Zk)
        hcols, hk1s = {}, {}
        # group running systems by Arnoldi index
        groups = {}
        for s in run:
            groups.setdefault(s.k, []).append(s.b)
        for k, bs in groups.items():
            full = len(bs) == B
            idx = None if full else torch.tensor(bs, device=op.device)
            if full:
                Z[:, k] = Zk
                # modified Gram-Schmidt (:76-78) with the fused device kernel:
                # one pass per index applies the previous projection and takes
                # the next inner product (rg_mgs_step)
                w = W.contiguous()
                hbuf = torch.empty((k + 1, B), dtype=op.torch_dtype, device=op.device)
                n2 = torch.empty(B, dtype=torch.float64, device=op.device)
                ld = (mr + 1) * n
                code = L.RG_C128 if op.torch_dtype == torch.complex128 else L.RG_F64
                L.check(op._lib.rg_mgs_arnoldi(code, B, n, L.ptr(w), n, L.ptr(V), ld, k,
                                               L.ptr(hbuf), L.ptr(n2), L.stream_ptr()))
                hk1 = torch.sqrt(n2)
                H = hbuf.t()                                  # [G, k+1]
            else:
                w = W.index_select(0, idx)                    # [G, n]
                Z[idx, k] = Zk.index_select(0, idx)
                hs = []
                for i in range(k + 1):                        # modified Gram-Schmidt (:76-78)
                    vi = V[idx, i]
                    h = torch.linalg.vecdot(vi, w)            # conj(v_i) . w  (np.vdot)
                    w = w - h[:, None] * vi
                    hs.append(h)
                hk1 = torch.linalg.vector_norm(w, dim=1)
                H = torch.stack(hs, dim=1)                     # [G, k+1]
            # one device->host copy per group: [G, k+2] = (h_0..h_k, ||w||)
            Hh = torch.cat([H, hk1.to(H.dtype)[:, None]], dim=1).cpu().numpy()
            for q, b in enumerate(bs):
                hcols[b] = Hh[q, :k + 1]
                hk1s[b] = float(np.real(Hh[q, k + 1]))
                systems[b]._w = w[q]
        hcol_h = {b: (hcols[b], hk1s[b]) for b in hcols}
        for s in run:
            hc, hk1 = hcol_h[s.b]
            k, H, cs, sn, g = s.k, s.H, s.cs, s.sn, s.g
            H[:k + 1, k] = hc
            H[k + 1, k] = hk1
            for i in range(k):                  # stored Givens rotations (:81-85)
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -np.conj(sn[i]) * H[i, k] + np.conj(cs[i]) * H[i + 1, k]
                H[i, k] = t
            denom = np.sqrt(np.abs(H[k, k]) ** 2 + np.abs(hk1) ** 2)   # new rotation (:86-93)
            if denom == 0.0:
                cs[k], sn[k] = 1.0, 0.0
            else:
                cs[k] = np.conj(H[k, k]) / denom
                sn[k] = np.conj(H[k + 1, k]) / denom
            H[k, k] = cs[k] * H[k, k] + sn[k] * H[k + 1, k]
            H[k + 1, k] = 0.0
            g[k + 1] = -np.conj(sn[k]) * g[k]
            g[k] = cs[k] * g[k]
            s.total += 1
            s.rel = float(np.abs(g[k + 1])) / s.fnorm
            s.trace.append(s.rel)
            happy = hk1 <= 1e-14 * max(1.0, float(np.abs(H[k, k])))
            s.k = k + 1
            if s.rel <= cfg.tol or happy:
                s.converged = True
                end_cycle = True
            else:
                if hk1 > 0:
                    V[s.b, s.k] = s._w / hk1
                end_cycle = s.k >= s.mr
            if end_cycle:
                _finish_cycle(op, Fd, U, s.b, s, cfg)
    wall = time.perf_counter() - t0
    Uo = U.cpu().numpy() if host else U
    return [(Uo[b], SolveReport(iterations=s.total, inner_iterations=s.total,
                                converged=s.converged, final_relative_residual=s.rel,
                                wall_time=wall, trace=np.array(s.trace), stagnated=s.stagnated))
            for b, s in enumerate(systems)]


def _finish_cycle(op, Fd, U, b, s, cfg):
    """Update, true residual, stagnation test (fgmres.py:386-404)."""
    k = s.k
    Hk = np.triu(s.H[:k, :k])
    if k == 0:
        y = np.zeros(0, dtype=s.npdt)
    else:
        try:
            y = np.linalg.solve(Hk, s.g[:k])
        except np.linalg.LinAlgError:
            y = np.linalg.lstsq(Hk, s.g[:k], rcond=None)[0]
    yt = torch.as_tensor(y).to(U.device, U.dtype)
    U[b] = U[b] + yt @ s.Z[b, :k]
    r = Fd[b] - _matvec_one(op, U, b)
    beta = float(torch.linalg.vector_norm(r).item())
    s.rel = beta / s.fnorm
    s.converged = s.rel <= cfg.tol
    if not s.converged and s.rel >= s.cycle_start_rel:
        s.stagnated = True
    s.outer += 1
    s.done = s.converged or s.stagnated or s.outer >= cfg.max_outer
    if not s.done:
        s.start_cycle(r, beta)


def _matvec(op, X):
    return op.matvec(X.reshape(op.batch, op.P)).reshape(op.batch, op.P)


def _matvec_one(op, U, b):
    return _matvec(op, U)[b]


def fgmres(A, f, precond_apply=None, cfg: FgmresConfig = None, u0=None):
    """GPU drop-in for fgmres.fgmres (single system, zero or given start)."""
    cfg = cfg or FgmresConfig()
    op = A if isinstance(A, GpuStencilOperator) else _op_for(A, f)
    if op.batch != 1:
        raise ValueError("use fgmres_batched for a batched operator")
    (u, rep), = fgmres_batched(op, f, precond_apply, cfg, U0=u0)
    return u.reshape(-1), rep

"""GPU FGMRES driver (fgmres.py:18-131) for the multilevel solves.

    fgmres(A, f, precond_apply=None, cfg=None, u0=None) -> (u, SolveReport)
    fgmres_batched(A, F, precond_apply=None, cfg=None)   -> [(u, SolveReport)]

The driver stays host Python as in the reference (FGMRES is
not on the hot path); vectors, the operator, modified Gram-Schmidt, the
Arnoldi normalisation and the solution update are device kernels, and the
preconditioner (e.g. the device V-cycle) runs on the device.  The small
Hessenberg / Givens recurrences run on the host exactly as fgmres.py:81-97
writes them (NumPy scalars: the reference's rounding), but OFF the critical
path: the device runs one Arnoldi step ahead.

  step k   device: z = M^-1 v_k ; w = A z ; MGS (rg_mgs_arnoldi) ; v_{k+1} =
           w / ||w|| and the packed Hessenberg column (rg_arnoldi_tail) ; an
           async copy of that column into pinned host memory + an event
  host     enqueues step k+1 (it needs only v_{k+1}, already on the device),
           THEN waits for step k's column and applies the Givens rotations

So the only host waits are for data the device produced a whole Arnoldi step
earlier; the device idles only at restarts (the y solve and the update need
the cycle's last column).  A step enqueued past a stop (convergence, happy
breakdown) is discarded, as the reference never computes it.

The batched form runs B independent FGMRES state machines; each system keeps
its own restart position and stops on its own.  Systems at the same Arnoldi
index share the batched MGS launches.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .errors import DivergenceError, SolveReport
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
    """Per-system FGMRES state (the locals of fgmres.py:31-131)."""

    def __init__(self, b, mr, npdt):
        self.b, self.mr, self.npdt = b, mr, npdt
        self.trace = []
        self.total = 0
        self.outer = 0
        self.converged = False
        self.stagnated = False
        self.done = False
        self.epoch = 0          # restart cycle id (tags in-flight steps)
        self.k = 0              # Arnoldi steps processed on the host in this cycle
        self.k_enq = 0          # Arnoldi steps enqueued on the device in this cycle
        self.end_cycle = False

    def start_cycle(self, beta):
        mr, dt = self.mr, self.npdt
        self.cycle_start_rel = self.rel
        self.H = np.zeros((mr + 1, mr), dtype=dt)
        self.cs = np.zeros(mr, dtype=dt)
        self.sn = np.zeros(mr, dtype=dt)
        self.g = np.zeros(mr + 1, dtype=dt)
        self.g[0] = beta
        self.k = 0
        self.k_enq = 0
        self.epoch += 1
        self.end_cycle = False


class _Step:
    """One enqueued Arnoldi step of a group of systems at index k."""

    def __init__(self, systems, k, hcol_host, event):
        self.entries = [(s, s.epoch) for s in systems]
        self.k = k
        self.hcol = hcol_host          # pinned [G, k+2]
        self.event = event


def _hierarchy_nocheck(precond):
    """A GpuHierarchy.apply bound method -> the same call without its
    host-synchronising finite test (the driver tests lazily)."""
    owner = getattr(precond, "__self__", None)
    if owner is not None and getattr(precond, "__name__", "") == "apply" and \
            type(owner).__name__ == "GpuHierarchy":
        return lambda R: owner.apply(R, check=False, clone=False), True
    return precond, False


def fgmres_batched(A, F, precond_apply=None, cfg: FgmresConfig = None, U0=None):
    """B independent FGMRES solves sharing batched operator / preconditioner
    calls, each system orthogonalised in the reference's order
    (fgmres.py:76-78)."""
    cfg = cfg or FgmresConfig()
    op = A if isinstance(A, GpuStencilOperator) else _op_for(A, F)
    host = _is_host(F)
    t0 = time.perf_counter()
    B, n = op.batch, op.P
    Fd = op.to_device(F)
    npdt = op.np_dtype
    code = L.RG_C128 if op.torch_dtype == torch.complex128 else L.RG_F64
    mr = cfg.restart
    precond = precond_apply if precond_apply is not None else (lambda r: r)
    precond, lazy_check = _hierarchy_nocheck(precond)
    dev = op.device
    U = torch.zeros_like(Fd) if U0 is None else op.to_device(U0).clone()
    V = torch.zeros((B, mr + 1, n), dtype=op.torch_dtype, device=dev)
    Z = torch.zeros((B, mr, n), dtype=op.torch_dtype, device=dev)
    lib, stream = op._lib, torch.cuda.current_stream()
    fn = torch.linalg.vector_norm(Fd, dim=1).cpu().numpy()
    systems = [_Sys(b, mr, npdt) for b in range(B)]
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
            V[b, 0] = Rr[b] / float(beta[b])
            s.start_cycle(float(beta[b]))

    def enqueue(run):
        """Device work of one Arnoldi step for the systems in `run` (each at
        its own s.k_enq); returns the in-flight _Step records."""
        ks = [s.k_enq for s in run]
        lock = len(run) == B and len(set(ks)) == 1
        if lock:
            Vk = V[:, ks[0]]
        else:
            Vk = torch.zeros((B, n), dtype=op.torch_dtype, device=dev)
            for s in run:
                Vk[s.b] = V[s.b, s.k_enq]
        Zk = precond(Vk)
        Zk = (Zk if isinstance(Zk, torch.Tensor) else torch.as_tensor(np.asarray(Zk))).to(
            dev, op.torch_dtype).reshape(B, n)
        W = _matvec(op, Zk)
        steps = []
        groups = {}
        for s in run:
            groups.setdefault(s.k_enq, []).append(s)
        for k, grp in groups.items():
            G = len(grp)
            if G == B:
                Z[:, k] = Zk
                w, Vg = W.contiguous(), V
            else:
                idx = [s.b for s in grp]
                for s in grp:
                    Z[s.b, k] = Zk[s.b]
                w = torch.stack([W[i] for i in idx])
                Vg = torch.stack([V[i] for i in idx])
            hbuf = torch.empty((k + 1, G), dtype=op.torch_dtype, device=dev)
            n2 = torch.empty(G, dtype=torch.float64, device=dev)
            hcol = torch.empty((G, k + 2), dtype=op.torch_dtype, device=dev)
            ld = (mr + 1) * n
            # modified Gram-Schmidt (:76-78), one fused pass per index
            L.check(lib.rg_mgs_arnoldi(code, G, n, L.ptr(w), n, L.ptr(Vg), ld, k, L.ptr(hbuf),
                                       L.ptr(n2), L.stream_ptr()))
            vnext = Vg[:, k + 1] if k + 1 <= mr else None
            if vnext is None:
                vnext = torch.empty((G, n), dtype=op.torch_dtype, device=dev)
            L.check(lib.rg_arnoldi_tail(code, G, n, L.ptr(w), n, L.ptr(vnext), ld, L.ptr(hbuf), k,
                                        L.ptr(n2), L.ptr(hcol), L.stream_ptr()))
            if G != B:
                for q, s in enumerate(grp):
                    V[s.b, k + 1] = vnext[q]
            hh = torch.empty((G, k + 2), dtype=op.torch_dtype, pin_memory=True)
            hh.copy_(hcol, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            steps.append(_Step(grp, k, hh, ev))
            for s in grp:
                s.k_enq += 1
        return steps

    def process(step):
        """Host side of one step (fgmres.py:79-107) for every system whose
        cycle is the one the step was enqueued in."""
        step.event.synchronize()
        Hh = step.hcol.numpy()
        k = step.k
        for q, (s, epoch) in enumerate(step.entries):
            if s.done or s.epoch != epoch or s.k != k or s.end_cycle:
                continue           # speculative step past a stop / restart
            hc, hk1 = Hh[q, :k + 1], float(np.real(Hh[q, k + 1]))
            if lazy_check and not (np.all(np.isfinite(hc)) and np.isfinite(hk1)):
                if not bool(torch.isfinite(Z[s.b, k]).all()):
                    m = _smoother_steps(precond_apply)
                    raise DivergenceError("smoother produced a non-finite iterate",
                                          inner_iteration=m)
            H, cs, sn, g = s.H, s.cs, s.sn, s.g
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
                s.end_cycle = True
            elif s.k >= s.mr:
                s.end_cycle = True

    pending = []
    while True:
        run = [s for s in systems if not s.done and not s.end_cycle and s.k_enq < s.mr]
        nxt = enqueue(run) if run else []
        for st in pending:                      # the previous step, while the device runs nxt
            process(st)
        pending = nxt
        ending = [s for s in systems if not s.done and s.end_cycle]
        if ending:
            for st in pending:                  # steps of other systems stay valid
                process(st)
            pending = []
            for s in ending:
                _finish_cycle(op, Fd, U, V, Z, s, cfg, lib, code)
        if all(s.done for s in systems):
            break
        if not pending and not any(not s.done and not s.end_cycle and s.k_enq < s.mr
                                   for s in systems):
            break                               # (defensive: nothing left to run)
    torch.cuda.current_stream().synchronize()
    wall = time.perf_counter() - t0
    Uo = U.cpu().numpy() if host else U
    return [(Uo[b], SolveReport(iterations=s.total, inner_iterations=s.total,
                                converged=s.converged, final_relative_residual=s.rel,
                                wall_time=wall, trace=np.array(s.trace), stagnated=s.stagnated))
            for b, s in enumerate(systems)]


def _smoother_steps(precond):
    owner = getattr(precond, "__self__", None)
    try:
        return owner.levels[0].sched.m
    except AttributeError:
        return 0


def _finish_cycle(op, Fd, U, V, Z, s, cfg, lib, code):
    """Update, true residual, stagnation test (fgmres.py:108-126)."""
    k = s.k
    Hk = np.triu(s.H[:k, :k])
    if k == 0:
        y = np.zeros(0, dtype=s.npdt)
    else:
        try:
            y = np.linalg.solve(Hk, s.g[:k])
        except np.linalg.LinAlgError:
            y = np.linalg.lstsq(Hk, s.g[:k], rcond=None)[0]
    if k > 0:
        yt = torch.as_tensor(np.ascontiguousarray(y)).to(U.device, U.dtype)
        L.check(lib.rg_krylov_update(code, op.P, L.ptr(U[s.b]), L.ptr(Z[s.b]), op.P, L.ptr(yt), k,
                                     L.stream_ptr()))
    r = Fd[s.b] - _matvec(op, U)[s.b]
    beta = float(torch.linalg.vector_norm(r).item())
    s.rel = beta / s.fnorm
    s.converged = s.rel <= cfg.tol
    if not s.converged and s.rel >= s.cycle_start_rel:
        s.stagnated = True
    s.outer += 1
    s.done = s.converged or s.stagnated or s.outer >= cfg.max_outer
    s.end_cycle = False
    if not s.done:
        V[s.b].zero_()
        Z[s.b].zero_()
        V[s.b, 0] = r / beta
        s.start_cycle(beta)


def _matvec(op, X):
    return op.matvec(X.reshape(op.batch, op.P)).reshape(op.batch, op.P)


def fgmres(A, f, precond_apply=None, cfg: FgmresConfig = None, u0=None):
    """GPU drop-in for fgmres.fgmres (single system, zero or given start)."""
    cfg = cfg or FgmresConfig()
    op = A if isinstance(A, GpuStencilOperator) else _op_for(A, f)
    if op.batch != 1:
        raise ValueError("use fgmres_batched for a batched operator")
    (u, rep), = fgmres_batched(op, f, precond_apply, cfg, U0=u0)
    return u.reshape(-1), rep

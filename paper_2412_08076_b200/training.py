"""GPU training unroll: the K-step unrolled
relative residual of training.py:61-104 and its reverse-mode gradient with
respect to the weight schedule (what tape.py:28-42 computes through the
recorded unroll, training.py:84-104 + tape.py:191-199).

    unrolled_relative_residual(A, f, omega, alpha, alpha_t, K, variant, P=None)
        -> float                                      (training.py:61-81)
    unrolled_residual_grad(A, f, omega, alpha, alpha_t, K, variant, P=None)
        -> (loss, d_omega, d_alpha, d_alpha_t)        (tape gradients of _unroll_tape)
    UnrollEngine(op, K, variant, P=None)              batched forward / backward
    UnrolledResidual.apply(engine, F, omega, alpha, alpha_t)
        -> loss[B]    torch.autograd.Function, so a torch weight network
                      (the reference MetaNet, metanet.py:86-126) trains on it

Forward: K calls of the fused inner-update kernel (rg_inner_update) that
keep every iterate (u_k, v_k histories, [K+1, B, P] float64 in HBM), then
the loss.  Backward: rg_unroll_adjoint_init / _step (csrc/adjoint.cuh), two
stencil kernels per step with the three schedule inner products reduced on
the device; only K x 3 x B scalars come back to the host.  d_alpha_t is
reported separately; for "nag" the reference ties alpha_t to alpha (one
Var), so its alpha gradient is d_alpha + d_alpha_t.

Iterates are bitwise those of the reference's forward (same kernels as
solve_stationary); the loss and gradients agree to ~1e-12 relative (the
reductions are fixed-order tree sums, not NumPy's).  float64, CONST9/VAR9
operators, P = None, weighted Jacobi, or GS / SOR / SSOR (TrainConfig.precond
"gs" / "ssor", training.py:47-58): the forward keeps p_k = B^{-1} r_k and the
reverse pass applies B^{-T} with the transposed wavefront solves.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L
from .errors import UnsupportedOperator
from .operator import GpuStencilOperator, as_operator, precond_scale
from .schedules import WeightSchedule


def _schedules(variant, omega, alpha, alpha_t, B):
    """One WeightSchedule per system ([B, m] or [m] arrays); nag runs as
    nagex with alpha_t given, so the two coefficient arrays stay separate."""
    om = np.atleast_2d(np.asarray(omega, dtype=float))
    m = om.shape[1]
    if om.shape[0] == 1:
        om = np.repeat(om, B, axis=0)

    def arr(x):
        if x is None:
            return np.zeros((B, m))
        x = np.atleast_2d(np.asarray(x, dtype=float))
        return np.repeat(x, B, axis=0) if x.shape[0] == 1 else x
    al, at = arr(alpha), arr(alpha_t)
    if variant == "plain":
        return [WeightSchedule(omega=om[b]) for b in range(B)]
    if variant == "mom":
        return [WeightSchedule(omega=om[b], alpha=al[b], variant="mom") for b in range(B)]
    if variant in ("nag", "nagex"):
        return [WeightSchedule(omega=om[b], alpha=al[b], alpha_tilde=at[b], variant="nagex")
                for b in range(B)]
    raise ValueError(f"unknown variant {variant!r}")


class UnrollEngine:
    """K-step unroll of a batch of systems (one operator batch) with the
    histories kept on the device for the reverse pass."""

    def __init__(self, op: GpuStencilOperator, K: int, variant: str, P=None):
        if op.np_dtype != np.float64 or op.kind not in (L.RG_CONST9, L.RG_VAR9):
            raise UnsupportedOperator("the training unroll runs on float64 CONST9/VAR9 operators")
        if K < 0:
            raise ValueError("unroll must be >= 0")
        from .precond import TriangularPreconditioner, tri_spec
        self.tri = None
        spec = tri_spec(P)
        if spec is not None:          # GS / SOR / SSOR (TrainConfig.precond "gs" / "ssor")
            self.tri = TriangularPreconditioner(op, *spec)
            P = None
        elif P is not None and getattr(P, "kind", None) not in ("weighted-jacobi", "identity") \
                and not hasattr(P, "scale"):
            raise UnsupportedOperator(
                f"preconditioner {getattr(P, 'kind', None)!r} has no GPU unroll path")
        self.op, self.K, self.variant, self.P = op, int(K), variant, P
        self.opT = op.transpose()
        B, n = op.batch, op.P
        dev = op.device
        self.U = torch.zeros((self.K + 1, B, n), dtype=torch.float64, device=dev)
        self.V = torch.zeros_like(self.U)
        self.f = torch.empty((B, n), dtype=torch.float64, device=dev)
        self.ubar = torch.empty_like(self.f)
        self.vbar = torch.empty_like(self.f)
        self.rbar = torch.empty_like(self.f)
        self.loss = torch.empty(B, dtype=torch.float64, device=dev)
        self.dots = torch.empty((max(self.K, 1), 3, B), dtype=torch.float64, device=dev)
        self.ds = None
        # every forward overwrites the histories and the adjoint seeds, so a
        # backward is only valid for the most recent forward: callers that
        # keep a generation (UnrolledResidual) are checked against it
        self.generation = 0
        if self.tri is not None:      # p_k = B^{-1} r_k history and scratch
            self.Pk = torch.empty((max(self.K, 1), B, n), dtype=torch.float64, device=dev)
            self.r = torch.empty_like(self.f)
            self.y = torch.empty_like(self.f)
            self.work = torch.empty_like(self.f)
            self.rpre = torch.empty_like(self.f)

    def forward(self, F, omega, alpha=None, alpha_t=None):
        """Loss per system (device tensor [B]) of the K-step unroll from 0."""
        from .richardson import DeviceSchedule
        op, B = self.op, self.op.batch
        sl = _schedules(self.variant, omega, alpha, alpha_t, B)
        if self.ds is None or self.ds.matches(sl, self.P) is None:
            self.ds = DeviceSchedule(op, sl, self.P)
        else:
            self.ds.load(sl, self.ds._scales(self.P))
        self.f.copy_(op.to_device(F).reshape(B, op.P))
        lib, s = op._lib, L.stream_ptr()
        sched = C.byref(self.ds.struct)
        m = self.ds.m
        nag = self.variant in ("nag", "nagex")
        for k in range(self.K):
            if self.tri is None:
                L.check(lib.rg_inner_update(op.handle, sched, k % m, L.ptr(self.U[k]),
                                            L.ptr(self.V[k]), L.ptr(self.U[k + 1]),
                                            L.ptr(self.V[k + 1]), L.ptr(self.f), None, 0, s))
                continue
            # r_k at u_k (or the look-ahead), p_k = B^{-1} r_k kept, then the update
            x = self.U[k]
            if nag:
                L.check(lib.rg_precond_update(op.handle, sched, k % m, None, L.ptr(self.U[k]),
                                              L.ptr(self.V[k]), L.ptr(self.y), s))
                x = self.y
            L.check(lib.rg_residual(op.handle, L.ptr(x), L.ptr(self.f), L.ptr(self.r), None, s))
            self.tri.apply_device(self.r, self.Pk[k], self.work)
            self.U[k + 1].copy_(self.U[k])
            self.V[k + 1].copy_(self.V[k])
            L.check(lib.rg_precond_update(op.handle, sched, k % m, L.ptr(self.Pk[k]),
                                          L.ptr(self.U[k + 1]), L.ptr(self.V[k + 1]), None, s))
        self._adjoint_init()
        self.generation += 1
        return self.loss

    def _adjoint_init(self):
        """Loss and the adjoint seeds (rbar, ubar, vbar) from u_K."""
        op = self.op
        L.check(op._lib.rg_unroll_adjoint_init(op.handle, self.opT.handle, L.ptr(self.U[self.K]),
                                               L.ptr(self.f), L.ptr(self.rbar), L.ptr(self.ubar),
                                               L.ptr(self.vbar), L.ptr(self.loss),
                                               L.stream_ptr()))

    def backward(self, generation=None):
        """(d_omega, d_alpha, d_alpha_t) as host arrays [B, m] for the last
        forward (each system's own loss).  The reverse pass consumes the
        adjoint seeds in place, so they are re-seeded from the stored u_K
        first: repeated backward calls for one forward give the same
        gradients.  `generation` (the value of self.generation right after
        the forward in question) makes a stale backward raise instead of
        silently differentiating a later forward."""
        if self.ds is None:
            raise RuntimeError("backward() before any forward()")
        if generation is not None and generation != self.generation:
            raise RuntimeError(
                f"the unroll engine ran forward again (generation {self.generation}) after the "
                f"forward being differentiated (generation {generation}); its histories are "
                "overwritten -- use one engine per pending backward")
        op, m = self.op, self.ds.m
        lib, s = op._lib, L.stream_ptr()
        sched = C.byref(self.ds.struct)
        self._adjoint_init()
        tkind = None
        if self.tri is not None:
            tkind = L.RG_TRI_SSOR_T if self.tri.mode == L.RG_TRI_SSOR else L.RG_TRI_SOR_T
        for k in range(self.K - 1, -1, -1):
            if self.tri is None:
                L.check(lib.rg_unroll_adjoint_step(op.handle, self.opT.handle, sched, k % m,
                                                   L.ptr(self.f), L.ptr(self.U[k]),
                                                   L.ptr(self.V[k]), L.ptr(self.ubar),
                                                   L.ptr(self.vbar), L.ptr(self.rbar),
                                                   L.ptr(self.dots[k]), s))
                continue
            # p_k from the history; rbar = B^{-T} (w vt) (precond.py:94,112-113)
            L.check(lib.rg_unroll_adjoint_step_ext(op.handle, self.opT.handle, sched, k % m,
                                                   L.ptr(self.V[k]), L.ptr(self.Pk[k]),
                                                   L.ptr(self.ubar), L.ptr(self.vbar),
                                                   L.ptr(self.rpre), None, L.ptr(self.dots[k]),
                                                   1, s))
            L.check(lib.rg_tri_apply(op.handle, tkind, self.tri._relax, L.ptr(self.rpre),
                                     L.ptr(self.rbar), L.ptr(self.work), s))
            L.check(lib.rg_unroll_adjoint_step_ext(op.handle, self.opT.handle, sched, k % m,
                                                   L.ptr(self.V[k]), None, L.ptr(self.ubar),
                                                   L.ptr(self.vbar), None, L.ptr(self.rbar),
                                                   L.ptr(self.dots[k]), 2, s))
        D = self.dots[:self.K].cpu().numpy()         # [K, 3, B]
        B = op.batch
        da, dw, dat = (np.zeros((B, m)) for _ in range(3))
        for k in range(self.K - 1, -1, -1):          # the tape's accumulation order
            i = k % m
            da[:, i] += D[k, 0]
            dw[:, i] += D[k, 1]
            dat[:, i] += D[k, 2]
        if self.variant == "plain":
            da[:] = 0.0
        if self.variant in ("plain", "mom"):
            dat[:] = 0.0
        return dw, da, dat


def _engine_for(A, f, K, variant, P):
    from .precond import tri_spec
    op = A if isinstance(A, GpuStencilOperator) else as_operator(A)
    if P is not None and tri_spec(P) is None:
        precond_scale(P, op.P)   # validates the kind (Jacobi / identity)
    return UnrollEngine(op, K, variant, P)


def unrolled_relative_residual(A, f, omega, alpha, alpha_t, K, variant, P=None):
    """training.py:61-81 on the device: ||f - A u_K|| / ||f||."""
    eng = _engine_for(A, f, K, variant, P)
    return float(eng.forward(f, omega, alpha, alpha_t)[0].item())


def unrolled_residual_grad(A, f, omega, alpha, alpha_t, K, variant, P=None):
    """Loss and its gradients w.r.t. omega, alpha, alpha_t (length-m arrays)
    for one system: what Tape.backward gives for _unroll_tape."""
    eng = _engine_for(A, f, K, variant, P)
    loss = float(eng.forward(f, omega, alpha, alpha_t)[0].item())
    dw, da, dat = eng.backward()
    return loss, dw[0], da[0], dat[0]


class UnrolledResidual(torch.autograd.Function):
    """loss[B] = unroll(F; omega, alpha, alpha_t) with a hand-written device
    adjoint; omega/alpha/alpha_t are [B, m] float64 tensors (any device)."""

    @staticmethod
    def forward(ctx, engine, F, omega, alpha, alpha_t):
        to_np = lambda t: None if t is None else t.detach().cpu().numpy()  # noqa: E731
        loss = engine.forward(F, to_np(omega), to_np(alpha), to_np(alpha_t)).clone()
        ctx.engine = engine
        ctx.generation = engine.generation
        ctx.devs = (omega.device, None if alpha is None else alpha.device,
                    None if alpha_t is None else alpha_t.device)
        return loss.to(omega.device)

    @staticmethod
    def backward(ctx, g):
        dw, da, dat = ctx.engine.backward(ctx.generation)
        gh = g.detach().cpu().numpy()[:, None]
        out = [torch.as_tensor(gh * x, dtype=torch.float64) for x in (dw, da, dat)]
        res = [out[0].to(ctx.devs[0])]
        res.append(None if ctx.devs[1] is None else out[1].to(ctx.devs[1]))
        res.append(None if ctx.devs[2] is None else out[2].to(ctx.devs[2]))
        return (None, None, *res)

"""Training unroll on the device (training.py:61-104, SURVEY.md §8(f)
item 3): the K-step loss and its reverse-mode schedule gradients vs the
reference's tape (tests/golden/unroll.npz) and the oracle's adjoint.  The
forward iterates are the solve kernels' (bitwise); the loss and gradients
go through fixed-order device reductions, so the bar is 1e-12 relative for
the loss and 1e-10 for the gradients."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2412_08076_b200 as G
from paper_2412_08076_b200 import training as T

pytestmark = pytest.mark.gpu


def _close(got, want, rtol=1e-10):
    got, want = np.asarray(got), np.asarray(want)
    scale = max(np.max(np.abs(want)), 1e-300)
    assert np.all(np.abs(got - want) <= rtol * scale), (got, want)


def test_unroll_matches_reference_tape(golden):
    d = golden("unroll")
    for k in range(int(d["count"])):
        g = lambda key: d[f"u{k}_{key}"]  # noqa: E731
        A = O.assemble_anisotropic(float(g("eps")), float(g("theta")), int(g("n")))
        pre = str(g("pre"))
        P = {"jacobi": lambda: G.JacobiScale.weighted_jacobi(A),
             "ssor": lambda: G.Preconditioner.ssor(A, 1.0),
             "gs": lambda: G.Preconditioner.gauss_seidel(A)}.get(pre, lambda: None)()
        variant = str(g("variant"))
        al = g("alpha") if variant != "plain" else None
        loss, dw, da, dat = T.unrolled_residual_grad(A, g("f"), g("omega"), al, g("alpha_t"),
                                                     int(g("K")), variant, P)
        assert abs(loss - float(g("loss"))) <= 1e-12 * float(g("loss"))
        _close(dw, g("d_omega"))
        _close(da, g("d_alpha"))
        _close(dat, g("d_alpha_t"))
        free = T.unrolled_relative_residual(A, g("f"), g("omega"), al, g("alpha_t"),
                                            int(g("K")), variant, P)
        assert abs(free - float(g("loss_free"))) <= 1e-12 * free


def test_batched_engine_and_autograd():
    rng = np.random.default_rng(5)
    B, n, m, K = 3, 40, 4, 20
    As = [O.assemble_anisotropic(10 ** rng.uniform(-2, 0), rng.uniform(0, np.pi), n)
          for _ in range(B)]
    op = G.GpuStencilOperator.stack([G.GpuStencilOperator.from_sparse(A) for A in As])
    F = rng.standard_normal((B, op.P))
    W = rng.uniform(0.05, 0.15, (B, m))
    Al = rng.uniform(0.1, 0.4, (B, m))
    At = rng.uniform(0.1, 0.4, (B, m))
    eng = T.UnrollEngine(op, K, "nagex")
    om = torch.tensor(W, requires_grad=True)
    al = torch.tensor(Al, requires_grad=True)
    at = torch.tensor(At, requires_grad=True)
    loss = T.UnrolledResidual.apply(eng, F, om, al, at)
    weights = torch.tensor([1.0, 2.0, 0.5], dtype=torch.float64)
    (loss * weights).sum().backward()
    for b in range(B):
        lo, dw, da, dat = O.unroll_grad(As[b], F[b], W[b], Al[b], At[b], K, "nagex")
        assert abs(float(loss[b].detach()) - lo) <= 1e-12 * lo
        _close(om.grad[b].numpy(), weights[b].item() * dw)
        _close(al.grad[b].numpy(), weights[b].item() * da)
        _close(at.grad[b].numpy(), weights[b].item() * dat)


def test_full_size_unroll_vs_oracle():
    """One 1023^2 system, K = 50 (the TrainConfig default unroll)."""
    rng = np.random.default_rng(6)
    A = O.assemble_anisotropic(1e-2, 0.4, 1024)
    f = rng.standard_normal(A.shape[0])
    w = np.array([0.1, 0.15, 0.12])
    a = np.array([0.3, 0.2, 0.25])
    sc = O.jacobi_scale(A)
    loss, dw, da, dat = T.unrolled_residual_grad(A, f, w * 4, a, a, 50, "nag",
                                                 G.JacobiScale(sc))
    lo, dwo, dao, dato = O.unroll_grad(A, f, w * 4, a, a, 50, "nag", sc)
    assert abs(loss - lo) <= 1e-12 * lo
    _close(dw, dwo)
    _close(da, dao)
    _close(dat, dato)


def test_var9_operator_unroll():
    """A variable-coefficient, non-symmetric 9-point operator (VAR9; the
    adjoint runs on its transpose)."""
    import scipy.sparse as sp
    rng = np.random.default_rng(8)
    A = O.assemble_anisotropic(0.05, 1.0, 16)
    Ac = (sp.diags(rng.uniform(0.5, 1.5, A.shape[0])) @ A).tocsr()
    op = G.GpuStencilOperator.from_sparse(Ac)
    assert op.kind == 3
    f = rng.standard_normal(Ac.shape[0])
    lam = np.abs(np.linalg.eigvals(Ac.toarray())).max()
    w = np.array([0.5, 0.8]) / lam
    a = np.array([0.3, 0.4])
    loss, dw, da, dat = T.unrolled_residual_grad(op, f, w, a, None, 15, "mom")
    lo, dwo, dao, dato = O.unroll_grad(Ac, f, w, a, np.zeros(2), 15, "mom")
    assert abs(loss - lo) <= 1e-12 * lo
    _close(dw, dwo)
    _close(da, dao)

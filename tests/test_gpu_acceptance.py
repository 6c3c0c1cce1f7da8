"""The reference's acceptance criteria that exercise the hot path
(test_acceptance.py:145-338), run on the device path: reduction chains
(criterion 4), the unroll gradient against central differences (5), the
exact spectral correction (6), V-cycle residual non-increase (7) and the
V-cycle-preconditioned FGMRES on Helmholtz (8)."""
import sys

import numpy as np
import pytest

import oracle as O
import paper_2412_08076_b200 as G
import paper_2412_08076_b200.fgmres  # noqa: E402,F401  (the package attribute is the function)
GG = sys.modules["paper_2412_08076_b200.fgmres"]
from paper_2412_08076_b200 import fns as GF
from paper_2412_08076_b200 import multigrid as GM
from paper_2412_08076_b200 import training as T

pytestmark = pytest.mark.gpu


def test_criterion_4_reduction_chain():
    """nag == nagex with alpha_tilde = alpha; plain == mom with alpha = 0
    (test_acceptance.py:162-177: <= 1e-14; here bitwise)."""
    A = O.assemble_anisotropic(0.1, 0.4, 16)
    f = np.random.default_rng(1).standard_normal(A.shape[0])
    w = np.array([0.1, 0.2, 0.15])
    a = np.array([0.3, 0.2, 0.1])
    u1, _ = G.solve_stationary(A, f, G.WeightSchedule(omega=w, alpha=a, variant="nag"),
                               tol=1e-10, max_outer=50)
    u2, _ = G.solve_stationary(A, f, G.WeightSchedule(omega=w, alpha=a, alpha_tilde=a,
                                                      variant="nagex"), tol=1e-10, max_outer=50)
    assert np.array_equal(u1, u2)
    u3, _ = G.solve_stationary(A, f, G.WeightSchedule(omega=w), tol=1e-10, max_outer=50)
    u4, _ = G.solve_stationary(A, f, G.WeightSchedule(omega=w, alpha=np.zeros(3), variant="mom"),
                               tol=1e-10, max_outer=50)
    assert np.array_equal(u3, u4)


def test_criterion_5_unroll_gradient_vs_central_differences():
    """Device adjoint of the K = 5 unroll against central differences of the
    device loss, relative to the gradient scale (test_acceptance.py:209-249)."""
    A = O.assemble_anisotropic(0.3, 0.8, 8)
    f = np.random.default_rng(11).standard_normal(A.shape[0])
    w = np.array([0.12, 0.2, 0.16])
    a = np.array([0.3, 0.5, 0.2])
    at = np.array([0.4, 0.1, 0.6])
    K = 5
    loss, dw, da, dat = T.unrolled_residual_grad(A, f, w, a, at, K, "nagex")
    g = np.concatenate([dw, da, dat])
    x = np.concatenate([w, a, at])

    def loss_at(v):
        return T.unrolled_relative_residual(A, f, v[:3], v[3:6], v[6:], K, "nagex")
    h = 1e-6
    scale = np.abs(g).max()
    worst = 0.0
    for i in range(9):
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        fd = (loss_at(xp) - loss_at(xm)) / (2 * h)
        worst = max(worst, abs(fd - g[i]) / scale)
    assert worst <= 1e-5, worst


def test_criterion_6_spectral_correction_exactness():
    """lambda_tilde = 1 / (sine-basis eigenvalues) solves in one correction
    (test_acceptance.py:252-263)."""
    n = 32
    A = O.assemble_anisotropic(1.0, 0.0, n)
    s = n - 1
    ii = (s // 2) * s + s // 2
    row = A[ii].toarray().ravel()
    st = {(dx, dy): row[ii + dx * s + dy] for dx in (-1, 0, 1) for dy in (-1, 0, 1)}
    # the stencil is even in each axis, so sine modes are eigenvectors
    k = np.arange(1, n)
    lam = sum(v * np.outer(np.cos(np.pi * k * dx / n), np.cos(np.pi * k * dy / n))
              for (dx, dy), v in st.items())
    corr = GF.SpectralCorrection(1.0 / lam.ravel(), n)
    f = np.random.default_rng(3).standard_normal(A.shape[0])
    u = GF.fns_lite_step(A, f, np.zeros(A.shape[0]), G.WeightSchedule(omega=np.array([0.1])), 0,
                         corr)
    rel = np.linalg.norm(f - A @ u) / np.linalg.norm(f)
    assert rel <= 1e-12, rel


def test_criterion_7_vcycle_residual_non_increase():
    """Chebyshev(2) smoothing, n = 32: every V-cycle from zero reduces the
    residual (test_acceptance.py:266-291)."""
    n = 32
    A = O.assemble_anisotropic(1.0, 0.0, n)
    ev = np.linalg.eigvalsh(A.toarray())
    sched = G.WeightSchedule(omega=G.chebyshev_weights(ev[-1], ev[0], 2))
    h = GM.build_hierarchy(A, n, coarsest=8, schedules=sched)
    rng = np.random.default_rng(5)
    for _ in range(20):
        f = rng.standard_normal(A.shape[0])
        u = GM.v_cycle(h, f)
        assert np.linalg.norm(f - A @ u) <= np.linalg.norm(f)


def test_criterion_8_helmholtz_vcycle_fgmres():
    """V-cycle-preconditioned FGMRES on the damped Helmholtz problem converges
    in fewer iterations than unpreconditioned FGMRES (test_acceptance.py:318-331)."""
    n = 64
    H = O.assemble_helmholtz(10 * np.pi, n)
    rng = np.random.default_rng(13)
    fh = rng.standard_normal(H.shape[0]) + 1j * rng.standard_normal(H.shape[0])
    cfg = GG.FgmresConfig(restart=20, tol=1e-6, max_outer=200)
    op = G.GpuStencilOperator.from_sparse(H)
    _, ident = GG.fgmres(op, fh, cfg=cfg)
    sched = G.WeightSchedule(omega=np.full(5, 0.8 / (8.0 * n ** 2)), alpha=np.full(5, 0.3),
                             variant="nag")
    hier = GM.build_hierarchy(H, n, coarsest=16, schedules=sched)
    u, pre = GG.fgmres(op, fh, precond_apply=lambda r: hier.apply(r), cfg=cfg)
    assert pre.converged and ident.iterations > pre.iterations
    assert np.linalg.norm(fh - H @ u) / np.linalg.norm(fh) <= 1e-5

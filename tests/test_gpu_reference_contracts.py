"""The reference's own behavioural tests for the hot path, restated on the
device path (grid-shaped operators: the drop-in takes structured-grid
matrices).  Sources: test_fns.py:18-90, test_multigrid.py:30-83,
test_fgmres.py:39-135, test_richardson.py:32-200 (selected contracts)."""
import sys

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
import paper_2412_08076_b200 as G
import paper_2412_08076_b200.fgmres  # noqa: F401  (the package attribute is the function)
from paper_2412_08076_b200 import fns as GF
from paper_2412_08076_b200 import multigrid as GM

GG = sys.modules["paper_2412_08076_b200.fgmres"]
pytestmark = pytest.mark.gpu


def _sine_mode(n, p, q):
    i = np.arange(1, n)
    return np.outer(np.sin(p * np.pi * i / n), np.sin(q * np.pi * i / n)).reshape(-1)


# ---------------------------------------------------------------- fns.py
def test_fns_zero_correction_equals_pure_smoothing():
    """test_fns.py:18-28."""
    rng = np.random.default_rng(0)
    n = 8
    A = O.assemble_anisotropic(1.0, 0.0, n)
    f = rng.standard_normal((n - 1) ** 2)
    sched = G.WeightSchedule(omega=np.array([0.1, 0.2]))
    corr = GF.SpectralCorrection(np.zeros((n - 1) ** 2), n)
    u = GF.fns_lite_step(A, f, np.zeros((n - 1) ** 2), sched, 4, corr)
    v = np.zeros((n - 1) ** 2)
    for k in range(4):
        v = v + sched.omega[k % 2] * (f - A.dot(v))
    assert np.allclose(u, v, atol=1e-15)


def test_fns_step_is_affine_in_inputs():
    """test_fns.py:43-59."""
    rng = np.random.default_rng(1)
    n = 8
    A = O.assemble_anisotropic(0.3, 0.7, n)
    size = (n - 1) ** 2
    sched = G.WeightSchedule(omega=np.array([0.1, 0.15]))
    corr = GF.SpectralCorrection(rng.standard_normal(size) * 0.1, n)
    u1, f1 = rng.standard_normal(size), rng.standard_normal(size)
    u2, f2 = rng.standard_normal(size), rng.standard_normal(size)
    a, b = 0.3, 0.7

    def step(u, f):
        return GF.fns_lite_step(A, f, u, sched, 3, corr)

    lhs = step(a * u1 + b * u2, a * f1 + b * f2)
    rhs = a * step(u1, f1) + b * step(u2, f2)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * max(1.0, np.max(np.abs(rhs)))


def test_fns_correction_mode_locality():
    """test_fns.py:62-78: a symbol supported on one sine mode annihilates a
    residual orthogonal to that mode."""
    n = 8
    size = (n - 1) ** 2
    for k in range(0, size, 5):
        lam = np.zeros(size)
        lam[k] = 1.0
        corr = GF.SpectralCorrection(lam, n)
        p, q = divmod(k, n - 1)
        mode = _sine_mode(n, p + 1, q + 1)
        other = _sine_mode(n, (p + 1) % (n - 1) + 1, q + 1)
        if abs(other @ mode) > 1e-12:
            continue
        assert np.max(np.abs(corr.apply(other))) <= 1e-12


def test_fns_solve_counts_inner_iterations():
    """test_fns.py:81-89 (exact inverse symbol: converges, M inner steps per
    alternation)."""
    rng = np.random.default_rng(2)
    n = 16
    A = O.assemble_anisotropic(1.0, 0.0, n)
    i = np.arange(1, n)
    cp = np.cos(i * np.pi / n)
    lam = ((8.0 - 2.0 * cp[:, None] - 2.0 * cp[None, :] - 4.0 * cp[:, None] * cp[None, :]) / 3.0)
    corr = GF.SpectralCorrection(1.0 / lam.reshape(-1), n)
    f = rng.standard_normal((n - 1) ** 2)
    u, rep = GF.solve_fns(A, f, G.WeightSchedule(omega=np.array([0.1])), corr, 2, tol=1e-10)
    assert rep.converged and rep.inner_iterations == 2 * rep.iterations
    assert np.linalg.norm(f - A.dot(u)) <= 1e-10 * np.linalg.norm(f)


def test_sine_basis_eigenvalues_closed_form_and_device():
    """fns.py:60-73: the CONST9 closed form and the device transform path
    (on the VAR9 form of the same operator) equal the reference's
    one-vector-at-a-time definition; isotropic case = the closed-form
    eigenvalues of test_transforms.py:40-52."""
    n = 12
    A = O.assemble_anisotropic(0.3, 0.9, n)
    size = (n - 1) ** 2
    ref = np.array([O.dst2(A.dot(O.dst2(np.eye(size)[k])))[k] for k in range(size)])
    lam = G.sine_basis_eigenvalues(A, n)
    assert np.max(np.abs(lam - ref)) <= 1e-13 * np.max(np.abs(ref))
    var9 = G.GpuStencilOperator("var9", n - 1, G.GpuStencilOperator.from_sparse(A)._full_planes(),
                                None, np.float64)
    lam2 = G.sine_basis_eigenvalues(var9, n, chunk=50)
    assert np.max(np.abs(lam2 - ref)) <= 1e-13 * np.max(np.abs(ref))
    iso = G.sine_basis_eigenvalues(O.assemble_anisotropic(1.0, 0.0, n), n).reshape(n - 1, n - 1)
    cp = np.cos(np.pi * np.arange(1, n) / n)
    expect = (8.0 - 2.0 * cp[:, None] - 2.0 * cp[None, :] - 4.0 * cp[:, None] * cp[None, :]) / 3.0
    assert np.max(np.abs(iso - expect)) <= 1e-13 * np.max(expect)


# ---------------------------------------------------------- multigrid.py
def test_vcycle_zero_fixed_point():
    """test_multigrid.py:79-83."""
    n = 16
    H = O.assemble_helmholtz(2 * np.pi * n / 10, n)
    sch = G.WeightSchedule(omega=np.full(4, 0.8 / (8 * n * n)), alpha=np.full(4, 0.3),
                           variant="nag")
    h = GM.build_hierarchy(H, n, coarsest=4, schedules=sch)
    out = GM.v_cycle(h, np.zeros((n - 1) ** 2, dtype=complex))
    assert np.array_equal(out, np.zeros((n - 1) ** 2))


def test_odd_n_rejected():
    """test_multigrid.py:30-32 (restriction needs an even n)."""
    with pytest.raises(ValueError):
        G.restrict(np.zeros(6 * 6), 7)
    with pytest.raises(ValueError):
        GM.restriction_matrix(7)


def test_restrict_prolong_bitwise_vs_csr():
    """restrict / prolong (multigrid.py:52-59) on the device equal the CSR
    transfer matvecs bit for bit (real and complex, single and batched)."""
    rng = np.random.default_rng(8)
    n = 32
    R, P = O.restriction(n), O.prolongation(n)
    x = rng.standard_normal((n - 1) ** 2)
    assert np.array_equal(G.restrict(x, n), R.dot(x))
    xc = rng.standard_normal((n // 2 - 1) ** 2) + 1j * rng.standard_normal((n // 2 - 1) ** 2)
    assert np.array_equal(G.prolong(xc, n), P.dot(xc))
    X = rng.standard_normal((3, (n - 1) ** 2))
    Y = G.restrict(X, n)
    for b in range(3):
        assert np.array_equal(Y[b], R.dot(X[b]))


# -------------------------------------------------------------- fgmres.py
def _diag_grid(d):
    return sp.diags(np.asarray(d, dtype=float)).tocsr()


def test_fgmres_identity_converges_in_one_iteration():
    """test_fgmres.py:39-44 (4 x 4 grid)."""
    f = np.random.default_rng(3).standard_normal(16)
    u, rep = G.fgmres(sp.identity(16, format="csr"), f)
    assert rep.converged and rep.iterations == 1
    assert np.allclose(u, f, atol=1e-12)


def test_fgmres_three_distinct_eigenvalues_three_iterations():
    """test_fgmres.py:47-54 (diagonal 1, 2, 5 repeated on a 4 x 4 grid)."""
    d = np.array([1.0, 2.0, 5.0] * 5 + [1.0])
    f = np.random.default_rng(4).standard_normal(16)
    u, rep = G.fgmres(_diag_grid(d), f, cfg=G.FgmresConfig(restart=16, tol=1e-12))
    assert rep.converged and rep.iterations <= 3
    assert np.linalg.norm(u - f / d) <= 1e-10


def test_fgmres_stagnation_flagged():
    """test_fgmres.py:113-121 (singular projection on a 2 x 2 grid)."""
    f = np.array([0.0, 1.0, 0.0, 0.0])
    u, rep = G.fgmres(_diag_grid([1.0, 0.0, 0.0, 0.0]), f,
                      cfg=G.FgmresConfig(restart=4, tol=1e-10, max_outer=5))
    assert not rep.converged and rep.stagnated


def test_fgmres_zero_rhs():
    """test_fgmres.py:124-128."""
    u, rep = G.fgmres(sp.identity(9, format="csr"), np.zeros(9))
    assert rep.converged and rep.iterations == 0
    assert np.array_equal(u, np.zeros(9))


def test_fgmres_invalid_config():
    """test_fgmres.py:131-135."""
    with pytest.raises(ValueError):
        G.FgmresConfig(restart=0)
    with pytest.raises(ValueError):
        G.FgmresConfig(tol=0.0)


# ---------------------------------------------------------- richardson.py
def test_identity_converges_in_one_inner_step():
    """test_richardson.py:127-135: A = I, omega = 1 solves in one step."""
    f = np.random.default_rng(5).standard_normal(25)
    u, rep = G.solve_stationary(sp.identity(25, format="csr"), f,
                                G.WeightSchedule(omega=np.array([1.0])), tol=1e-12,
                                check="inner")
    assert rep.converged and rep.inner_iterations == 1
    assert np.array_equal(u, f)


def test_zero_momentum_degenerates_to_plain():
    """test_richardson.py:100-106: mom/nag with alpha = 0 give the plain
    iterates bitwise."""
    rng = np.random.default_rng(6)
    A = O.assemble_anisotropic(0.1, 0.4, 96)
    f = rng.standard_normal(A.shape[0])
    w = np.full(4, 0.3)
    u0, r0 = G.solve_stationary(A, f, G.WeightSchedule(omega=w), tol=1e-300, max_outer=3)
    for var in ("mom", "nag"):
        u1, r1 = G.solve_stationary(A, f, G.WeightSchedule(omega=w, alpha=np.zeros(4), variant=var),
                                    tol=1e-300, max_outer=3)
        assert r1.inner_iterations == r0.inner_iterations
        assert np.array_equal(u1, u0), var


def test_scale_invariance_of_counts():
    """test_richardson.py:179-189: scaling f scales u and keeps the counts."""
    rng = np.random.default_rng(7)
    A = O.assemble_anisotropic(0.5, 0.2, 32)
    f = rng.standard_normal(A.shape[0])
    lam = np.linalg.eigvalsh(A.toarray())
    s = G.WeightSchedule(omega=G.chebyshev_weights(lam[-1], lam[0], 8))
    u1, r1 = G.solve_stationary(A, f, s, tol=1e-8)
    u2, r2 = G.solve_stationary(A, 4.0 * f, s, tol=1e-8)
    assert r1.iterations == r2.iterations and r1.inner_iterations == r2.inner_iterations
    assert np.array_equal(4.0 * u1, u2)   # power-of-two scaling is exact in f64

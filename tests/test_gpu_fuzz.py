"""Seeded randomized parity sweep of the device path against the oracle:
solve_stationary over grid sizes on both sides of every kernel switch
(cluster solver <= 4096 unknowns, blocked sweep above), variants, Jacobi,
check modes and schedule lengths; the DST at random sizes (FFT and dense
paths); FNS steps.  Same bars as the targeted tests: f64 iterates bitwise
with equal counts (or the same divergence index), traces 1e-12, DST 1e-13,
FNS 1e-12."""
import numpy as np
import pytest

import oracle as O
import paper_2412_08076_b200 as G
from paper_2412_08076_b200 import fns as GF

pytestmark = pytest.mark.gpu


def _case(rng):
    n = int(rng.choice([5, 9, 17, 33, 48, 64, 65, 80, 100, 129]))
    variant = str(rng.choice(["plain", "mom", "nag", "nagex"]))
    m = int(rng.integers(1, 21))
    jac = bool(rng.integers(0, 2))
    check = str(rng.choice(["outer", "inner"]))
    eps, theta = 10 ** rng.uniform(-2, 0), rng.uniform(0, np.pi)
    return n, variant, m, jac, check, eps, theta


@pytest.mark.parametrize("seed", range(60))
def test_fuzz_solve_stationary(seed):
    rng = np.random.default_rng(1000 + seed)
    n, variant, m, jac, check, eps, theta = _case(rng)
    A = O.assemble_anisotropic(eps, theta, n)
    f = rng.standard_normal(A.shape[0])
    lam = np.linalg.eigvalsh(A.toarray()) if A.shape[0] <= 4300 else None
    lmax = lam[-1] if lam is not None else 8.0 * max(1.0, 1.0 / eps)
    scale = O.jacobi_scale(A) if jac else None
    s0 = (2.0 / 3.0) / A.diagonal()[0] if jac else 1.0
    w = rng.uniform(0.2, 1.0, m) / (s0 * lmax)
    if rng.integers(0, 4) == 0:
        w = w * 3.0                                     # often divergent
    al = rng.uniform(0.0, 0.6, m)
    at = rng.uniform(0.0, 0.6, m)
    kw = {} if variant == "plain" else {"alpha": al}
    if variant == "nagex":
        kw["alpha_tilde"] = at
    sched = G.WeightSchedule(omega=w, variant=variant, **kw)
    P = G.Preconditioner.weighted_jacobi(A) if jac else None
    tol, max_outer = 10 ** rng.uniform(-8, -3), int(rng.integers(0, 40))
    try:
        uo, ro = O.solve_stationary(A, f, w, None if variant == "plain" else al,
                                    at if variant == "nagex" else None, variant=variant,
                                    scale=scale, tol=tol, max_outer=max_outer, check=check)
    except O.OracleDivergence as e:
        with pytest.raises(G.DivergenceError) as ei:
            G.solve_stationary(A, f, sched, P=P, tol=tol, max_outer=max_outer, check=check)
        assert ei.value.inner_iteration == e.inner_iteration
        return
    u, rep = G.solve_stationary(A, f, sched, P=P, tol=tol, max_outer=max_outer, check=check)
    assert rep.iterations == ro["iterations"] and rep.inner_iterations == ro["inner_iterations"]
    assert np.array_equal(u, uo)
    t, to = np.asarray(rep.trace), np.asarray(ro["trace"])
    assert t.shape == to.shape and np.all(np.abs(t - to) <= 1e-12 * np.abs(to))


@pytest.mark.parametrize("seed", range(16))
def test_fuzz_dst_and_fns(seed):
    rng = np.random.default_rng(2000 + seed)
    side = int(rng.choice([3, 7, 10, 31, 50, 63, 127, 200, 255, 511]))
    x = rng.standard_normal((2, side * side))
    y = GF.dst2(x)
    for b in range(2):
        assert np.linalg.norm(y[b] - O.dst2(x[b])) <= 1e-13 * np.linalg.norm(x[b])
    n = side + 1
    if n <= 128:
        A = O.assemble_anisotropic(10 ** rng.uniform(-3, 0), rng.uniform(0, np.pi), n)
        f = rng.standard_normal(A.shape[0])
        u0 = rng.standard_normal(A.shape[0])
        lam = 0.01 * rng.standard_normal(A.shape[0])
        w = rng.uniform(0.05, 0.2, int(rng.integers(1, 5)))
        M = int(rng.integers(0, 9))
        u = GF.fns_lite_step(A, f, u0, G.WeightSchedule(omega=w), M, GF.SpectralCorrection(lam, n))
        uo = O.fns_lite_step(A, f, u0, w, M, lam)
        assert np.linalg.norm(u - uo) <= 1e-12 * np.linalg.norm(uo)

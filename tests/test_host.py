"""Host-side logic that needs no GPU: stencil extraction, problem mirrors,
schedules, and the C-ABI library itself (loads, exports every symbol)."""
import re
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2412_08076_b200 import _lib as L
from paper_2412_08076_b200.errors import UnsupportedOperator
from paper_2412_08076_b200.operator import classify, extract_planes
from paper_2412_08076_b200.problems import (OFFSETS9, AnisotropicProblem, HelmholtzProblem,
                                            anisotropic_stencil, helmholtz_stencil)
from paper_2412_08076_b200.schedules import (WeightSchedule, chebyshev_weights, leja_order,
                                             stencil_symbol_bounds)

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_header_symbol():
    """librichgpu.so loads without a GPU and exports all of include/*.h."""
    from paper_2412_08076_b200 import build
    build.build()
    lib = L.load()
    declared = set()
    for h in (ROOT / "include").glob("*.h"):
        declared |= set(re.findall(r"^\s*(?:int|const char\s*\*)\s+(rg_\w+)\s*\(", h.read_text(), re.M))
    assert declared, "no declarations found"
    assert declared == set(L.SYMBOLS), declared ^ set(L.SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.rg_version() == 1


@pytest.mark.parametrize("seed", range(4))
def test_anisotropic_stencil_bitwise_vs_csr(seed):
    """The 9 coefficients computed without assembly equal every row of the
    oracle's (== reference's) CSR assembly, bit for bit."""
    rng = np.random.default_rng(seed)
    for _ in range(8):
        eps, th, n = 10 ** rng.uniform(-6, 0), rng.uniform(0, np.pi), int(rng.integers(3, 30))
        A = O.assemble_anisotropic(eps, th, n)
        s, planes, present = extract_planes(A)
        kind, c = classify(s, planes, present)
        assert kind == "const9"
        mine = anisotropic_stencil(AnisotropicProblem(eps, th, n))
        assert np.array_equal(mine, c), (eps, th, n)
        assert np.array_equal(np.signbit(mine), np.signbit(c))


def test_dropped_entries_seven_point():
    A = O.assemble_anisotropic(0.5, 0.0, 24)
    s, planes, present = extract_planes(A)
    kind, c = classify(s, planes, present)
    assert kind == "const9" and np.count_nonzero(c) == 7
    assert np.array_equal(c, anisotropic_stencil(AnisotropicProblem(0.5, 0.0, 24)))


def test_helmholtz_extraction():
    n = 64
    w = 2 * np.pi * n / 10
    A = O.assemble_helmholtz(w, n)
    s, planes, present = extract_planes(A)
    kind, (off, diag) = classify(s, planes, present)
    assert kind == "diag5"
    off2, diag2 = helmholtz_stencil(HelmholtzProblem(w, n))
    assert np.array_equal(off, off2) and np.array_equal(diag, diag2)
    assert np.array_equal(diag, A.diagonal())


def test_galerkin_levels_are_var9():
    n = 32
    A = O.assemble_helmholtz(2 * np.pi * 3, n)
    levels, _ = O.build_hierarchy(A, n, coarsest=8)
    for L_ in levels[1:]:
        s, planes, present = extract_planes(L_["A"])
        kind, _ = classify(s, planes, present)
        assert kind == "var9"
        # scatter back reproduces the CSR exactly
        dense = L_["A"].toarray()
        x, y = np.divmod(np.arange(s * s), s)
        for q, (dx, dy) in enumerate(OFFSETS9):
            ok = (x + dx >= 0) & (x + dx < s) & (y + dy >= 0) & (y + dy < s)
            i = np.nonzero(ok)[0]
            assert np.array_equal(planes[q, i], dense[i, (x[i] + dx) * s + y[i] + dy])


def test_non_grid_matrices_rejected():
    import scipy.sparse as sp
    with pytest.raises(UnsupportedOperator):
        extract_planes(sp.identity(5, format="csr"))
    M = sp.lil_matrix((16, 16))
    M[0, 15] = 1.0
    with pytest.raises(UnsupportedOperator):
        extract_planes(M.tocsr())


def test_weight_schedule_validation():
    with pytest.raises(ValueError):
        WeightSchedule(omega=[0.1, 0.2], alpha=[0.1, 0.0])
    with pytest.raises(ValueError):
        WeightSchedule(omega=[0.1], alpha=[0.1], alpha_tilde=[0.2], variant="nag")
    with pytest.raises(ValueError):
        WeightSchedule(omega=[0.1], variant="heavy")
    s = WeightSchedule(omega=[0.1, 0.2], alpha=[0.3, 0.4], variant="nag")
    assert np.array_equal(s.alpha_tilde, s.alpha) and s.m == 2
    s = WeightSchedule(omega=0.5)
    assert s.m == 1 and np.array_equal(s.alpha, [0.0])


def test_chebyshev_closed_forms():
    # m = 1: omega = 2 / (lmax + lmin)  (test_schedules.py:9-24 analogue)
    assert np.allclose(chebyshev_weights(3.0, 1.0, 1), [0.5])
    w = chebyshev_weights(3.0, 1.0, 2)
    assert np.allclose(sorted(1 / w), sorted([2 - np.sqrt(0.5), 2 + np.sqrt(0.5)]))
    assert np.array_equal(chebyshev_weights(4.0, 0.5, 7), O.chebyshev_weights(4.0, 0.5, 7))


def test_leja_is_permutation_starting_at_largest_root():
    w = chebyshev_weights(8.0, 1e-3, 32)
    lw = leja_order(w)
    assert sorted(lw) == sorted(w)
    assert lw[0] == w.min()  # largest root 1/omega first


def test_symbol_bounds_match_dense_spectrum():
    p = AnisotropicProblem(0.1, 0.5, 24)
    c = anisotropic_stencil(p)
    lmax, lmin = stencil_symbol_bounds(c, p.n)
    lam = np.linalg.eigvalsh(O.assemble_anisotropic(0.1, 0.5, 24).toarray())
    assert lmax >= lam[-1] * (1 - 1e-3) and lmax <= lam[-1] * 1.05
    assert lam[0] / 8 <= lmin <= lam[0] * 1.001


@pytest.mark.reference
def test_reference_objects_are_accepted(richlab):
    """The drop-in consumes richlab's own objects: SparseMatrix (CSR arrays),
    Preconditioner.weighted_jacobi (scale recovered exactly through apply),
    WeightSchedule (duck-typed)."""
    from paper_2412_08076_b200.operator import precond_scale
    from paper_2412_08076_b200.richardson import _sched_list
    R = richlab
    p = R.AnisotropicProblem(0.01, 0.8, 24)
    A = R.assemble_anisotropic(p)
    s1, pl1, pr1 = extract_planes(A)
    s2, pl2, pr2 = extract_planes(A.to_scipy())
    assert s1 == s2 == 23 and np.array_equal(pl1, pl2) and np.array_equal(pr1, pr2)
    kind, c = classify(s1, pl1, pr1)
    assert kind == "const9" and np.array_equal(c, anisotropic_stencil(AnisotropicProblem(0.01, 0.8, 24)))
    P = R.Preconditioner.weighted_jacobi(A)
    sc = precond_scale(P, A.ncols)
    assert sc.ndim == 0 and sc == (2.0 / 3.0) / A.diagonal()[0]
    with pytest.raises(UnsupportedOperator):
        precond_scale(R.Preconditioner.ssor(A), A.ncols)
    ws = R.WeightSchedule(omega=[0.1, 0.2], alpha=[0.3, 0.4], variant="nag")
    (s,) = _sched_list(ws, 1)
    assert np.array_equal(s.alpha_tilde, [0.3, 0.4]) and s.m == 2
    H = R.assemble_helmholtz(R.HelmholtzProblem(2 * np.pi * 64 / 10, 64))
    kind, (off, diag) = classify(*extract_planes(H))
    assert kind == "diag5" and np.array_equal(diag, H.diagonal())

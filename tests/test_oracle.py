"""Pin the oracle (CPU restatement) against the reference's own outputs.

tests/golden/*.npz were produced by the unmodified reference
(tests/golden/make_golden.py).  The oracle must reproduce them bitwise:
same iterates, same iteration counts, same traces.  When the reference is
importable (dev container) it is also compared directly on fresh draws.
"""
import numpy as np
import pytest

import oracle as O
from conftest import sweep_case


def test_cfg1_bitwise(golden):
    d = golden("cfg1")
    A = O.assemble_anisotropic(float(d["eps"]), float(d["theta"]), int(d["n"]))
    u, rep = O.solve_stationary(A, d["f"], d["omega"], tol=1e-6)
    assert rep["iterations"] == d["iterations"] == 190
    assert rep["inner_iterations"] == d["inner_iterations"] == 1520
    assert np.array_equal(u, d["u"])
    assert np.array_equal(rep["trace"], d["trace"])


def test_sweep_cases_bitwise(golden):
    d = golden("sweeps")
    for i in range(int(d["count"])):
        c = sweep_case(d, i)
        A = O.assemble_anisotropic(c["eps"], c["theta"], c["n"])
        sc = O.jacobi_scale(A) if c["jacobi"] else None
        u, rep = O.solve_stationary(A, c["f"], c["omega"], c["alpha"], c["alpha_tilde"],
                                    str(c["variant"]), scale=sc, tol=c["tol"],
                                    max_outer=c["max_outer"], check=str(c["check"]))
        assert rep["iterations"] == c["iterations"], i
        assert rep["inner_iterations"] == c["inner_iterations"], i
        assert np.array_equal(u, c["u"]), i
        assert np.array_equal(rep["trace"], c["trace"]), i


def test_edge_cases(golden):
    d = golden("edge")
    A = O.assemble_anisotropic(0.3, 0.7, 12)
    with pytest.raises(O.OracleDivergence) as e:
        O.solve_stationary(A, d["div_f"], [50.0, 0.2], max_outer=5000)
    assert e.value.inner_iteration == d["div_inner"]
    assert str(e.value) == str(d["div_msg"])
    with pytest.raises(O.OracleDivergence) as e:
        O.solve_stationary(A, d["div_f"], [5.0, 0.1, 0.1], [0.1] * 3, variant="nag",
                           max_outer=5000)
    assert e.value.inner_iteration == d["divnag_inner"]
    u, rep = O.solve_stationary(A, np.zeros(A.shape[0]), [0.1])
    assert rep["iterations"] == d["zero_iterations"] and np.array_equal(rep["trace"], d["zero_trace"])
    u, rep = O.solve_stationary(A, d["init_f"], [0.1], u0=d["init_u0"])
    assert rep["iterations"] == d["init_iterations"] and np.array_equal(u, d["init_u"])
    A7 = O.assemble_anisotropic(0.5, 0.0, 24)
    assert A7.nnz == d["s7_nnz"]
    u, rep = O.solve_stationary(A7, d["s7_f"], d["s7_omega"], tol=1e-300, max_outer=9)
    assert np.array_equal(u, d["s7_u"]) and np.array_equal(rep["trace"], d["s7_trace"])


def test_outer_sweep_sequence(golden):
    d = golden("edge")
    A = O.assemble_anisotropic(0.05, 1.1, 16)
    sc = O.jacobi_scale(A)
    u = np.zeros(A.shape[0])
    v = np.zeros(A.shape[0])
    for k in range(3):
        u, v, h = O.outer_sweep(A, d["os_f"], u, v, [0.9, 1.3, 0.7], [0.2, 0.3, 0.1],
                                variant="nag", scale=sc, outer_count=k)
        assert np.array_equal(u, d["os_u"][k]) and np.array_equal(v, d["os_v"][k])
        assert h == d["os_hist"][k]


def test_helmholtz(golden):
    d = golden("helmholtz")
    A = O.assemble_helmholtz(float(d["omega_phys"]), int(d["n"]))
    assert np.array_equal(A.diagonal(), d["diag"])
    assert np.array_equal(A.dot(d["x"]), d["y"])
    u, rep = O.solve_stationary(A, d["f"], d["w"], np.full(4, 0.3), variant="nag", tol=1e-300,
                                max_outer=6)
    assert np.array_equal(u, d["u"]) and np.array_equal(rep["trace"], d["trace"])


def test_fns(golden):
    d = golden("fns")
    assert np.array_equal(O.dst2(d["x31"]), d["d31"])
    assert np.array_equal(O.dst2(d["x63"]), d["d63"])
    A = O.assemble_anisotropic(float(d["eps"]), float(d["theta"]), int(d["n"]))
    u1 = O.fns_lite_step(A, d["f"], np.zeros(A.shape[0]), np.full(8, 0.5), 8, d["lam"])
    assert np.array_equal(u1, d["u1"])
    u, rep = O.solve_fns(A, d["f"], np.full(8, 0.5), d["lam"], 8, tol=1e-300, max_iters=5)
    assert np.array_equal(u, d["u5"]) and np.array_equal(rep["trace"], d["trace5"])


def test_multigrid(golden):
    d = golden("multigrid")
    n = int(d["n"])
    A = O.assemble_helmholtz(float(d["omega_phys"]), n)
    levels, lu = O.build_hierarchy(A, n, coarsest=8)
    assert len(levels) == d["depth"]
    for k, L in enumerate(levels):
        assert np.array_equal(L["A"].data, d[f"A{k}_data"])
        assert np.array_equal(L["A"].indices, d[f"A{k}_indices"])
    assert np.array_equal(O.restriction(32).dot(d["r32"]), d["R32"])
    assert np.array_equal(O.prolongation(32).dot(d["e16"]), d["P16"])
    sched = dict(omega=np.full(4, 0.8 / (8 * n * n)), alpha=np.full(4, 0.3),
                 alpha_tilde=np.full(4, 0.3), variant="nag")
    u = O.v_cycle(levels, lu, d["f"], sched)
    assert np.array_equal(u, d["u"])
    ug, rep = O.fgmres(A, d["f"], lambda r: O.v_cycle(levels, lu, r, sched), restart=5,
                       tol=1e-6, max_outer=4)
    assert rep["iterations"] == d["fg_iterations"]
    assert np.array_equal(rep["trace"], d["fg_trace"]) and np.array_equal(ug, d["fg_u"])


def test_table2_known_answer(golden):
    d = golden("table2")
    for k in range(2):
        A = O.assemble_anisotropic(float(d[f"e{k}_eps"]), 0.0, 64)
        f = np.random.default_rng(0).standard_normal(A.shape[0])
        _, rep = O.solve_stationary(A, f, d[f"e{k}_omega"])
        assert rep["iterations"] == d[f"e{k}_iterations"]


@pytest.mark.reference
def test_oracle_matches_reference_fresh_draws(richlab):
    R = richlab
    rng = np.random.default_rng(123)
    for _ in range(6):
        eps, th, n = 10 ** rng.uniform(-4, 0), rng.uniform(0, np.pi), int(rng.integers(8, 40))
        A = R.assemble_anisotropic(R.AnisotropicProblem(eps, th, n))
        Ao = O.assemble_anisotropic(eps, th, n)
        assert np.array_equal(A.values, Ao.data) and np.array_equal(A.col_indices, Ao.indices)
        f = rng.standard_normal(A.ncols)
        lam = np.linalg.eigvalsh(A.to_dense())
        w = R.chebyshev_weights(lam[-1], lam[0], 5)
        u, rep = R.solve_stationary(A, f, R.WeightSchedule(omega=w), tol=1e-7)
        uo, ro = O.solve_stationary(Ao, f, w, tol=1e-7)
        assert np.array_equal(u, uo) and rep.iterations == ro["iterations"]


def _tri_from_golden(A, name):
    return {"gs": ("gauss-seidel", 1.0), "sor14": ("sor", 1.4), "ssor10": ("ssor", 1.0),
            "ssor13": ("ssor", 1.3)}[name]


def test_tri_precond_apply(golden):
    """GS / SOR / SSOR maps (precond.py:79-118) vs the reference's outputs."""
    d = golden("precond")
    for k in range(int(d["n_apply"])):
        A = O.assemble_anisotropic(float(d[f"a{k}_eps"]), float(d[f"a{k}_theta"]),
                                   int(d[f"a{k}_n"]))
        for name in ("gs", "sor14", "ssor10", "ssor13"):
            kind, relax = _tri_from_golden(A, name)
            z = O.tri_precond(A, kind, relax)(d[f"a{k}_r"])
            assert np.array_equal(z, d[f"a{k}_{name}"]), (k, name)


def test_tri_precond_solves(golden):
    """SSOR/SOR/GS-preconditioned solve_stationary vs the reference."""
    d = golden("precond")
    for k in range(int(d["n_solve"])):
        g = lambda key: d[f"s{k}_{key}"]  # noqa: E731
        A = O.assemble_anisotropic(float(g("eps")), float(g("theta")), int(g("n")))
        pre = O.tri_precond(A, str(g("kind")), float(g("relax")))
        try:
            u, rep = O.solve_stationary(A, g("f"), g("omega"), g("alpha"), g("alpha_tilde"),
                                        str(g("variant")), scale=pre, tol=float(g("tol")),
                                        max_outer=60)
        except O.OracleDivergence as e:
            assert e.inner_iteration == int(g("diverged"))
            continue
        assert int(g("diverged")) == -1
        assert np.array_equal(u, g("u")) and np.array_equal(rep["trace"], g("trace"))
        assert rep["iterations"] == int(g("iterations")) and rep["inner_iterations"] == int(g("inner"))


def test_unroll_grad_vs_reference_tape(golden):
    """Training unroll (training.py:61-104): loss and tape gradients."""
    d = golden("unroll")
    for k in range(int(d["count"])):
        g = lambda key: d[f"u{k}_{key}"]  # noqa: E731
        A = O.assemble_anisotropic(float(g("eps")), float(g("theta")), int(g("n")))
        pre = str(g("pre"))
        sc = O.jacobi_scale(A) if pre == "jacobi" else (
            O.tri_precond(A, {"gs": "gauss-seidel"}.get(pre, pre), 1.0) if pre in ("ssor", "gs")
            else None)
        if callable(sc):
            continue   # the oracle adjoint covers Jacobi; tri maps are checked on the device
        loss, dw, da, dat = O.unroll_grad(A, g("f"), g("omega"), g("alpha"), g("alpha_t"),
                                          int(g("K")), str(g("variant")), sc)
        assert loss == float(g("loss_free"))
        for got, want in ((dw, g("d_omega")), (da, g("d_alpha")), (dat, g("d_alpha_t"))):
            assert np.allclose(got, want, rtol=1e-12, atol=1e-15), (k, got, want)

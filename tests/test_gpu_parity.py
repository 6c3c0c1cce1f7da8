"""GPU solve loop vs the reference (golden fixtures) and the oracle.

Bar (north_star): f64 iterates bitwise equal (they are: same op order, no
FMA), identical iteration counts, residual traces within 1e-12 relative (the
norm is a different but deterministic reduction than BLAS ddot); f32 within
1e-5 of the f64 oracle.
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2412_08076_b200 as G
from conftest import sweep_case

pytestmark = pytest.mark.gpu

TRACE_RTOL = 1e-12


def _close_trace(a, b, rtol=TRACE_RTOL):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    assert np.all(np.abs(a - b) <= rtol * np.abs(b)), np.max(np.abs(a - b) / np.abs(b))


def _sched(c):
    kw = {}
    if c["variant"] != "plain":
        kw["alpha"] = c["alpha"]
    if c["variant"] == "nagex":
        kw["alpha_tilde"] = c["alpha_tilde"]
    return G.WeightSchedule(omega=c["omega"], variant=str(c["variant"]), **kw)


def test_cfg1_golden_bitwise(golden):
    """SURVEY §7.3 minimum slice: cfg1 solved on the GPU == reference."""
    d = golden("cfg1")
    A = O.assemble_anisotropic(float(d["eps"]), float(d["theta"]), int(d["n"]))
    u, rep = G.solve_stationary(A, d["f"], G.WeightSchedule(omega=d["omega"]), tol=1e-6)
    assert rep.converged
    assert rep.iterations == d["iterations"] == 190
    assert rep.inner_iterations == d["inner_iterations"] == 1520
    assert np.array_equal(u, d["u"])
    _close_trace(rep.trace, d["trace"])


@pytest.mark.parametrize("block_T", [0, 1, 3, 8])
def test_sweep_cases_golden(golden, block_T):
    """All variants x Jacobi x check, converged and fixed-sweep runs."""
    d = golden("sweeps")
    for i in range(int(d["count"])):
        c = sweep_case(d, i)
        A = O.assemble_anisotropic(c["eps"], c["theta"], c["n"])
        P = G.JacobiScale(O.jacobi_scale(A)) if c["jacobi"] else None
        u, rep = G.solve_stationary(A, c["f"], _sched(c), P=P, tol=c["tol"],
                                    max_outer=c["max_outer"], check=str(c["check"]),
                                    block_T=block_T)
        assert rep.iterations == c["iterations"], (i, rep.iterations, c["iterations"])
        assert rep.inner_iterations == c["inner_iterations"], i
        assert rep.converged == bool(c["converged"]), i
        assert np.array_equal(u, c["u"]), (i, np.max(np.abs(u - c["u"])))
        _close_trace(rep.trace, c["trace"])


def test_batched_equals_per_system(golden):
    """A batch of systems with different stopping points: each system's
    result equals its own golden run (active masks stop finished systems)."""
    d = golden("sweeps")
    idx = [i for i in range(int(d["count"]))
           if sweep_case(d, i)["variant"] == "plain" and sweep_case(d, i)["n"] == 16
           and not sweep_case(d, i)["jacobi"] and sweep_case(d, i)["check"] == "outer"]
    cases = [sweep_case(d, i) for i in idx]
    ops = [G.GpuStencilOperator.from_sparse(O.assemble_anisotropic(c["eps"], c["theta"], c["n"]))
           for c in cases]
    op = G.GpuStencilOperator.stack(ops)
    # same tolerance needed for a batch: use the converging runs only
    cases = [c for c in cases if c["tol"] == 1e-8]
    op = G.GpuStencilOperator.stack([ops[k] for k, c in enumerate(
        [sweep_case(d, i) for i in idx]) if c["tol"] == 1e-8])
    F = np.stack([c["f"] for c in cases])
    res = G.solve_stationary_batched(op, F, [_sched(c) for c in cases], tol=1e-8, max_outer=400)
    for (u, rep), c in zip(res, cases):
        assert rep.iterations == c["iterations"]
        assert np.array_equal(u, c["u"])


def test_edge_cases(golden):
    d = golden("edge")
    A = O.assemble_anisotropic(0.3, 0.7, 12)
    with pytest.raises(G.DivergenceError) as e:
        G.solve_stationary(A, d["div_f"], G.WeightSchedule(omega=[50.0, 0.2]), max_outer=5000)
    assert e.value.inner_iteration == d["div_inner"]
    assert str(e.value).split(" at ")[1] == str(d["div_msg"]).split(" at ")[1]
    with pytest.raises(G.DivergenceError) as e:
        G.solve_stationary(A, d["div_f"], G.WeightSchedule(omega=[5.0, 0.1, 0.1],
                                                           alpha=[0.1] * 3, variant="nag"),
                           max_outer=5000)
    assert e.value.inner_iteration == d["divnag_inner"]
    u, rep = G.solve_stationary(A, np.zeros(A.shape[0]), G.WeightSchedule(omega=[0.1]))
    assert rep.iterations == d["zero_iterations"] and np.array_equal(rep.trace, d["zero_trace"])
    assert rep.converged and not np.any(u)
    u, rep = G.solve_stationary(A, d["init_f"], G.WeightSchedule(omega=[0.1]), u0=d["init_u0"])
    assert rep.iterations == d["init_iterations"] == 0 and np.array_equal(u, d["init_u"])
    _close_trace(rep.trace, d["init_trace"], rtol=1e-6)
    u, rep = G.solve_stationary(A, d["div_f"], G.WeightSchedule(omega=[0.1]), max_outer=0)
    assert not rep.converged and len(rep.trace) == 1
    _close_trace(rep.trace, d["zero_outer_trace"])
    A7 = O.assemble_anisotropic(0.5, 0.0, 24)
    u, rep = G.solve_stationary(A7, d["s7_f"], G.WeightSchedule(omega=d["s7_omega"]),
                                tol=1e-300, max_outer=9)
    assert np.array_equal(u, d["s7_u"])
    _close_trace(rep.trace, d["s7_trace"])
    with pytest.raises(ValueError):
        G.solve_stationary(A, d["div_f"], G.WeightSchedule(omega=[0.1]), tol=0.0)
    with pytest.raises(ValueError):
        G.solve_stationary(A, d["div_f"], G.WeightSchedule(omega=[0.1]), check="middle")
    with pytest.raises(G.DimensionMismatch):
        G.solve_stationary(A, d["div_f"][:-1], G.WeightSchedule(omega=[0.1]))


def test_outer_sweep_and_identity(golden):
    d = golden("edge")
    A = O.assemble_anisotropic(0.05, 1.1, 16)
    P = G.JacobiScale(O.jacobi_scale(A))
    sched = G.WeightSchedule(omega=[0.9, 1.3, 0.7], alpha=[0.2, 0.3, 0.1], variant="nag")
    st = G.IterationState.start(A.shape[0])
    for k in range(3):
        G.outer_sweep(A, d["os_f"], st, sched, P)
        assert np.array_equal(st.u, d["os_u"][k]) and np.array_equal(st.v, d["os_v"][k])
    assert np.allclose(st.residual_history, d["os_hist"], rtol=1e-12, atol=0)
    import scipy.sparse as sp
    st = G.IterationState.start(4)
    G.outer_sweep(sp.identity(4, format="csr"), np.array([1.0, 2.0, 3.0, 4.0]), st,
                  G.WeightSchedule(omega=[1.0]))
    assert np.array_equal(st.u, d["id_u"])
    st = G.IterationState.start(4)
    with pytest.raises(G.DivergenceError) as e:
        for _ in range(60):
            G.outer_sweep(sp.identity(4, format="csr") * 1e4, np.ones(4), st,
                          G.WeightSchedule(omega=[1e300, 1e300]))
    assert e.value.inner_iteration == d["osdiv_inner"]
    assert str(e.value) == str(d["osdiv_msg"])


def test_helmholtz_matvec_and_nag(golden):
    d = golden("helmholtz")
    A = O.assemble_helmholtz(float(d["omega_phys"]), int(d["n"]))
    op = G.GpuStencilOperator.from_sparse(A)
    assert op.kind == 2  # DIAG5
    assert np.array_equal(op.matvec(d["x"]), d["y"])
    s = G.WeightSchedule(omega=d["w"], alpha=np.full(4, 0.3), variant="nag")
    u, rep = G.solve_stationary(op, d["f"], s, tol=1e-300, max_outer=6)
    assert np.array_equal(u, d["u"])
    _close_trace(rep.trace, d["trace"])


def test_var9_matvec_galerkin(golden):
    d = golden("multigrid")
    import scipy.sparse as sp
    for k in range(1, int(d["depth"])):
        A = sp.csr_matrix((d[f"A{k}_data"], d[f"A{k}_indices"], d[f"A{k}_indptr"]))
        op = G.GpuStencilOperator.from_sparse(A)
        assert op.kind == 3
        rng = np.random.default_rng(k)
        x = rng.standard_normal(A.shape[0]) + 1j * rng.standard_normal(A.shape[0])
        assert np.array_equal(op.matvec(x), A.dot(x))
        assert np.array_equal(op.rmatvec(x), A.T.dot(x))


def test_const9_matvec_rmatvec_random():
    rng = np.random.default_rng(3)
    for n in (3, 17, 64, 200):
        A = O.assemble_anisotropic(10 ** rng.uniform(-5, 0), rng.uniform(0, np.pi), n)
        op = G.GpuStencilOperator.from_sparse(A)
        x = rng.standard_normal(A.shape[0])
        assert np.array_equal(op.matvec(x), A.dot(x))
        assert np.array_equal(op.rmatvec(x), A.T.dot(x))
        r, n2 = op.residual(x, 2 * x)
        ref = 2 * x - A.dot(x)
        assert np.array_equal(r.cpu().numpy().ravel(), ref)
        assert abs(np.sqrt(n2.item()) - np.linalg.norm(ref)) <= 1e-13 * np.linalg.norm(ref)


def test_f32_within_1e5_of_f64_oracle():
    """cfg2 precision mode: float32 iterates vs the float64 reference."""
    rng = np.random.default_rng(2)
    A = O.assemble_anisotropic(10 ** rng.uniform(-3, 0), rng.uniform(0, np.pi), 64)
    f = rng.standard_normal(A.shape[0])
    w = np.full(16, 0.127)
    a = np.full(16, 0.12)
    op32 = G.GpuStencilOperator.from_sparse(A, dtype=np.float32)
    s = G.WeightSchedule(omega=w, alpha=a, variant="nag")
    u32, rep32 = G.solve_stationary(op32, f.astype(np.float32), s, tol=1e-300, max_outer=20)
    u64, ro = O.solve_stationary(A, f, w, a, variant="nag", tol=1e-300, max_outer=20)
    assert np.linalg.norm(u32 - u64) <= 1e-5 * np.linalg.norm(u64)
    assert np.all(np.abs(rep32.trace - ro["trace"]) <= 1e-5 * ro["trace"])


def test_full_size_one_sweep_bitwise():
    """BASELINE size (1023^2, Jacobi Richardson m=32): one outer sweep on the
    GPU (temporal blocking on) equals the oracle bit for bit."""
    rng = np.random.default_rng(3)
    eps, th, n = 10 ** rng.uniform(-4, 0), rng.uniform(0, np.pi), 1024
    A = O.assemble_anisotropic(eps, th, n)
    f = rng.standard_normal(A.shape[0])
    sc = O.jacobi_scale(A)
    c = G.anisotropic_stencil(G.AnisotropicProblem(eps, th, n))
    lmax, lmin = G.stencil_symbol_bounds(c, n)
    w = G.leja_order(G.chebyshev_weights(sc[0] * lmax, sc[0] * lmin, 32))
    u, rep = G.solve_stationary(A, f, G.WeightSchedule(omega=w), P=G.JacobiScale(sc),
                                tol=1e-300, max_outer=1)
    uo, ro = O.solve_stationary(A, f, w, scale=sc, tol=1e-300, max_outer=1)
    assert rep.inner_iterations == ro["inner_iterations"] == 32
    assert np.array_equal(u, uo)
    _close_trace(rep.trace, ro["trace"])


def test_block_depths_agree_bitwise():
    """Every temporal-blocking depth produces the same bits (T=1..8), NAG too."""
    rng = np.random.default_rng(4)
    A = O.assemble_anisotropic(0.02, 0.9, 150)
    f = rng.standard_normal(A.shape[0])
    lam_hi = 3.5
    for variant, kw in (("plain", {}), ("mom", {"alpha": np.full(10, 0.3)}),
                        ("nag", {"alpha": np.full(10, 0.3)})):
        w = np.full(10, 0.8 / lam_hi) if variant != "plain" else \
            G.chebyshev_weights(lam_hi, 0.01, 10)
        s = G.WeightSchedule(omega=w, variant=variant, **kw)
        outs = []
        for T in range(1, 9):
            u, rep = G.solve_stationary(A, f, s, tol=1e-300, max_outer=3, block_T=T)
            outs.append((u, rep.trace))
        for u, tr in outs[1:]:
            assert np.array_equal(u, outs[0][0])
        uo, _ = O.solve_stationary(A, f, s.omega, s.alpha, s.alpha_tilde, variant, tol=1e-300,
                                   max_outer=3)
        assert np.array_equal(outs[0][0], uo)


def test_torch_inputs_stay_on_device():
    A = O.assemble_anisotropic(0.1, 0.3, 32)
    f = torch.randn(A.shape[0], dtype=torch.float64, device="cuda")
    u, rep = G.solve_stationary(A, f, G.WeightSchedule(omega=[0.2, 0.3]), tol=1e-300,
                                max_outer=2)
    assert isinstance(u, torch.Tensor) and u.is_cuda
    uo, _ = O.solve_stationary(A, f.cpu().numpy(), [0.2, 0.3], tol=1e-300, max_outer=2)
    assert np.array_equal(u.cpu().numpy(), uo)


def test_f32_cfg2_hard_system_within_1e5():
    """cfg2 system 0 (eps 3e-4, the worst-conditioned of the first draws):
    f32 vectors with f64 arithmetic stay within 1e-5 of the f64 oracle after
    the full 200 NAG(16) sweeps (pure f32 arithmetic gives 1.4e-5)."""
    from paper_2412_08076_b200 import configs as CF
    c = CF.cfg2(batch=1)
    p, s, f = c["problems"][0], c["schedules"][0], c["F"][0]
    A = O.assemble_anisotropic(p.epsilon, p.theta, 256)
    op32 = G.GpuStencilOperator.from_problems([p], dtype=np.float32)
    u32, rep = G.solve_stationary(op32, f.astype(np.float32), s, tol=1e-300, max_outer=200)
    uo, ro = O.solve_stationary(A, f, s.omega, s.alpha, variant="nag", tol=1e-300, max_outer=200)
    assert np.linalg.norm(u32 - uo) <= 1e-5 * np.linalg.norm(uo)
    assert np.all(np.abs(rep.trace - ro["trace"]) <= 1e-5 * ro["trace"])


def test_spectral_bounds_vs_oracle_recipe(golden):
    """GPU power iterations (spectral.py drop-in): the cfg1 50-step recipe and
    the converged estimators agree with the reference's numbers."""
    from paper_2412_08076_b200 import spectral as GS
    d = golden("cfg1")
    A = O.assemble_anisotropic(float(d["eps"]), float(d["theta"]), int(d["n"]))
    lmax, _ = GS.power_iterations(A, 50, seed=0)
    assert abs(lmax - float(d["lmax50"])) <= 1e-12 * abs(float(d["lmax50"]))
    sig = 1.01 * lmax
    ls, _ = GS.power_iterations(A, 50, seed=0, shift=sig)
    assert abs((sig - ls) - float(d["lmin50"])) <= 1e-10 * float(d["lmin50"])
    b = GS.estimate_lambda_max(A, tol=1e-10)
    lam = np.linalg.eigvalsh(A.toarray())
    assert abs(b.lambda_max - lam[-1]) <= 1e-6 * lam[-1]
    with pytest.raises(GS.PowerIterationError):
        GS.estimate_lambda_min(A, b.lambda_max, tol=1e-14, max_iter=20)


def test_cfg2_full_system_bitwise():
    """One full cfg2 system at BASELINE size (255^2, NAG(16), 200 sweeps,
    MLP weights) on the GPU equals the oracle bit for bit."""
    from paper_2412_08076_b200 import configs as CF
    c = CF.cfg2(batch=2)
    p, s, f = c["problems"][1], c["schedules"][1], c["F"][1]
    A = O.assemble_anisotropic(p.epsilon, p.theta, 256)
    u, rep = G.solve_stationary(A, f, s, tol=1e-300, max_outer=200)
    uo, ro = O.solve_stationary(A, f, s.omega, s.alpha, variant="nag", tol=1e-300, max_outer=200)
    assert rep.inner_iterations == ro["inner_iterations"] == 3200
    assert np.array_equal(u, uo)
    _close_trace(rep.trace, ro["trace"])


def test_table2_known_answer_counts(golden):
    """Acceptance criterion 1 analogue (test_acceptance.py:42-66): Chebyshev
    m=3, N=64, theta=0, seed 0 -- the GPU reproduces the reference's
    iteration counts exactly."""
    d = golden("table2")
    for k in range(2):
        A = O.assemble_anisotropic(float(d[f"e{k}_eps"]), 0.0, 64)
        f = np.random.default_rng(0).standard_normal(A.shape[0])
        _, rep = G.solve_stationary(A, f, G.WeightSchedule(omega=d[f"e{k}_omega"]))
        assert rep.iterations == d[f"e{k}_iterations"]
        assert rep.inner_iterations == d[f"e{k}_inner"]


@pytest.mark.parametrize("variant", ["plain", "nag"])
def test_batch_above_64_systems_blocked(variant):
    """70 systems on 79^2 grids: the blocked sweep runs in launches of at most
    64 systems (kernel-parameter coefficients).  plain: Jacobi + Leja-ordered
    Chebyshev weights, systems converge at different sweeps and are skipped
    afterwards; nag: the same weights with momentum 0.3, most systems
    diverge at different inner indices.  Systems 0, 63, 64, 69 and a random
    one equal their own oracle runs: bitwise iterates and counts, or the same
    DivergenceError inner index."""
    rng = np.random.default_rng(70)
    B, n, m = 70, 80, 8
    probs = [G.AnisotropicProblem(10 ** rng.uniform(-1, 0), rng.uniform(0, np.pi), n)
             for _ in range(B)]
    op = G.GpuStencilOperator.from_problems(probs)
    F = rng.standard_normal((B, op.P))
    scheds, P = [], []
    for p in probs:
        lmax, lmin = G.stencil_symbol_bounds(G.anisotropic_stencil(p), n)
        s = 2.0 / 3.0 / G.anisotropic_stencil(p)[4]
        w = G.leja_order(G.chebyshev_weights(s * lmax, s * lmin, m))
        if variant == "plain":
            scheds.append(G.WeightSchedule(omega=w))
            P.append(G.JacobiScale(np.float64(s)))
        else:
            scheds.append(G.WeightSchedule(omega=w * s, alpha=np.full(m, 0.3), variant="nag"))
    res = G.solve_stationary_batched(op, F, scheds, P if variant == "plain" else None,
                                     tol=1e-2, max_outer=80)
    if variant == "plain":
        assert len({r.iterations for _, r in res}) > 1, "systems should stop at different sweeps"
    for b in sorted({0, 63, 64, 69, int(rng.integers(1, 62))}):
        A = O.assemble_anisotropic(probs[b].epsilon, probs[b].theta, n)
        s = scheds[b]
        u, rep = res[b]
        try:
            if variant == "plain":
                uo, ro = O.solve_stationary(A, F[b], s.omega, scale=O.jacobi_scale(A), tol=1e-2,
                                            max_outer=80)
            else:
                uo, ro = O.solve_stationary(A, F[b], s.omega, s.alpha, variant="nag", tol=1e-2,
                                            max_outer=80)
        except O.OracleDivergence as e:
            assert u is None and isinstance(rep, G.DivergenceError), b
            assert rep.inner_iteration == e.inner_iteration, b
            continue
        assert rep.iterations == ro["iterations"] and rep.inner_iterations == ro["inner_iterations"]
        assert np.array_equal(u, uo), b
        _close_trace(rep.trace, ro["trace"])


@pytest.mark.parametrize("m,check,variant", [(20, "outer", "plain"), (8, "inner", "plain"),
                                             (20, "outer", "mom"), (12, "inner", "mom")])
def test_cluster_solver_decision_paths(m, check, variant):
    """The single-launch cluster solver's two plain/mom loops: the per-sweep
    batched decision (check="outer", m <= 16) and the per-step lagged one
    (check="inner" or m > 16), against the oracle: bitwise iterates, equal
    counts, traces within 1e-12; a divergent schedule raises at the same
    inner index."""
    rng = np.random.default_rng(m)
    A = O.assemble_anisotropic(0.2, 0.6, 48)
    f = rng.standard_normal(A.shape[0])
    lam = np.linalg.eigvalsh(A.toarray())
    w = G.leja_order(G.chebyshev_weights(lam[-1], lam[0], m))
    al = np.full(m, 0.1) if variant == "mom" else None
    s = G.WeightSchedule(omega=w, alpha=al, variant=variant) if al is not None else \
        G.WeightSchedule(omega=w)
    if variant == "mom":   # heavy ball: constant 1/lambda_max, alpha 0.8
        w, al = np.full(m, 1.0 / lam[-1]), np.full(m, 0.8)
        s = G.WeightSchedule(omega=w, alpha=al, variant=variant)
    u, rep = G.solve_stationary(A, f, s, tol=1e-7, check=check, max_outer=2000)
    uo, ro = O.solve_stationary(A, f, w, al, variant=variant, tol=1e-7, check=check,
                                max_outer=2000)
    assert ro["converged"]
    assert rep.iterations == ro["iterations"] and rep.inner_iterations == ro["inner_iterations"]
    assert np.array_equal(u, uo)
    _close_trace(rep.trace, ro["trace"])
    # divergence: weights far above 2 / lambda_max
    sd = G.WeightSchedule(omega=np.full(m, 3.0 / lam[-1]))
    with pytest.raises(G.DivergenceError) as ei:
        G.solve_stationary(A, f, sd, tol=1e-7, check=check, max_outer=2000)
    with pytest.raises(O.OracleDivergence) as eo:
        O.solve_stationary(A, f, np.full(m, 3.0 / lam[-1]), tol=1e-7, check=check, max_outer=2000)
    assert ei.value.inner_iteration == eo.value.inner_iteration

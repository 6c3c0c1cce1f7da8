"""BASELINE-size parity: the full cfg2 / cfg3 / cfg4 / cfg5 runs against
goldens produced by the unmodified reference (tests/golden/make_golden_full.py,
SURVEY.md §8(d)).

* cfg3 (richardson.py:77-141 with weighted Jacobi, 8 x 1023^2 to 1e-6):
  identical outer / inner counts and convergence flags, traces within 1e-12,
  u bitwise (sha256).
* cfg2 (NAG(16), 64 x 255^2, 200 sweeps): u bitwise (sha256) for all 64
  systems in f64, traces within 1e-12; the f32-vector mode within 1e-5.
* cfg4 (fns.py:87-105, 4 x 1023^2, 100 alternations): the DST is not
  pocketfft-bitwise, so traces and the u digest (norm, 1024 sampled entries,
  4 seeded projections) are compared to a tolerance (bar below).
* cfg5 (fgmres.py:31-131 with the V-cycle of multigrid.py:141-163, 4 right-
  hand sides of 1023^2 c128): same Arnoldi-step counts and flags, recurrence
  residual history and the u digest to the bar below.

The inputs are regenerated from their seeds (their sha256 is checked against
the golden first) except the network-produced schedules, which the goldens
carry.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

sys.path.insert(0, str(Path(__file__).parent / "golden"))
from digest import digest, sha  # noqa: E402

import paper_2412_08076_b200 as G  # noqa: E402
from paper_2412_08076_b200 import configs as CF  # noqa: E402
from paper_2412_08076_b200.schedules import WeightSchedule  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"

# Tolerance paths (the DST is not pocketfft-bitwise; the MGS dot products and
# the coarsest solve are not BLAS / LAPACK-bitwise):
#  * cfg4: traces and the u digest within 1e-12 (the north-star bar);
#  * cfg5: the recurrence residual history within 1e-11 (measured 1.7e-12
#    after 100 Arnoldi steps); u within 1e-8 -- FGMRES(20) has not converged
#    (rel ~0.31), so u = sum Z_k y_k carries the conditioning of the 20 x 20
#    Hessenberg least-squares solves: ~1e-16 V-cycle differences reach u at
#    ~3e-9 while the residual norms agree to 1e-12.
FNS_BAR = 1e-12
FGMRES_TRACE_BAR = 1e-11
FGMRES_U_BAR = 1e-8


def _gold(name):
    p = GOLD / f"{name}.npz"
    if not p.exists():
        pytest.skip(f"{p.name} not generated (tests/golden/make_golden_full.py)")
    return np.load(p)


def _trace_rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


# ----------------------------------------------------------------- cfg3
def test_cfg3_full_solve_to_tol():
    g = _gold("full_cfg3")
    wl = CF.cfg3()
    B = len(wl["problems"])
    assert int(g["count"]) == B
    for b in range(B):
        assert sha(wl["F"][b]) == str(g[f"s{b}_f_sha"]), f"cfg3 f of system {b} differs"
        assert np.array_equal(wl["schedules"][b].omega, g[f"s{b}_omega"])
        assert wl["scales"][b] == float(g[f"s{b}_scale"])
    op = G.GpuStencilOperator.from_problems(wl["problems"])
    P = [G.JacobiScale(np.float64(s)) for s in wl["scales"]]
    res = G.solve_stationary_batched(op, wl["F"], wl["schedules"], P, tol=float(g["tol"]),
                                     max_outer=int(g["max_outer"]))
    for b, (u, rep) in enumerate(res):
        assert rep.iterations == int(g[f"s{b}_iterations"]), b
        assert rep.inner_iterations == int(g[f"s{b}_inner"]), b
        assert bool(rep.converged) == bool(g[f"s{b}_converged"]), b
        assert _trace_rel(rep.trace, g[f"s{b}_trace"]) <= 1e-12, b
        assert sha(np.ascontiguousarray(u)) == str(g[f"s{b}_u_sha"]), f"cfg3 u of system {b}"


# ----------------------------------------------------------------- cfg2
@pytest.fixture(scope="module")
def cfg2_inputs():
    g = _gold("full_cfg2")
    c = CF.cfg2()
    B = int(g["count"])
    scheds = [WeightSchedule(omega=g[f"s{b}_omega"], alpha=g[f"s{b}_alpha"], variant="nag")
              for b in range(B)]
    for b in range(B):
        assert sha(c["F"][b]) == str(g[f"s{b}_f_sha"]), f"cfg2 f of system {b} differs"
    return g, c, scheds


def test_cfg2_full_f64_bitwise(cfg2_inputs):
    g, c, scheds = cfg2_inputs
    op = G.GpuStencilOperator.from_problems(c["problems"])
    res = G.solve_stationary_batched(op, c["F"], scheds, None, tol=1e-300,
                                     max_outer=int(g["outer"]))
    for b, (u, rep) in enumerate(res):
        assert rep.iterations == int(g[f"s{b}_iterations"])
        assert rep.inner_iterations == int(g[f"s{b}_inner"])
        assert _trace_rel(rep.trace, g[f"s{b}_trace"]) <= 1e-12, b
        assert sha(np.ascontiguousarray(u)) == str(g[f"s{b}_u_sha"]), f"cfg2 u of system {b}"


def test_cfg2_full_f32_vectors(cfg2_inputs):
    """f32 vectors / f64 arithmetic against the f64 reference: 1e-5 (north star)."""
    g, c, scheds = cfg2_inputs
    op = G.GpuStencilOperator.from_problems(c["problems"], dtype=np.float32)
    res = G.solve_stationary_batched(op, c["F"].astype(np.float32), scheds, None, tol=1e-300,
                                     max_outer=int(g["outer"]))
    worst = 0.0
    for b, (u, rep) in enumerate(res):
        u64 = np.asarray(u, dtype=np.float64)
        d = digest(u64)
        norm = float(g[f"s{b}_u_norm"])
        worst = max(worst, abs(d["norm"] - norm) / norm,
                    float(np.linalg.norm(d["sample"] - g[f"s{b}_u_sample"]) /
                          np.linalg.norm(g[f"s{b}_u_sample"])))
        assert _trace_rel(rep.trace, g[f"s{b}_trace"]) <= 1e-5, b
    assert worst <= 1e-5, worst


# ----------------------------------------------------------------- cfg4
def test_cfg4_full_100_alternations():
    g = _gold("full_cfg4")
    from paper_2412_08076_b200 import fns as GF
    c = CF.cfg4(device="cuda")
    B = int(g["count"])
    sched = WeightSchedule(omega=np.full(8, 0.5))
    worst_trace, worst_u = 0.0, 0.0
    for b in range(B):
        p = c["problems"][b]
        f = c["F"][b]
        assert sha(f) == str(g[f"s{b}_f_sha"])
        lam = CF.fns_symbol_portable(p.theta, p.epsilon, p.n)
        assert sha(lam) == str(g[f"s{b}_lam_sha"]), \
            "the CPU conv-net symbol differs from the golden's (different BLAS rounding)"
        op = G.GpuStencilOperator.from_problems([p])
        u, rep = GF.solve_fns(op, f, sched, GF.SpectralCorrection(lam, p.n), int(g["M"]),
                              tol=1e-300, max_iters=int(g["alternations"]))
        assert rep.iterations == int(g[f"s{b}_iterations"])
        worst_trace = max(worst_trace, _trace_rel(rep.trace, g[f"s{b}_trace"]))
        d = digest(u)
        norm = float(g[f"s{b}_u_norm"])
        worst_u = max(worst_u, abs(d["norm"] - norm) / norm,
                      float(np.linalg.norm(d["sample"] - g[f"s{b}_u_sample"]) /
                            np.linalg.norm(g[f"s{b}_u_sample"])),
                      float(np.max(np.abs(d["proj"] - g[f"s{b}_u_proj"]) /
                                   np.abs(g[f"s{b}_u_proj"]))))
    print(f"cfg4 100 alternations: trace max rel {worst_trace:.3g}, u digest max rel {worst_u:.3g}")
    assert worst_trace <= FNS_BAR, worst_trace
    assert worst_u <= FNS_BAR, worst_u


# ----------------------------------------------------------------- cfg5
def test_cfg5_full_fgmres_vcycle():
    g = _gold("full_cfg5")
    import oracle as O   # host CSR assembly only (the hierarchy's Galerkin setup input)
    import importlib
    GG = importlib.import_module("paper_2412_08076_b200.fgmres")
    from paper_2412_08076_b200 import multigrid as GM
    c = CF.cfg5(device="cuda")
    hp, F = c["problem"], c["F"]
    B = int(g["count"])
    for b in range(B):
        assert sha(F[b]) == str(g[f"s{b}_f_sha"])
    sched = WeightSchedule(omega=g["s0_omega"], alpha=g["s0_alpha"], variant="nag")
    A = O.assemble_helmholtz(hp.angular_frequency, hp.n)
    h = GM.build_hierarchy(A, hp.n, coarsest=int(g["coarsest"]), schedules=sched, batch=B)
    assert h.depth == int(g["s0_depth"])
    op = G.GpuStencilOperator.from_problems([hp]).broadcast(B)
    res = GG.fgmres_batched(op, F, precond_apply=h.apply,
                            cfg=GG.FgmresConfig(restart=int(g["restart"]), tol=1e-6,
                                                max_outer=int(g["max_outer"])))
    worst_trace, worst_u = 0.0, 0.0
    for b, (u, rep) in enumerate(res):
        assert rep.iterations == int(g[f"s{b}_iterations"]), b
        assert bool(rep.converged) == bool(g[f"s{b}_converged"])
        assert bool(rep.stagnated) == bool(g[f"s{b}_stagnated"])
        worst_trace = max(worst_trace, _trace_rel(rep.trace, g[f"s{b}_trace"]))
        d = digest(u)
        norm = float(g[f"s{b}_u_norm"])
        worst_u = max(worst_u, abs(d["norm"] - norm) / norm,
                      float(np.linalg.norm(d["sample"] - g[f"s{b}_u_sample"]) /
                            np.linalg.norm(g[f"s{b}_u_sample"])),
                      float(np.max(np.abs(d["proj"] - g[f"s{b}_u_proj"]) /
                                   np.abs(g[f"s{b}_u_proj"]))))
    print(f"cfg5 FGMRES(20)x5: trace max rel {worst_trace:.3g}, u digest max rel {worst_u:.3g}")
    assert worst_trace <= FGMRES_TRACE_BAR, worst_trace
    assert worst_u <= FGMRES_U_BAR, worst_u

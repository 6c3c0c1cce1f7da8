"""Generate tests/golden/*.npz by running the UNMODIFIED reference (richlab).

Run in the dev container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture stores the seeded inputs next to the reference's outputs so
the tests never need the reference at run time.  Inputs follow SURVEY.md
§8(d) where a config is named; the rest are small variations that exercise
each code path (variants, Jacobi, check modes, edge cases).
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("RICHLAB_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import richlab as R  # noqa: E402
from richlab import fns as RF  # noqa: E402
from richlab import multigrid as RM  # noqa: E402
from richlab.richardson import DivergenceError  # noqa: E402

OUT = Path(__file__).resolve().parent


def interior_row(A, s):
    """The 9 CSR coefficients of the centre node (zero if absent)."""
    i = (s // 2) * s + s // 2
    c = np.zeros(9, dtype=A.values.dtype)
    for jj in range(A.row_starts[i], A.row_starts[i + 1]):
        j = A.col_indices[jj]
        dx, dy = j // s - i // s, j % s - i % s
        c[(dx + 1) * 3 + (dy + 1)] = A.values[jj]
    return c


def power50(A, seed=0, steps=50):
    """cfg1 recipe: 50 power steps (mirrors spectral.py:31-57 without the
    convergence test), then 50 shifted steps with sigma = 1.01 lmax."""
    def run(mv):
        rng = np.random.default_rng(seed)
        x = rng.standard_normal(A.ncols)
        x /= np.linalg.norm(x)
        lam = 0.0
        for _ in range(steps):
            y = mv(x)
            lam = float(np.real(np.vdot(x, y)))
            x = y / np.linalg.norm(y)
        return lam
    lmax = run(A.matvec)
    sigma = 1.01 * lmax
    lmin = sigma - run(lambda x: sigma * x - A.matvec(x))
    return lmax, lmin


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz ({(OUT / f'{name}.npz').stat().st_size // 1024} KiB)")


def cfg1():
    p = R.AnisotropicProblem(1e-2, np.pi / 6, 64)
    A = R.assemble_anisotropic(p)
    f = np.random.default_rng(0).standard_normal(A.ncols)
    lmax, lmin = power50(A)
    omega = R.chebyshev_weights(1.01 * lmax, lmin, 8)
    u, rep = R.solve_stationary(A, f, R.WeightSchedule(omega=omega), tol=1e-6)
    save("cfg1", eps=1e-2, theta=np.pi / 6, n=64, f=f, omega=omega, lmax50=lmax, lmin50=lmin,
         stencil=interior_row(A, 63), u=u, trace=rep.trace, iterations=rep.iterations,
         inner_iterations=rep.inner_iterations, converged=rep.converged)


def sweep_cases():
    """variants x Jacobi x check on small random anisotropic grids."""
    rng = np.random.default_rng(11)
    out = {}
    idx = 0
    for n in (16, 20):
        for variant in ("plain", "mom", "nag", "nagex"):
            for jac in (False, True):
                for check in ("outer", "inner"):
                    eps = float(10 ** rng.uniform(-3, 0))
                    th = float(rng.uniform(0, np.pi))
                    p = R.AnisotropicProblem(eps, th, n)
                    A = R.assemble_anisotropic(p)
                    f = rng.standard_normal(A.ncols)
                    P = R.Preconditioner.weighted_jacobi(A) if jac else None
                    Ad = A.to_dense()
                    if jac:
                        Ad = Ad * (P.apply(np.ones(A.ncols)))[:, None]
                    lam = np.linalg.eigvals(Ad).real
                    m = 4
                    if variant == "plain":
                        w = R.chebyshev_weights(lam.max() * 1.02, lam.min(), m)
                    else:  # stable heavy-ball / Nesterov range
                        w = np.array([0.9, 1.1, 0.7, 1.0]) / lam.max()
                    al = np.array([0.3, 0.5, 0.4, 0.6])
                    kw = {}
                    if variant != "plain":
                        kw["alpha"] = al
                    if variant == "nagex":
                        kw["alpha_tilde"] = np.array([0.5, 0.2, 0.7, 0.4])
                    s = R.WeightSchedule(omega=w, variant=variant, **kw)
                    for mode, tol, mo in (("conv", 1e-8, 400), ("fixed", 1e-300, 5)):
                        try:
                            u, rep = R.solve_stationary(A, f, s, P=P, tol=tol, max_outer=mo,
                                                        check=check)
                            res = dict(u=u, trace=rep.trace, iterations=rep.iterations,
                                       inner_iterations=rep.inner_iterations,
                                       converged=rep.converged,
                                       final=rep.final_relative_residual, diverged=-1)
                        except DivergenceError as e:
                            res = dict(u=np.zeros(0), trace=np.zeros(0), iterations=-1,
                                       inner_iterations=-1, converged=False, final=np.nan,
                                       diverged=e.inner_iteration)
                        key = f"c{idx}"
                        out.update({f"{key}_{k}": v for k, v in res.items()})
                        out.update({f"{key}_eps": eps, f"{key}_theta": th, f"{key}_n": n,
                                    f"{key}_variant": variant, f"{key}_jacobi": jac,
                                    f"{key}_check": check, f"{key}_tol": tol,
                                    f"{key}_max_outer": mo, f"{key}_f": f, f"{key}_omega": w,
                                    f"{key}_alpha": s.alpha, f"{key}_alpha_tilde": s.alpha_tilde})
                        idx += 1
    out["count"] = idx
    save("sweeps", **out)


def edge_cases():
    out = {}
    # divergence: far too large weight (test_richardson.py:191-197 analogue on a grid)
    p = R.AnisotropicProblem(0.3, 0.7, 12)
    A = R.assemble_anisotropic(p)
    f = np.random.default_rng(5).standard_normal(A.ncols)
    try:
        R.solve_stationary(A, f, R.WeightSchedule(omega=[50.0, 0.2]), max_outer=5000)
        raise SystemExit("expected divergence")
    except DivergenceError as e:
        out.update(div_f=f, div_inner=e.inner_iteration, div_msg=str(e))
    # NAG divergence is only detected at sweep ends
    try:
        R.solve_stationary(A, f, R.WeightSchedule(omega=[5.0, 0.1, 0.1], alpha=[0.1, 0.1, 0.1],
                                                  variant="nag"), max_outer=5000)
        raise SystemExit("expected divergence")
    except DivergenceError as e:
        out.update(divnag_inner=e.inner_iteration, divnag_msg=str(e))
    # zero right-hand side
    u, rep = R.solve_stationary(A, np.zeros(A.ncols), R.WeightSchedule(omega=[0.1]))
    out.update(zero_iterations=rep.iterations, zero_trace=rep.trace)
    # already converged initial guess
    ustar = np.random.default_rng(6).standard_normal(A.ncols)
    fb = A.matvec(ustar)
    u, rep = R.solve_stationary(A, fb, R.WeightSchedule(omega=[0.1]), u0=ustar, tol=1e-6)
    out.update(init_f=fb, init_u0=ustar, init_iterations=rep.iterations, init_trace=rep.trace,
               init_u=u)
    # max_outer = 0
    u, rep = R.solve_stationary(A, f, R.WeightSchedule(omega=[0.1]), max_outer=0)
    out.update(zero_outer_trace=rep.trace, zero_outer_conv=rep.converged)
    # 7-point stencil (dropped entries), eps=0.5 theta=0
    p7 = R.AnisotropicProblem(0.5, 0.0, 24)
    A7 = R.assemble_anisotropic(p7)
    f7 = np.random.default_rng(7).standard_normal(A7.ncols)
    lam7 = np.linalg.eigvalsh(A7.to_dense())
    w7 = R.chebyshev_weights(lam7[-1], lam7[0], 5)
    u, rep = R.solve_stationary(A7, f7, R.WeightSchedule(omega=w7), tol=1e-300, max_outer=9)
    out.update(s7_stencil=interior_row(A7, 23), s7_nnz=A7.nnz, s7_f=f7, s7_omega=w7, s7_u=u,
               s7_trace=rep.trace)
    # identity on a 2x2 grid (test_richardson.py:32-37 analogue)
    I4 = R.SparseMatrix.identity(4)
    st = R.IterationState.start(4)
    R.outer_sweep(I4, np.array([1.0, 2.0, 3.0, 4.0]), st, R.WeightSchedule(omega=[1.0]))
    out.update(id_u=st.u)
    # outer_sweep sequence with NAG, Jacobi
    pn = R.AnisotropicProblem(0.05, 1.1, 16)
    An = R.assemble_anisotropic(pn)
    fn = np.random.default_rng(8).standard_normal(An.ncols)
    Pn = R.Preconditioner.weighted_jacobi(An)
    sn = R.WeightSchedule(omega=[0.9, 1.3, 0.7], alpha=[0.2, 0.3, 0.1], variant="nag")
    st = R.IterationState.start(An.ncols)
    us, vs = [], []
    for _ in range(3):
        R.outer_sweep(An, fn, st, sn, Pn)
        us.append(st.u.copy())
        vs.append(st.v.copy())
    out.update(os_f=fn, os_u=np.stack(us), os_v=np.stack(vs),
               os_hist=np.array(st.residual_history))
    # outer_sweep non-finite detection (test_richardson.py:52-64 analogue)
    st = R.IterationState.start(4)
    sched = R.WeightSchedule(omega=[1e300, 1e300])
    try:
        for _ in range(60):
            R.outer_sweep(I4.scaled(1e4), np.ones(4), st, sched)
        raise SystemExit("expected divergence")
    except DivergenceError as e:
        out.update(osdiv_inner=e.inner_iteration, osdiv_msg=str(e))
    save("edge", **out)


def helmholtz():
    n = 32
    hp = R.HelmholtzProblem(2 * np.pi * n / 10, n)
    A = R.assemble_helmholtz(hp)
    rng = np.random.default_rng(9)
    x = rng.standard_normal(A.ncols) + 1j * rng.standard_normal(A.ncols)
    y = A.matvec(x)
    f = (rng.standard_normal(A.ncols)).astype(np.complex128)
    w = np.full(4, 0.8 / (8 * n * n))
    s = R.WeightSchedule(omega=w, alpha=np.full(4, 0.3), variant="nag")
    u, rep = R.solve_stationary(A, f, s, tol=1e-300, max_outer=6)
    save("helmholtz", n=n, omega_phys=hp.angular_frequency, x=x, y=y, diag=A.diagonal(), f=f,
         w=w, u=u, trace=rep.trace)


def fns_dst():
    rng = np.random.default_rng(10)
    x31 = rng.standard_normal(31 * 31)
    x63 = rng.standard_normal(63 * 63)
    n = 32
    p = R.AnisotropicProblem(1e-3, 0.4, n)
    A = R.assemble_anisotropic(p)
    f = rng.standard_normal(A.ncols)
    lam = 0.01 * rng.standard_normal(A.ncols)
    corr = RF.SpectralCorrection(lam, n)
    sch = R.WeightSchedule(omega=np.full(8, 0.5))
    u1 = RF.fns_lite_step(A, f, np.zeros(A.ncols), sch, 8, corr)
    u, rep = RF.solve_fns(A, f, sch, corr, 8, tol=1e-300, max_iters=5)
    # exact-inverse correction (test_fns.py:31-40 analogue): eps=1 stencil is diagonalised
    p1 = R.AnisotropicProblem(1.0, 0.0, 16)
    A1 = R.assemble_anisotropic(p1)
    lam1 = 1.0 / RF.sine_basis_eigenvalues(A1, 16)
    f1 = rng.standard_normal(A1.ncols)
    u_ex = RF.fns_lite_step(A1, f1, np.zeros(A1.ncols), R.WeightSchedule(omega=[0.0]), 0,
                            RF.SpectralCorrection(lam1, 16))
    save("fns", x31=x31, d31=R.dst2(x31), x63=x63, d63=R.dst2(x63), n=n, eps=1e-3, theta=0.4,
         f=f, lam=lam, u1=u1, u5=u, trace5=rep.trace, lam1=lam1, f1=f1, u_exact=u_ex)


def multigrid():
    n = 32
    hp = R.HelmholtzProblem(2 * np.pi * 3, n)  # 10.7 points per wavelength
    A = R.assemble_helmholtz(hp)
    s = R.WeightSchedule(omega=np.full(4, 0.8 / (8 * n * n)), alpha=np.full(4, 0.3),
                         variant="nag")
    H = RM.build_hierarchy(A, n, coarsest=8, schedules=s)
    rng = np.random.default_rng(12)
    f = rng.standard_normal(A.ncols) + 1j * rng.standard_normal(A.ncols)
    u = RM.v_cycle(H, f)
    r32 = rng.standard_normal(31 * 31)
    e16 = rng.standard_normal(15 * 15)
    out = dict(n=n, omega_phys=hp.angular_frequency, f=f, u=u, r32=r32,
               R32=RM.restrict(r32, 32), e16=e16, P16=RM.prolong(e16, 32), depth=H.depth)
    for k, lvl in enumerate(H.levels):
        out[f"A{k}_data"] = lvl.A.values
        out[f"A{k}_indices"] = lvl.A.col_indices
        out[f"A{k}_indptr"] = lvl.A.row_starts
    ug, rep = R.fgmres(A, f, precond_apply=lambda r: RM.v_cycle(H, r),
                       cfg=R.FgmresConfig(restart=5, tol=1e-6, max_outer=4))
    out.update(fg_u=ug, fg_trace=rep.trace, fg_iterations=rep.iterations,
               fg_converged=rep.converged, fg_stagnated=rep.stagnated)
    save("multigrid", **out)


def table2():
    """Criterion-1 style known answer (test_acceptance.py:42-66): Chebyshev
    m=3, N=64, theta=0, dense bounds, seed 0, two epsilons."""
    out = {}
    for k, eps in enumerate((1.0, 1e-2)):
        A = R.assemble_anisotropic(R.AnisotropicProblem(eps, 0.0, 64))
        b = R.dense_spectral_bounds(A)
        w = R.chebyshev_weights(b.lambda_max, b.lambda_min, 3)
        f = np.random.default_rng(0).standard_normal(A.ncols)
        _, rep = R.solve_stationary(A, f, R.WeightSchedule(omega=w))
        out.update({f"e{k}_eps": eps, f"e{k}_omega": w, f"e{k}_iterations": rep.iterations,
                    f"e{k}_inner": rep.inner_iterations, f"e{k}_final": rep.final_relative_residual})
    save("table2", **out)


def precond():
    """GS / SOR / SSOR maps (precond.py:79-118) and SSOR-preconditioned
    solves (the paper's NAGex + SSOR family) on small anisotropic grids."""
    rng = np.random.default_rng(21)
    out = {}
    for k, n in enumerate((2, 9, 33)):
        eps, th = float(10 ** rng.uniform(-3, 0)), float(rng.uniform(0, np.pi))
        A = R.assemble_anisotropic(R.AnisotropicProblem(eps, th, n))
        r = rng.standard_normal(A.ncols)
        out.update({f"a{k}_n": n, f"a{k}_eps": eps, f"a{k}_theta": th, f"a{k}_r": r})
        for name, P in (("gs", R.Preconditioner.gauss_seidel(A)),
                        ("sor14", R.Preconditioner.sor(A, 1.4)),
                        ("ssor10", R.Preconditioner.ssor(A, 1.0)),
                        ("ssor13", R.Preconditioner.ssor(A, 1.3))):
            out[f"a{k}_{name}"] = P.apply(r)
    cases = (("ssor", 1.0, "plain", 4, 1e-8), ("ssor", 1.2, "nagex", 3, 1e-8),
             ("gauss-seidel", 1.0, "mom", 2, 1e-8), ("sor", 1.5, "nag", 3, 1e-300),
             ("ssor", 1.0, "plain", 1, 1e-8))
    for k, (kind, relax, variant, m, tol) in enumerate(cases):
        n = 24
        eps, th = float(10 ** rng.uniform(-2, 0)), float(rng.uniform(0, np.pi))
        A = R.assemble_anisotropic(R.AnisotropicProblem(eps, th, n))
        f = rng.standard_normal(A.ncols)
        P = {"ssor": lambda: R.Preconditioner.ssor(A, relax),
             "sor": lambda: R.Preconditioner.sor(A, relax),
             "gauss-seidel": lambda: R.Preconditioner.gauss_seidel(A)}[kind]()
        BA = np.column_stack([P.apply(A.matvec(e)) for e in np.eye(A.ncols)])
        lam = np.linalg.eigvals(BA)
        lmax, lmin = float(lam.real.max()), float(lam.real.min())
        if variant == "plain":
            w = R.chebyshev_weights(lmax, lmin, m)
            if k == 4:
                w = np.array([4.0 / lmax])      # divergent on purpose
        else:
            w = np.linspace(0.8, 1.1, m) / lmax
        kw = {} if variant == "plain" else {"alpha": np.linspace(0.2, 0.5, m)}
        if variant == "nagex":
            kw["alpha_tilde"] = np.linspace(0.6, 0.3, m)
        sch = R.WeightSchedule(omega=w, variant=variant, **kw)
        try:
            u, rep = R.solve_stationary(A, f, sch, P=P, tol=tol, max_outer=60)
            res = dict(u=u, trace=rep.trace, iterations=rep.iterations,
                       inner=rep.inner_iterations, converged=rep.converged, diverged=-1)
        except DivergenceError as e:
            res = dict(u=np.zeros(0), trace=np.zeros(0), iterations=-1, inner=-1,
                       converged=False, diverged=e.inner_iteration)
        out.update({f"s{k}_{a}": b for a, b in res.items()})
        out.update({f"s{k}_kind": kind, f"s{k}_relax": relax, f"s{k}_variant": variant,
                    f"s{k}_n": n, f"s{k}_eps": eps, f"s{k}_theta": th, f"s{k}_f": f,
                    f"s{k}_omega": sch.omega, f"s{k}_alpha": sch.alpha,
                    f"s{k}_alpha_tilde": sch.alpha_tilde, f"s{k}_tol": tol})
    out["n_apply"] = 3
    out["n_solve"] = len(cases)
    save("precond", **out)


def unroll():
    """Training unroll (training.py:61-104): the tape-free loss and the tape
    gradients of _unroll_tape w.r.t. omega / alpha / alpha_t (separate Vars)."""
    from richlab import training as RT
    from richlab.tape import Tape
    rng = np.random.default_rng(31)
    out = {}
    cases = [("plain", None), ("mom", None), ("nag", None), ("nagex", None),
             ("plain", "jacobi"), ("nag", "jacobi"), ("mom", "jacobi"),
             ("nagex", "ssor"), ("plain", "gs"), ("mom", "ssor")]
    for k, (variant, pre) in enumerate(cases):
        n = int(rng.choice([12, 17]))
        eps, th = float(10 ** rng.uniform(-2, 0)), float(rng.uniform(0, np.pi))
        A = R.assemble_anisotropic(R.AnisotropicProblem(eps, th, n))
        f = rng.standard_normal(A.ncols)
        m, K = 3, 11
        P = {"jacobi": lambda: R.Preconditioner.weighted_jacobi(A),
             "ssor": lambda: R.Preconditioner.ssor(A, relax=1.0),       # training.py:52-53
             "gs": lambda: R.Preconditioner.gauss_seidel(A)}.get(pre, lambda: None)()
        lam = np.linalg.eigvalsh(A.to_dense()).max()
        scale = (2.0 / 3.0) / A.diagonal()[0] if pre == "jacobi" else 1.0
        if pre in ("ssor", "gs"):
            w = rng.uniform(0.3, 0.9, m)       # B^{-1} A has its spectrum in (0, 1]
        else:
            w = rng.uniform(0.3, 0.9, m) / (lam * scale)
        a = rng.uniform(0.1, 0.5, m)
        at = rng.uniform(0.1, 0.5, m) if variant == "nagex" else a.copy()
        tape = Tape()
        om = tape.var(w)
        al = tape.var(a) if variant != "plain" else None
        atv = tape.var(at)
        loss = RT._unroll_tape(A, f, om, al, atv, K, variant, P)
        tape.backward(loss)
        free = RT.unrolled_relative_residual(A, f, w, a if variant != "plain" else np.zeros(m),
                                             at, K, variant, P)
        out.update({f"u{k}_variant": variant, f"u{k}_pre": pre or "none", f"u{k}_n": n,
                    f"u{k}_eps": eps, f"u{k}_theta": th, f"u{k}_f": f, f"u{k}_K": K,
                    f"u{k}_omega": w, f"u{k}_alpha": a, f"u{k}_alpha_t": at,
                    f"u{k}_loss": float(loss.value), f"u{k}_loss_free": free,
                    f"u{k}_d_omega": om.grad,
                    f"u{k}_d_alpha": al.grad if al is not None else np.zeros(m),
                    f"u{k}_d_alpha_t": atv.grad if atv.grad is not None else np.zeros(m)})
    out["count"] = len(cases)
    save("unroll", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    cfg1()
    sweep_cases()
    edge_cases()
    helmholtz()
    fns_dst()
    multigrid()
    table2()
    precond()
    unroll()

"""Generate BASELINE-size goldens (tests/golden/full_*.npz) by running the
UNMODIFIED reference (richlab) on the full configs of SURVEY.md §8(d).

Run once, offline, in the dev container (the reference and these CPU hours
are not available on the GPU box):

    OPENBLAS_NUM_THREADS=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden_full.py [cfg2 cfg3 cfg4 cfg5]

The full-size vectors are far too large to commit, so each golden stores:

* the small inputs the GPU test cannot regenerate bit for bit on another
  machine (the schedules produced by the random-init PyTorch networks);
* a sha256 of every regenerated input (f, the cfg4 symbol), so a test can
  prove it fed the same bits;
* the reference's outputs: iteration counts, the full residual trace, and a
  digest of u -- sha256 of its bytes (for the bitwise paths), its 2-norm and
  sum, 1024 seeded sampled entries, and 4 projections onto seeded N(0,1)
  vectors (for the paths compared to a tolerance).

Reference calls (file:line in /root/reference/pkg/src/richlab):
  cfg2  solve_stationary(..., variant nag, tol=1e-300, max_outer=200)   richardson.py:77-141
  cfg3  solve_stationary(..., P=weighted_jacobi, tol=1e-6, max_outer=1e4) richardson.py:77-141
  cfg4  solve_fns(..., M=8, tol=1e-300, max_iters=100)                   fns.py:87-105
  cfg5  fgmres(H, f, v_cycle, FgmresConfig(20, 1e-6, 5))                 fgmres.py:31-131,
                                                                          multigrid.py:141-163
"""
from __future__ import annotations

import os
import sys
import time
from multiprocessing import get_context
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

REF = os.environ.get("RICHLAB_SRC", "/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, REF)
sys.path.insert(0, str(ROOT))
OUT = Path(__file__).resolve().parent

sys.path.insert(0, str(OUT))
from digest import digest, sha  # noqa: E402


def _pool(fn, jobs, procs):
    with get_context("fork").Pool(procs) as pool:
        return pool.map(fn, jobs)


# ----------------------------------------------------------------- cfg2
def _cfg2_job(b):
    import richlab as R
    from paper_2412_08076_b200 import configs
    c = configs.cfg2()
    p = c["problems"][b]
    A = R.assemble_anisotropic(R.AnisotropicProblem(p.epsilon, p.theta, p.n))
    s = c["schedules"][b]
    f = c["F"][b]
    t0 = time.perf_counter()
    u, rep = R.solve_stationary(A, f, R.WeightSchedule(omega=s.omega, alpha=s.alpha, variant="nag"),
                                tol=1e-300, max_outer=c["outer"])
    return dict(b=b, f_sha=sha(f), omega=s.omega, alpha=s.alpha, trace=rep.trace,
                iterations=rep.iterations, inner=rep.inner_iterations,
                wall=time.perf_counter() - t0, **digest(u, "u_"))


def cfg2(procs):
    res = _pool(_cfg2_job, list(range(64)), procs)
    out = {"count": len(res), "outer": 200}
    for r in res:
        b = r.pop("b")
        out.update({f"s{b}_{k}": v for k, v in r.items()})
    save("full_cfg2", **out)


# ----------------------------------------------------------------- cfg3
def _cfg3_job(b):
    import richlab as R
    from paper_2412_08076_b200 import configs
    c = configs.cfg3(first=b, count=1)
    p = c["problems"][0]
    A = R.assemble_anisotropic(R.AnisotropicProblem(p.epsilon, p.theta, p.n))
    P = R.Preconditioner.weighted_jacobi(A)
    scale = P.apply(np.ones(A.ncols))
    assert np.all(scale == c["scales"][0]), "Jacobi scale differs from the host recipe"
    s = c["schedules"][0]
    f = c["F"][0]
    t0 = time.perf_counter()
    u, rep = R.solve_stationary(A, f, R.WeightSchedule(omega=s.omega), P=P, tol=1e-6,
                                max_outer=10_000)
    wall = time.perf_counter() - t0
    print(f"cfg3 system {b}: {rep.iterations} outer / {rep.inner_iterations} inner, "
          f"converged={rep.converged}, {wall:.0f} s", flush=True)
    return dict(b=b, f_sha=sha(f), eps=p.epsilon, theta=p.theta, omega=s.omega,
                scale=c["scales"][0], trace=rep.trace, iterations=rep.iterations,
                inner=rep.inner_iterations, converged=rep.converged,
                final=rep.final_relative_residual, wall=wall, **digest(u, "u_"))


def cfg3(procs, systems=range(8)):
    res = _pool(_cfg3_job, list(systems), procs)
    out = {"count": len(res), "tol": 1e-6, "max_outer": 10_000}
    for r in res:
        b = r.pop("b")
        out.update({f"s{b}_{k}": v for k, v in r.items()})
    save("full_cfg3", **out)


# ----------------------------------------------------------------- cfg4
def _cfg4_job(b):
    import richlab as R
    from richlab import fns as RF
    from paper_2412_08076_b200 import configs
    c = configs.cfg4(device="cpu")
    p = c["problems"][b]
    A = R.assemble_anisotropic(R.AnisotropicProblem(p.epsilon, p.theta, p.n))
    lam = configs.fns_symbol_portable(p.theta, p.epsilon, p.n)
    f = c["F"][b]
    corr = RF.SpectralCorrection(lam, p.n)
    t0 = time.perf_counter()
    u, rep = RF.solve_fns(A, f, R.WeightSchedule(omega=np.full(8, 0.5)), corr, c["M"],
                          tol=1e-300, max_iters=c["alternations"])
    return dict(b=b, f_sha=sha(f), lam_sha=sha(lam), trace=rep.trace,
                iterations=rep.iterations, wall=time.perf_counter() - t0, **digest(u, "u_"))


def cfg4(procs):
    res = _pool(_cfg4_job, list(range(4)), procs)
    out = {"count": len(res), "alternations": 100, "M": 8}
    for r in res:
        b = r.pop("b")
        out.update({f"s{b}_{k}": v for k, v in r.items()})
    save("full_cfg4", **out)


# ----------------------------------------------------------------- cfg5
def _cfg5_job(b):
    import richlab as R
    from richlab import multigrid as RM
    from paper_2412_08076_b200 import configs
    c = configs.cfg5(device="cpu")
    hp = c["problem"]
    A = R.assemble_helmholtz(R.HelmholtzProblem(hp.angular_frequency, hp.n))
    s = c["schedule"]
    sched = R.WeightSchedule(omega=s.omega, alpha=s.alpha, variant="nag")
    H = RM.build_hierarchy(A, hp.n, coarsest=c["coarsest"], schedules=sched)
    f = c["F"][b]
    t0 = time.perf_counter()
    u, rep = R.fgmres(A, f, precond_apply=lambda r: RM.v_cycle(H, r),
                      cfg=R.FgmresConfig(restart=c["restart"], tol=1e-6, max_outer=c["max_outer"]))
    wall = time.perf_counter() - t0
    print(f"cfg5 rhs {b}: {rep.iterations} Arnoldi steps, converged={rep.converged}, "
          f"{wall:.0f} s", flush=True)
    return dict(b=b, f_sha=sha(f), omega=s.omega, alpha=s.alpha, depth=H.depth,
                trace=rep.trace, iterations=rep.iterations, converged=rep.converged,
                stagnated=rep.stagnated, wall=wall, **digest(u, "u_"))


def cfg5(procs):
    res = _pool(_cfg5_job, list(range(4)), procs)
    out = {"count": len(res), "restart": 20, "max_outer": 5, "coarsest": 16}
    for r in res:
        b = r.pop("b")
        out.update({f"s{b}_{k}": v for k, v in r.items()})
    save("full_cfg5", **out)


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz ({(OUT / f'{name}.npz').stat().st_size // 1024} KiB)", flush=True)


if __name__ == "__main__":
    procs = int(os.environ.get("GOLDEN_PROCS", len(os.sched_getaffinity(0))))
    names = sys.argv[1:] or ["cfg2", "cfg4", "cfg5", "cfg3"]
    for name in names:
        t = time.perf_counter()
        globals()[name](procs)
        print(f"{name}: {time.perf_counter() - t:.0f} s", flush=True)

"""Measure all five BASELINE.json configs on one B200.

For each config: GPU throughput / time on the full-size seeded inputs
(configs.py), a parity check against the CPU oracle on a bounded subset,
and the oracle's CPU time on a bounded sample (one process per system,
OPENBLAS_NUM_THREADS=1).  bench.py remains the headline (cfg3) line; this
script writes the per-config evidence (profiles/configs_rNN.json).

python profiles/configs_bench.py [--only 1,2,3,4,5] [--out profiles/configs_r01.json]
"""
from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import argparse  # noqa: E402
import json  # noqa: E402
import multiprocessing as mp  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402
from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import oracle as O  # noqa: E402  (checker + CPU baseline only)
import paper_2412_08076_b200 as G  # noqa: E402
from paper_2412_08076_b200 import configs as CF  # noqa: E402
import paper_2412_08076_b200.fgmres  # noqa: E402,F401  (the package attribute is the function)
GG = sys.modules["paper_2412_08076_b200.fgmres"]
from paper_2412_08076_b200 import fns as GF  # noqa: E402
from paper_2412_08076_b200 import multigrid as GM  # noqa: E402

HBM = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (
    ROOT / "MEASURED_PEAKS.json").exists() else 6650.0


def cuda_time(fn, reps=1):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _pool_map(fn, args, procs):
    with mp.get_context("fork").Pool(procs) as pool:
        return pool.map(fn, args)


# ------------------------------------------------------------------ cfg1
def run_cfg1():
    c = CF.cfg1()
    p, f, s = c["problem"], c["f"], c["schedule"]
    op = G.GpuStencilOperator.from_problems([p])
    G.solve_stationary(op, f, s, tol=1e-6)          # warm-up
    times = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        u, rep = G.solve_stationary(op, f, s, tol=1e-6)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    A = O.assemble_anisotropic(p.epsilon, p.theta, p.n)
    t0 = time.perf_counter()
    uo, ro = O.solve_stationary(A, f, s.omega, tol=1e-6)
    tcpu = time.perf_counter() - t0
    upd = rep.inner_iterations * 63 * 63
    return {"config": "cfg1 Richardson(8) 63^2 f64 to 1e-6", "gpu_time_to_tol_s": float(np.median(times)),
            "updates_per_s": upd / float(np.median(times)),
            "note": "latency-bound: 1520 dependent inner steps of a 3969-point system on one 16-CTA cluster (time through the API, H2D f and D2H u included)",
            "outer": rep.iterations, "inner": rep.inner_iterations,
            "cpu_time_to_tol_s": tcpu, "cpu_cores": 1,
            "parity": {"bitwise_u": bool(np.array_equal(u, uo)),
                       "same_counts": rep.iterations == ro["iterations"],
                       "trace_max_rel": float(np.max(np.abs(rep.trace - ro["trace"]) / ro["trace"]))}}


# ------------------------------------------------------------------ cfg2
def _cfg2_cpu(args):
    eps, theta, n, f, w, a, sweeps = args
    A = O.assemble_anisotropic(eps, theta, n)
    t0 = time.perf_counter()
    O.solve_stationary(A, f, w, a, variant="nag", tol=1e-300, max_outer=sweeps)
    return time.perf_counter() - t0


def _cfg2_ref(args):
    eps, theta, n, f, w, a, sweeps = args
    A = O.assemble_anisotropic(eps, theta, n)
    return O.solve_stationary(A, f, w, a, variant="nag", tol=1e-300, max_outer=sweeps)[0]


def run_cfg2():
    c = CF.cfg2()
    probs, F, sch, outer, m = c["problems"], c["F"], c["schedules"], c["outer"], c["m"]
    out = {"config": "cfg2 NAG(16) 64 x 255^2, 200 outer sweeps"}
    upd = len(probs) * 255 * 255 * outer * m
    for dt, name in ((np.float64, "f64"), (np.float32, "f32")):
        op = G.GpuStencilOperator.from_problems(probs, dtype=dt)
        S = G.StationarySolver(op, sch, None, tol=1e-300, max_outer=outer)

        def go():
            S.begin(F.astype(dt))
            S.run(first_batch=outer, max_batch=outer)
        go()
        t = cuda_time(go)
        res = S.results(like_numpy=True)
        out[name] = {"time_s": t, "updates_per_s": upd / t,
                     "hbm_frac_at_40B": (upd / t) * (40 if dt == np.float64 else 20) / (HBM * 1e9),
                     "note": "u, v, f of 64 x 255^2 = %d MB: L2-resident (126 MB L2); the fraction "
                             "counts algorithmic bytes against the HBM peak" %
                             (3 * 64 * 255 * 255 * (8 if dt == np.float64 else 4) // 2**20)}
        out[name]["_u"] = [res[b][0] for b in range(len(probs))]
    # parity over all 64 systems: oracle runs in parallel (f64 bitwise, f32 rel)
    procs = min(16, len(os.sched_getaffinity(0)))
    refs = _pool_map(_cfg2_ref, [(p.epsilon, p.theta, 256, F[b], sch[b].omega, sch[b].alpha, outer)
                                 for b, p in enumerate(probs)], procs)
    u64, u32 = out["f64"].pop("_u"), out["f32"].pop("_u")
    out["f64"]["parity_bitwise_all"] = bool(all(np.array_equal(a, r) for a, r in zip(u64, refs)))
    errs = np.array([rel(a, r) for a, r in zip(u32, refs)])
    out["f32"]["parity_rel_vs_f64_oracle"] = {"max": float(errs.max()), "median": float(np.median(errs)),
                                             "n_above_1e-5": int(np.sum(errs > 1e-5))}
    procs = min(16, len(os.sched_getaffinity(0)))
    sweeps = 10
    args = [(probs[b].epsilon, probs[b].theta, 256, F[b], sch[b].omega, sch[b].alpha, sweeps)
            for b in range(procs)]
    t0 = time.perf_counter()
    _pool_map(_cfg2_cpu, args, procs)
    wall = time.perf_counter() - t0
    out["cpu"] = {"updates_per_s": procs * 255 * 255 * sweeps * m / wall, "cores": procs,
                  "sample": f"{procs} systems x {sweeps} NAG sweeps (incl. assembly) in parallel"}
    return out


# ------------------------------------------------------------------ cfg4
def _cfg4_cpu(args):
    eps, theta, n, f, lam = args
    A = O.assemble_anisotropic(eps, theta, n)
    t0 = time.perf_counter()
    O.fns_lite_step(A, f, np.zeros(A.shape[0]), np.full(8, 0.5), 8, lam)
    return time.perf_counter() - t0


def run_cfg4():
    c = CF.cfg4()
    probs, F, lam, M, alts = c["problems"], c["F"], c["lam"], c["M"], c["alternations"]
    op = G.GpuStencilOperator.from_problems(probs)
    eng = GF.FnsEngine(op, c["schedule"], GF.SpectralCorrection(lam, 1024), M)
    Fd = op.to_device(F)

    def alternations(k):
        eng.u[0].zero_()
        eng.cur = 0
        for _ in range(k):
            u = eng.step(Fd)
            op.residual(u, Fd, want_r=False)          # rel per alternation (fns.py:99)
    alternations(2)
    t = cuda_time(lambda: alternations(alts))
    eng.u[0].zero_()
    eng.cur = 0
    u1 = eng.step(Fd).cpu().numpy()
    alg = 4 * 1023 ** 2 * (24 * M + 32 + 16) * alts        # smoothing + correction + norm
    out = {"config": "cfg4 FNS 4 x 1023^2, M=8 + DST correction, 100 alternations",
           "gpu_time_100_alternations_s": t, "gpu_ms_per_alternation": 1e3 * t / alts,
           "smoothing_updates_per_s": 4 * 1023 ** 2 * M * alts / t,
           "roofline": {"bound": "hbm", "algorithmic_bytes_per_alternation": alg / alts,
                        "achieved_GBs": alg / t / 1e9, "frac": alg / t / 1e9 / HBM}}
    A0 = O.assemble_anisotropic(probs[0].epsilon, probs[0].theta, 1024)
    lam0 = lam[0].cpu().numpy()
    uo = O.fns_lite_step(A0, F[0], np.zeros(A0.shape[0]), np.full(8, 0.5), 8, lam0)
    out["parity_rel_first_alternation"] = rel(u1[0], uo)
    procs = min(4, len(os.sched_getaffinity(0)))
    args = [(probs[b].epsilon, probs[b].theta, 1024, F[b], lam[b].cpu().numpy()) for b in range(procs)]
    tc = _pool_map(_cfg4_cpu, args, procs)
    out["cpu"] = {"s_per_alternation_per_system": float(np.mean(tc)), "cores": procs,
                  "sample": f"{procs} systems x 1 alternation in parallel"}
    return out


# ------------------------------------------------------------------ cfg5
def run_cfg5():
    c = CF.cfg5()
    hp, F, s = c["problem"], c["F"], c["schedule"]
    n = hp.n
    t0 = time.perf_counter()
    A = O.assemble_helmholtz(hp.angular_frequency, n)        # CSR only for host setup
    h = GM.build_hierarchy(A, n, coarsest=c["coarsest"], schedules=s, batch=len(F))
    t_setup = time.perf_counter() - t0
    op = G.GpuStencilOperator.from_problems([hp]).broadcast(len(F))
    Fd = op.to_device(F)
    h.apply(Fd)
    tv = cuda_time(lambda: h.apply(Fd), reps=3)
    cfg = GG.FgmresConfig(restart=c["restart"], tol=1e-6, max_outer=c["max_outer"])
    # warm-up (module loading, pool growth) with a 2-step FGMRES
    GG.fgmres_batched(op, Fd, precond_apply=lambda R: h.apply(R),
                      cfg=GG.FgmresConfig(restart=2, tol=1e-6, max_outer=1))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = GG.fgmres_batched(op, Fd, precond_apply=lambda R: h.apply(R), cfg=cfg)
    torch.cuda.synchronize()
    tf = time.perf_counter() - t0
    m = len(s.omega)
    alg = 0.0
    for k, lvl in enumerate(h.levels[:-1]):
        per = 96 if k == 0 else 80 + 144
        alg += len(F) * lvl.op.P * (2 * m * per + 64)    # pre+post smoothing + residual/transfers
    out = {"config": "cfg5 Helmholtz 4 x 1023^2 c128, V-cycle(NAG16, depth 7) in FGMRES(20) x5",
           "roofline_vcycle": {"bound": "hbm", "algorithmic_bytes": alg, "achieved_GBs": alg / tv / 1e9,
                               "frac": alg / tv / 1e9 / HBM},
           "depth": h.depth, "host_setup_s": t_setup, "gpu_ms_per_vcycle_batch4": 1e3 * tv,
           "fgmres_total_s": tf, "fgmres_iterations": [r.iterations for _, r in res],
           "fgmres_final_rel": [float(r.final_relative_residual) for _, r in res],
           "converged": [bool(r.converged) for _, r in res]}
    # parity: one V-cycle of system 0 vs the oracle (CPU ~2-3 s)
    levels, lu = O.build_hierarchy(A, n, coarsest=c["coarsest"])
    sd = dict(omega=s.omega, alpha=s.alpha, alpha_tilde=s.alpha_tilde, variant="nag")
    t0 = time.perf_counter()
    vo = O.v_cycle(levels, lu, F[0], sd)
    tcpu = time.perf_counter() - t0
    vg = h.apply(Fd)[0].cpu().numpy()
    out["parity_rel_vcycle"] = rel(vg, vo)
    out["cpu"] = {"s_per_vcycle_per_system": tcpu, "cores": 1}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="1,2,4,5")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    runs = {"1": run_cfg1, "2": run_cfg2, "4": run_cfg4, "5": run_cfg5}
    res = {"gpu": torch.cuda.get_device_name(0), "hbm_gbs": HBM}
    for k in a.only.split(","):
        t0 = time.perf_counter()
        res[f"cfg{k}"] = runs[k]()
        res[f"cfg{k}"]["script_wall_s"] = time.perf_counter() - t0
        print(json.dumps({f"cfg{k}": res[f"cfg{k}"]}), flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

"""Per-config lines of bench.py: every BASELINE.json config at full size.

bench.py's headline is cfg3; this module measures the other configs (and the
north-star NAG(16) sweep at 8 x 1023^2) in the same run so that each one
carries, from the driver's own box:

  value / unit    device-timed throughput (or time) with inputs resident
  roofline        algorithmic bytes per unit / time vs the
                  measured HBM peak
  e2e             the same metric through the public API with host (pinned
                  where the API takes tensors) buffers, H2D and D2H inside
  cpu_baseline    the oracle port (the reference's algorithm with the same
                  SciPy/NumPy calls) on a bounded sample on this box's cores
  parity          an in-run oracle check on a bounded subset (the full-length
                  comparisons are the -m gpu tests against tests/golden/full_*)

The oracle is imported here only as the checker and the CPU baseline.
Workloads come from paper_2412_08076_b200/configs.py.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np


def _hbm_peak(root):
    import json
    p = root / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


def _cuda_time(fn, reps=1):
    import torch
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def _wall(fn):
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0, out


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb else float(np.linalg.norm(a - b))


def _pool(fn, args, procs):
    with mp.get_context("fork").Pool(procs) as pool:
        return pool.map(fn, args)


def _cores(cap=32):
    return min(cap, len(os.sched_getaffinity(0)))


def _roof(bytes_, seconds, peak, src, per_unit, note=""):
    gbs = bytes_ / seconds / 1e9
    d = {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
         "peak_source": src, "bytes_per_unit": per_unit}
    if note:
        d["note"] = note
    return d


# ----------------------------------------------------------------- cfg1
def cfg1(ctx):
    import torch
    import oracle as O
    import paper_2412_08076_b200 as G
    from paper_2412_08076_b200 import configs as CF
    c = CF.cfg1()
    p, f, s = c["problem"], c["f"], c["schedule"]
    op = G.GpuStencilOperator.from_problems([p])
    fd = op.to_device(f)
    G.solve_stationary(op, fd, s, tol=1e-6)              # warm-up (solver cache, graph)
    dev_t = []
    for _ in range(5):
        dev_t.append(_cuda_time(lambda: G.solve_stationary(op, fd, s, tol=1e-6)))
    e2e_t = []
    for _ in range(5):
        t, (u, rep) = _wall(lambda: G.solve_stationary(op, f, s, tol=1e-6))
        e2e_t.append(t)
    A = O.assemble_anisotropic(p.epsilon, p.theta, p.n)
    t0 = time.perf_counter()
    uo, ro = O.solve_stationary(A, f, s.omega, tol=1e-6)
    tcpu = time.perf_counter() - t0
    P = (p.n - 1) ** 2
    tdev, te2e = float(np.median(dev_t)), float(np.median(e2e_t))
    return {"workload": "cfg1: Richardson(8), 63^2, f64, to ||r||/||f|| < 1e-6",
            "metric": "time to 1e-6", "value": tdev, "unit": "s", "higher_is_better": False,
            "updates_per_s": rep.inner_iterations * P / tdev,
            "roofline": {"bound": "latency", "note": "3969-point system: 1520 dependent inner "
                         "steps on one 16-CTA cluster, state resident in distributed shared "
                         "memory (0 HBM bytes per step); ~%.2f us per inner step" %
                         (1e6 * tdev / rep.inner_iterations)},
            "e2e": {"value": te2e, "unit": "s", "h2d_bytes_per_step": int(f.nbytes),
                    "d2h_bytes_per_step": int(f.nbytes),
                    "api": "solve_stationary(op, f_numpy, schedule, tol=1e-6)"},
            "cpu_baseline": {"value": tcpu, "unit": "s", "cores": 1, "kind": "port",
                             "sample": "the whole cfg1 solve to 1e-6 (oracle port)"},
            "counts": {"outer": rep.iterations, "inner": rep.inner_iterations},
            "parity": {"bitwise_u": bool(np.array_equal(u, uo)),
                       "same_counts": bool(rep.iterations == ro["iterations"] and
                                           rep.inner_iterations == ro["inner_iterations"]),
                       "trace_max_rel": float(np.max(np.abs(rep.trace - ro["trace"]) / ro["trace"]))}}


# ----------------------------------------------------------------- cfg2
def _cfg2_cpu(args):
    import oracle as O
    eps, theta, n, f, w, a, sweeps = args
    A = O.assemble_anisotropic(eps, theta, n)
    t0 = time.perf_counter()
    u, _ = O.solve_stationary(A, f, w, a, variant="nag", tol=1e-300, max_outer=sweeps)
    return time.perf_counter() - t0, u


def cfg2(ctx):
    import torch
    import paper_2412_08076_b200 as G
    from paper_2412_08076_b200 import configs as CF
    c = CF.cfg2()
    probs, F, sch, outer, m = c["problems"], c["F"], c["schedules"], c["outer"], c["m"]
    B, P = len(probs), 255 * 255
    upd = B * P * outer * m
    peak, src = ctx["peak"]
    # oracle: full 200 sweeps of the first `npar` systems (parity) -- in parallel
    npar = min(4, _cores())
    ref = _pool(_cfg2_cpu, [(probs[b].epsilon, probs[b].theta, 256, F[b], sch[b].omega,
                             sch[b].alpha, outer) for b in range(npar)], npar)
    out = {}
    for dt, name, bpu in ((np.float64, "cfg2_f64", 40), (np.float32, "cfg2_f32", 20)):
        op = G.GpuStencilOperator.from_problems(probs, dtype=dt)
        Fd = torch.as_tensor(F.astype(dt)).to(op.device)
        S = G.StationarySolver(op, sch, None, tol=1e-300, max_outer=outer)

        def go():
            S.begin(Fd)
            S.run(first_batch=outer, max_batch=outer)
        go()
        t = _cuda_time(go)
        res = S.results(like_numpy=True)
        Fh = torch.from_numpy(F.astype(dt)).pin_memory()
        Uh = torch.empty_like(Fh).pin_memory()
        G.solve_stationary_batched(op, Fh, sch, None, tol=1e-300, max_outer=outer, out=Uh)
        te, _ = _wall(lambda: G.solve_stationary_batched(op, Fh, sch, None, tol=1e-300,
                                                         max_outer=outer, out=Uh))
        mb = 3 * B * P * np.dtype(dt).itemsize / 2**20
        par = {}
        if dt == np.float64:
            par["bitwise_u_systems"] = [bool(np.array_equal(res[b][0], ref[b][1]))
                                        for b in range(npar)]
        else:
            par["max_rel_vs_f64_oracle"] = max(_rel(res[b][0], ref[b][1]) for b in range(npar))
            par["bar"] = 1e-5
        par["subset"] = f"systems 0..{npar - 1}, all {outer} sweeps, oracle in-run"
        out[name] = {
            "workload": f"cfg2: NAG(16), 64 x 255^2, {outer} outer sweeps, "
                        f"{'f64' if dt == np.float64 else 'f32 vectors / f64 arithmetic'}",
            "metric": "grid-point updates/s", "value": upd / t, "unit": "grid-point updates/s",
            "higher_is_better": True,
            "roofline": _roof(upd * bpu, t, peak, src, f"{bpu} B/update",
                              f"u, v, f = {mb:.0f} MB: L2-resident (126 MB L2); algorithmic "
                              "bytes against the HBM peak"),
            "e2e": {"value": upd / te, "unit": "grid-point updates/s",
                    "h2d_bytes_per_step": int(Fh.numel() * Fh.element_size()),
                    "d2h_bytes_per_step": int(Uh.numel() * Uh.element_size()),
                    "api": "solve_stationary_batched(op, F_pinned, schedules, tol=1e-300, "
                           "max_outer=200, out=U_pinned)"},
            "parity": par}
    # CPU: cores x 10 sweeps of distinct systems
    procs = _cores(16)
    sweeps = 10
    t0 = time.perf_counter()
    times = _pool(_cfg2_cpu, [(probs[b % B].epsilon, probs[b % B].theta, 256, F[b % B],
                               sch[b % B].omega, sch[b % B].alpha, sweeps) for b in range(procs)],
                  procs)
    per_core = np.mean([P * sweeps * m / tt for tt, _ in times])
    cpu = {"value": procs * per_core, "unit": "grid-point updates/s", "cores": procs,
           "kind": "port", "sample": f"{procs} processes x 1 system x {sweeps} NAG(16) sweeps"}
    out["cfg2_f64"]["cpu_baseline"] = cpu
    out["cfg2_f32"]["cpu_baseline"] = dict(cpu, note="the reference is float64 only")
    return out


# ----------------------------------------------------------------- cfg3 (CPU time to tol)
def cfg3_cpu_time_to_tol(cpu_line, inner_iterations, P):
    """Extrapolated CPU time for the cfg3 batch to 1e-6: the measured per-core
    oracle rate x the inner iterations the systems actually need, one
    process per system (so the batch takes as long as its slowest system)."""
    if not cpu_line or not inner_iterations:
        return None
    per_core = cpu_line["value"] / cpu_line["cores"]
    per_sys = [k * P / per_core for k in inner_iterations]
    return {"value": float(max(per_sys)), "unit": "s", "extrapolated": True,
            "per_system_s": [float(x) for x in per_sys], "cores": len(per_sys),
            "from": "cpu_baseline per-core updates/s x actual inner_iterations per system "
                    "(one process per system)"}


def cfg3_dropin(ctx, wl, n_side, tol, max_outer):
    """cfg3 through the reference-signature call a migrating richlab user
    makes: solve_stationary(A_csr, f_numpy, schedule, P, tol) per system, the
    matrices assembled once outside the timing (the memoised CSR -> stencil
    extraction is paid on the first, untimed pass)."""
    import torch
    import oracle as O
    import paper_2412_08076_b200 as G
    As = [O.assemble_anisotropic(p.epsilon, p.theta, n_side) for p in wl["problems"]]
    Ps = [G.JacobiScale(np.float64(s)) for s in wl["scales"]]
    F = wl["F"]

    def run():
        reps = []
        for A, f, s, Pb in zip(As, F, wl["schedules"], Ps):
            u, rep = G.solve_stationary(A, f, s, P=Pb, tol=tol, max_outer=max_outer)
            reps.append(rep)
        return reps
    t_first, _ = _wall(run)
    t, reps = _wall(run)
    P = (n_side - 1) ** 2
    upd = sum(r.inner_iterations for r in reps) * P
    device = sum(r.wall_time for r in reps)
    return {"value": upd / t, "unit": "grid-point updates/s", "seconds": t,
            "first_call_seconds": t_first,
            "h2d_bytes_per_step": int(F.nbytes), "d2h_bytes_per_step": int(F.nbytes),
            "api": "for each system: solve_stationary(A_scipy_csr, f_numpy, schedule, "
                   "P=JacobiScale, tol=1e-6, max_outer=10000) (richardson.py:77 signature)",
            "host_overhead_per_call_s": max(0.0, (t - device) / len(reps)),
            "inner_iterations": [int(r.inner_iterations) for r in reps]}


# ----------------------------------------------------------------- NAG(16) north-star sweep
def _nag_cpu(args):
    import oracle as O
    eps, theta, n, f, w, a = args
    A = O.assemble_anisotropic(eps, theta, n)
    t0 = time.perf_counter()
    u, v, _ = O.outer_sweep(A, f, np.zeros_like(f), np.zeros_like(f), w, a, variant="nag")
    return time.perf_counter() - t0, u


def nag16_sweep(ctx):
    import torch
    import paper_2412_08076_b200 as G
    from paper_2412_08076_b200 import configs as CF
    c = CF.nag_sweep()
    probs, F, sch, m = c["problems"], c["F"], c["schedules"], c["m"]
    B, P = len(probs), (probs[0].n - 1) ** 2
    peak, src = ctx["peak"]
    op = G.GpuStencilOperator.from_problems(probs)
    Fd = op.to_device(F)
    S = G.StationarySolver(op, sch, None, tol=1e-300, max_outer=10**7)
    S.begin(Fd)
    S.run_sweeps(3)
    sweeps = 20
    t = _cuda_time(lambda: S.run_sweeps(sweeps))
    upd = B * P * m * sweeps
    # e2e: one sweep-limited solve through the API with pinned host buffers
    Fh = torch.from_numpy(F).pin_memory()
    Uh = torch.empty_like(Fh).pin_memory()
    G.solve_stationary_batched(op, Fh, sch, None, tol=1e-300, max_outer=sweeps, out=Uh)
    te, res = _wall(lambda: G.solve_stationary_batched(op, Fh, sch, None, tol=1e-300,
                                                       max_outer=sweeps, out=Uh))
    # parity: system 0, one sweep from zero, vs the oracle's outer_sweep
    S1 = G.StationarySolver(op, sch, None, tol=1e-300, max_outer=1)
    S1.begin(Fd)
    S1.run()
    u1 = S1.results(like_numpy=True)
    npar = 1
    tc, uo = _nag_cpu((probs[0].epsilon, probs[0].theta, probs[0].n, F[0], sch[0].omega,
                       sch[0].alpha))
    procs = _cores(16)
    times = _pool(_nag_cpu, [(probs[b % B].epsilon, probs[b % B].theta, probs[b % B].n,
                              F[b % B], sch[b % B].omega, sch[b % B].alpha)
                             for b in range(procs)], procs)
    per_core = np.mean([P * m / tt for tt, _ in times])
    return {"workload": "north-star NAG(16) sweeps: 8 anisotropic systems on 1023^2 (cfg3's "
                        "systems), f64, weights from cfg2's random-init MLP",
            "metric": "grid-point updates/s", "value": upd / t, "unit": "grid-point updates/s",
            "higher_is_better": True,
            "roofline": _roof(upd * 40, t, peak, src, "40 B/update (u, v r/w; f r)",
                              "temporal blocking: frac may exceed 1 (SURVEY.md §8(d))"),
            "e2e": {"value": upd / te, "unit": "grid-point updates/s",
                    "h2d_bytes_per_step": int(F.nbytes), "d2h_bytes_per_step": int(F.nbytes),
                    "api": f"solve_stationary_batched(op, F_pinned, schedules, tol=1e-300, "
                           f"max_outer={sweeps}, out=U_pinned)"},
            "cpu_baseline": {"value": procs * per_core, "unit": "grid-point updates/s",
                             "cores": procs, "kind": "port",
                             "sample": f"{procs} processes x 1 system (1023^2) x 1 NAG(16) sweep"},
            "parity": {"bitwise_u_system0_one_sweep": bool(np.array_equal(u1[0][0], uo)),
                       "subset": f"{npar} system, 1 sweep (16 inner) from zero"}}


# ----------------------------------------------------------------- cfg4
def _cfg4_cpu(args):
    import oracle as O
    eps, theta, n, f, lam = args
    A = O.assemble_anisotropic(eps, theta, n)
    t0 = time.perf_counter()
    u = O.fns_lite_step(A, f, np.zeros(A.shape[0]), np.full(8, 0.5), 8, lam)
    return time.perf_counter() - t0, u


def cfg4(ctx):
    import torch
    import paper_2412_08076_b200 as G
    from paper_2412_08076_b200 import configs as CF
    from paper_2412_08076_b200 import fns as GF
    c = CF.cfg4()
    probs, F, lam, M, alts = c["problems"], c["F"], c["lam"], c["M"], c["alternations"]
    B, P = len(probs), 1023 ** 2
    peak, src = ctx["peak"]
    op = G.GpuStencilOperator.from_problems(probs)
    eng = GF.FnsEngine(op, c["schedule"], GF.SpectralCorrection(lam, 1024), M)
    Fd = op.to_device(F)

    def alternations(k):
        eng.u[0].zero_()
        eng.cur = 0
        for i in range(k):
            # rel per alternation (fns.py:99): the residual norm of alternation i
            # rides on alternation i + 1's first sweep, the last one is a pass of its own
            eng.step(Fd, want_norm=i >= 1)
        eng.residual_norm2(Fd)
    alternations(2)
    t = _cuda_time(lambda: alternations(alts))
    per_alt = t / alts
    alg = B * P * (24 * M + 32)            # smoothing (with the fused residual norm) + correction
    # e2e: the reference signature per system, numpy in / out
    corr_all = GF.SpectralCorrection(lam, 1024)
    Fp = torch.from_numpy(np.ascontiguousarray(F)).pin_memory()
    GF.solve_fns_batched(op, Fp, c["schedule"], corr_all, M, tol=1e-300, max_iters=2)
    te, res = _wall(lambda: GF.solve_fns_batched(op, Fp, c["schedule"], corr_all, M, tol=1e-300,
                                                 max_iters=alts))
    # parity: first alternation of system 0
    eng.u[0].zero_()
    eng.cur = 0
    u1 = eng.step(Fd)[0].cpu().numpy()
    procs = min(B, _cores())
    out = _pool(_cfg4_cpu, [(probs[b].epsilon, probs[b].theta, 1024, F[b], lam[b].cpu().numpy())
                            for b in range(procs)], procs)
    tcpu = float(np.mean([x[0] for x in out]))
    return {"workload": "cfg4: FNS, 4 x 1023^2, eps=1e-3, M=8 smoothing steps + DST-I "
                        "correction per alternation, f64",
            "metric": "time per alternation (4 systems)", "value": per_alt, "unit": "s",
            "higher_is_better": False,
            "hundred_alternations_s": t,
            "roofline": _roof(alg, per_alt, peak, src,
                              f"{24 * M + 32} B/point/alternation (8 x 24 B smoothing, the "
                              "residual norm fused into its first step, + 32 B correction)"),
            "e2e": {"value": te / alts, "unit": "s", "seconds_total": te,
                    "h2d_bytes_per_step": int(F.nbytes) // alts,
                    "d2h_bytes_per_step": int(F.nbytes) // alts,
                    "api": "solve_fns_batched(op, F_pinned_host, schedule, corr, 8, tol=1e-300, "
                           "max_iters=100) -> numpy; value = total / 100 (one residual-norm "
                           "read per alternation, as fns.py:99)",
                    "note": "per-step bytes are the per-solve H2D/D2H amortised over 100 steps"},
            "cpu_baseline": {"value": tcpu, "unit": "s", "cores": procs, "kind": "port",
                             "sample": f"{procs} systems x 1 alternation in parallel "
                                       "(one process per system)"},
            "parity": {"rel_first_alternation_system0": _rel(u1, out[0][1]), "bar": 1e-12}}


# ----------------------------------------------------------------- cfg5
def cfg5(ctx):
    import torch
    import oracle as O
    import paper_2412_08076_b200 as G
    from paper_2412_08076_b200 import configs as CF
    import importlib
    GG = importlib.import_module("paper_2412_08076_b200.fgmres")
    from paper_2412_08076_b200 import multigrid as GM
    c = CF.cfg5()
    hp, F, s = c["problem"], c["F"], c["schedule"]
    n = hp.n
    B = len(F)
    peak, src = ctx["peak"]
    A = O.assemble_helmholtz(hp.angular_frequency, n)
    h = GM.build_hierarchy(A, n, coarsest=c["coarsest"], schedules=s, batch=B)
    op = G.GpuStencilOperator.from_problems([hp]).broadcast(B)
    Fd = op.to_device(F)
    h.apply(Fd)
    tv = _cuda_time(lambda: h.apply(Fd), reps=5)
    cfg = GG.FgmresConfig(restart=c["restart"], tol=1e-6, max_outer=c["max_outer"])
    # warm-up at full size: the Krylov bases (2 x 1.4 GB) come from the caching
    # allocator afterwards, not from cudaMalloc inside the timed call
    GG.fgmres_batched(op, Fd, precond_apply=h.apply, cfg=cfg)
    tf, res = _wall(lambda: GG.fgmres_batched(op, Fd, precond_apply=h.apply, cfg=cfg))
    Fh = torch.from_numpy(F).pin_memory()
    GG.fgmres_batched(op, Fh, precond_apply=h.apply, cfg=cfg)     # host-buffer path warm (allocator)
    te, res_e = _wall(lambda: GG.fgmres_batched(op, Fh, precond_apply=h.apply, cfg=cfg))
    steps = max(r.iterations for _, r in res)
    m = len(s.omega)
    alg = 0.0
    for k, lvl in enumerate(h.levels[:-1]):
        per = 96 if k == 0 else 80 + 144
        alg += B * lvl.op.P * (2 * m * per + 64)    # pre+post smoothing + residual/transfers
    levels, lu = O.build_hierarchy(A, n, coarsest=c["coarsest"])
    sd = dict(omega=s.omega, alpha=s.alpha, alpha_tilde=s.alpha_tilde, variant="nag")
    t0 = time.perf_counter()
    vo = O.v_cycle(levels, lu, F[0], sd)
    tcpu = time.perf_counter() - t0
    vg = h.apply(Fd)[0].cpu().numpy()
    return {"workload": "cfg5: Helmholtz 4 x 1023^2 c128 (kh = 2 pi/10, sponge), V-cycle "
                        "(NAG(16) smoother, depth 7) as the preconditioner of FGMRES(20) x 5",
            "metric": "time per V-cycle (4 right-hand sides)", "value": tv, "unit": "s",
            "higher_is_better": False,
            "fgmres": {"seconds": tf, "arnoldi_steps": [int(r.iterations) for _, r in res],
                       "final_rel": [float(r.final_relative_residual) for _, r in res],
                       "overhead_vs_vcycles": tf / (steps * tv)},
            "roofline": _roof(alg, tv, peak, src,
                              "96 B/update fine level (c128 NAG + per-node diagonal), 224 B/update "
                              "Galerkin levels, + 64 B/point residual and transfers",
                              "temporal blocking on levels 0-2: frac may exceed 1"),
            "e2e": {"value": te, "unit": "s (FGMRES(20) x 5, 4 right-hand sides)",
                    "h2d_bytes_per_step": int(F.nbytes), "d2h_bytes_per_step": int(F.nbytes),
                    "api": "fgmres_batched(op, F_pinned_host, precond_apply=hierarchy.apply, "
                           "FgmresConfig(20, 1e-6, 5)) -> numpy"},
            "cpu_baseline": {"value": tcpu, "unit": "s per V-cycle per right-hand side",
                             "cores": 1, "kind": "port",
                             "sample": "1 V-cycle of right-hand side 0 (oracle port); 100 "
                                       "applications x 4 right-hand sides extrapolate linearly",
                             "extrapolated_fgmres_s": tcpu * 100 * B},
            "parity": {"rel_vcycle_rhs0": _rel(vg, vo), "bar": 1e-12}}


def precond_ssor(ctx):
    """GS/SOR/SSOR application on cfg3's 8 x 1023^2
    systems: the cluster wavefront of csrc/tri.cuh."""
    import torch
    import oracle as O
    import paper_2412_08076_b200 as G
    from paper_2412_08076_b200 import configs as CF
    c = CF.cfg3(first=0, count=8, n=1024, m=32)
    op = G.GpuStencilOperator.from_problems(c["problems"])
    B, P, side = op.batch, op.P, op.side
    R = torch.randn(B, P, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    Z, W = torch.empty_like(R), torch.empty_like(R)
    out = {}
    for kind, relax, sweeps in (("sor", 1.5, 1), ("ssor", 1.0, 2)):
        pre = G.TriangularPreconditioner(op, kind, relax)
        pre.apply_device(R, Z, W)
        t = _cuda_time(lambda: pre.apply_device(R, Z, W), reps=10)
        out[kind] = {"seconds": t, "ns_per_dependent_step": t * 1e9 / (sweeps * (3 * side - 2)),
                     "point_solves_per_s": sweeps * B * P / t}
    Rh = R.cpu().numpy()
    Rp = torch.from_numpy(Rh).pin_memory()
    pre = G.TriangularPreconditioner(op, "ssor", 1.0)
    te, Zh = _wall(lambda: pre.apply(Rp))
    A0 = O.assemble_anisotropic(c["problems"][0].epsilon, c["problems"][0].theta, 1024)
    f = O.tri_precond(A0, "ssor", 1.0)
    f(Rh[0])
    t0 = time.perf_counter()
    zo = f(Rh[0])
    tcpu = time.perf_counter() - t0
    z0 = Zh[0] if not isinstance(Zh, torch.Tensor) else Zh[0].cpu().numpy()
    return {"workload": "SSOR application z = B^{-1} r, 8 x 1023^2 (cfg3's systems), f64",
            "metric": "time per application (8 systems)", "value": out["ssor"]["seconds"], "unit": "s",
            "higher_is_better": False, "sor": out["sor"], "ssor": out["ssor"],
            "roofline": {"bound": "latency",
                         "note": "lexicographic substitution: 3 side - 2 = 3067 dependent steps per sweep "
                                 "(slope-2 wavefront); a bare shuffle + select + 2 DFMA step measures 41 "
                                 "cycles = 21 ns (profiles/micro/fp64_chain.cu)"},
            "e2e": {"value": te, "unit": "s", "h2d_bytes_per_step": int(Rh.nbytes),
                    "d2h_bytes_per_step": int(Rh.nbytes),
                    "api": "TriangularPreconditioner(op, 'ssor', 1.0).apply(r_pinned_host) -> numpy"},
            "cpu_baseline": {"value": tcpu, "unit": "s per application per system", "cores": 1,
                             "kind": "port",
                             "sample": "1 SSOR application of system 0 (SuperLU triangular solves, "
                                       "factorisation outside the timing)"},
            "parity": {"rel_system0": _rel(z0, zo), "bar": 1e-13}}


RUNNERS = {"cfg1": cfg1, "cfg2": cfg2, "nag16_sweep": nag16_sweep, "cfg4": cfg4, "cfg5": cfg5,
           "precond_ssor": precond_ssor}


def run_all(root, only=None):
    """{name: line} for every config (errors are reported per config, the
    bench line itself still prints)."""
    ctx = {"peak": _hbm_peak(root)}
    out = {}
    for name, fn in RUNNERS.items():
        if only and name not in only:
            continue
        t0 = time.perf_counter()
        try:
            r = fn(ctx)
        except Exception as exc:  # noqa: BLE001
            r = {"error": f"{type(exc).__name__}: {exc}"}
        wall = time.perf_counter() - t0
        if "workload" in r or "error" in r:
            r["wall_s"] = wall
            out[name] = r
        else:
            for k, v in r.items():
                v["wall_s"] = wall
                out[k] = v
    return out

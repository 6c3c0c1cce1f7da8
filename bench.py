"""Benchmark: batched Jacobi-Richardson(32) sweeps on 1023^2 anisotropic grids.

Workload (BASELINE.json configs[2], the north-star "batched N=1023
Richardson(m) stencil sweeps"; SURVEY.md §8(d) cfg 3; recipe in
paper_2412_08076_b200/configs.py:cfg3): 8 independent anisotropic systems per
GPU on 1024x1024 cells (1023^2 unknowns, f64), theta ~ U[0, pi],
lg eps ~ U[-4, 0], f ~ N(0,1) (rng = default_rng(3)), weighted Jacobi
(relax 2/3), m = 32 Chebyshev weights of the Jacobi-scaled operator in Leja
order.  Synthetic seeded inputs: the reference has no dataset.

One step = one outer sweep (32 inner updates) over all systems of a GPU.
  value     grid-point updates/s, whole job (all ranks), iterates resident in HBM
  e2e       same metric through the public API: one e2e step is a full
            solve_stationary_batched(..., tol=1e-6) with pinned host f in and
            u out (H2D/D2H inside the timing); updates = sum of inner_iterations
  roofline  dominant kernel (temporally blocked sweep): algorithmic bytes per
            launch (24 B per point-update) / CUDA-event time
  time_to_tol  wall time of that API solve (all 8 systems to ||r||/||f|| < 1e-6)
  cpu_time_to_tol  the CPU oracle's time for the same batch to 1e-6, extrapolated
            from its measured per-core rate x the actual inner iterations
  e2e_dropin  cfg3 through the reference signature solve_stationary(A_csr,
            f_numpy, ...) per system (what a migrating richlab user calls)
  configs   one line per other BASELINE config (cfg1, cfg2 f64/f32, cfg4, cfg5)
            and the north-star NAG(16) sweep at 8 x 1023^2: value, roofline,
            e2e, cpu_baseline and an in-run oracle parity check each
            (bench_configs.py); rank 0 at N=1 only

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import argparse  # noqa: E402
import json  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402
from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "grid-point updates/s + time-to-1e-6 residual (1 B200, % HBM roofline) vs CPU ref"
UNIT = "grid-point updates/s"
N_SIDE = 1024            # cells per side -> 1023^2 unknowns
SYSTEMS_PER_GPU = 8
M = 32
BYTES_PER_UPDATE = 24    # plain Richardson f64: read u, f; write u
FP64_PER_POINT_STEP = 22  # blocked kernel SASS: 11 DMUL + 10 DADD + 1 DFMA per point-step
TOL = 1e-6
MAX_OUTER_TOL = 10_000


# ------------------------------------------------------------------ inputs
def workload(rank):
    """cfg3 systems rank*8 .. rank*8+7 of the seeded stream (configs.cfg3)."""
    from paper_2412_08076_b200 import configs
    return configs.cfg3(first=rank * SYSTEMS_PER_GPU, count=SYSTEMS_PER_GPU, n=N_SIDE, m=M)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except (ValueError, IndexError):
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() in ("active", "1"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU side
def _cpu_worker_init(eps, theta, n, seed_f, w):
    global _W
    import oracle as O
    A = O.assemble_anisotropic(eps, theta, n)
    f = np.random.default_rng(seed_f).standard_normal(A.shape[0])
    u = np.zeros(A.shape[0])
    _W = dict(A=A, f=f, u=u, v=np.zeros_like(u), r=f - A.dot(u), scale=O.jacobi_scale(A), w=w,
              i=0)


def _cpu_worker_steps(k):
    """k inner steps of Jacobi Richardson on this worker's system (the
    oracle's restatement of richardson.py:111-125, same SciPy/NumPy calls,
    including the reference's a*v term with a = 0 for the plain variant)."""
    A, f, sc, w = _W["A"], _W["f"], _W["scale"], _W["w"]
    u, v, r, i0 = _W["u"], _W["v"], _W["r"], _W["i"]
    t0 = time.perf_counter()
    for i in range(i0, i0 + k):
        v = 0.0 * v + w[i % M] * (sc * r)
        u = u + v
        r = f - A.dot(u)
        float(np.linalg.norm(r))
    _W.update(u=u, v=v, r=r, i=i0 + k)
    return time.perf_counter() - t0


class CpuReference:
    """The oracle port of the reference path on all host cores: one process
    per system (OPENBLAS_NUM_THREADS=1, as SURVEY.md §8(d) prescribes)."""

    def __init__(self, workers=None, n=N_SIDE):
        import multiprocessing as mp
        self.cores = workers or min(32, len(os.sched_getaffinity(0)))
        wl = workload(0)
        ctx = mp.get_context("fork")
        self.pools = []
        for k in range(self.cores):
            p = wl["problems"][k % len(wl["problems"])]
            w = wl["schedules"][k % len(wl["problems"])].omega
            self.pools.append(ctx.Pool(1, initializer=_cpu_worker_init,
                                       initargs=(p.epsilon, p.theta, n, 100 + k, w)))
        self.n = n
        for p in self.pools:   # wait for assembly
            p.apply(_cpu_worker_steps, (0,))

    def run(self, k):
        """Wall time for every worker to run k inner steps concurrently."""
        t0 = time.perf_counter()
        res = [p.apply_async(_cpu_worker_steps, (k,)) for p in self.pools]
        for r in res:
            r.get()
        return time.perf_counter() - t0

    def updates(self, k):
        return self.cores * (self.n - 1) ** 2 * k

    def close(self):
        for p in self.pools:
            p.terminate()


# ------------------------------------------------------------------ dist
def dist_setup():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    return rank, world, local


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------ arms
def config_dict():
    return {"workload": "cfg3: 8 anisotropic systems/GPU on 1024^2 cells (1023^2 unknowns), "
                        "weighted-Jacobi Richardson(32), Leja-ordered Chebyshev weights, f64",
            "systems_per_gpu": SYSTEMS_PER_GPU, "grid": N_SIDE - 1, "m": M,
            "step": "one outer sweep (32 inner updates) of every system",
            "l2": "no flush: per-GPU working set 3 x 67 MB > 126 MB L2",
            "seed": 3}


def run_reference(args, rank, world):
    """--impl reference: the CPU port of the reference path, rank 0 only."""
    if rank != 0:
        return None
    ref = CpuReference()
    k_inner = 2   # inner steps per worker per step (bounded sample)
    for _ in range(args.warmup):
        ref.run(k_inner)
    times = [ref.run(k_inner) for _ in range(args.steps)]
    ref.close()
    t = float(np.sum(times))
    upd = ref.updates(k_inner) * args.steps
    value = upd / t
    sample = (f"{ref.cores} processes x 1 system (1023^2) x {k_inner} Jacobi-Richardson inner "
              f"steps per step, oracle port (SciPy CSR matvec + NumPy), OPENBLAS_NUM_THREADS=1")
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": ref.cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_gpu(args, rank, world, local):
    import torch
    import paper_2412_08076_b200 as G

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    wl = workload(rank)
    probs, scheds, scales = wl["problems"], wl["schedules"], wl["scales"]
    op = G.GpuStencilOperator.from_problems(probs, dtype=np.float64, device=dev)
    F = wl["F"]
    P = [G.JacobiScale(np.float64(s)) for s in scales]
    B, Pn = op.batch, op.P

    # ---- device-resident timed sweeps
    S = G.StationarySolver(op, scheds, P, tol=1e-300, max_outer=10**7, block_T=args.block_T)
    S.begin(F_dev(op, F))
    stream = torch.cuda.current_stream()
    launches_per_step = None
    for _ in range(args.warmup):
        n0 = S.info()[2]
        steps = 0
        while steps < M:
            steps += S.step()
        launches_per_step = S.info()[2] - n0
    torch.cuda.synchronize()
    kernel, block_T, seg_rows = S.plan()
    # one CUDA event pair per step (sweep); the launches of a sweep are
    # back to back on the stream, so a sweep's duration / its launches is
    # the average launch duration of the dominant kernel
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    chunk_T = []
    barrier(world)
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            steps = 0
            while steps < M:
                k = S.step()
                if i == 0:
                    chunk_T.append(k)
                steps += k
            ev[i][1].record(stream)
        stop.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    t_local = start.elapsed_time(stop) / 1e3
    t = max_over_ranks(t_local, world)
    upd_step = B * Pn * M
    value = world * upd_step * args.steps / t
    e = args.steps * launches_per_step                     # our kernel launches in the region
    dur = np.array([ev[i][0].elapsed_time(ev[i][1]) / 1e3 for i in range(args.steps)])
    avg = float(dur.sum() / e)                             # average launch duration
    avg_T = float(M / launches_per_step)
    alg_bytes = BYTES_PER_UPDATE * B * Pn * avg_T          # per launch (average)
    achieved = alg_bytes / avg / 1e9
    peak = _peak_hbm()
    share = float(dur.sum() / t_local)
    # the bound that actually limits the sweep: FP64 issue.  22 FP64
    # instructions per COMPUTED point-step (11 DMUL + 10 DADD + 1 DFMA: the
    # reference's unfused CSR-order sum, SASS-counted), halo recomputation
    # of the kernel's tiling included
    side = N_SIDE - 1
    computed = sum(_computed_point_steps(kernel, side, T_, seg_rows) for T_ in chunk_T) * B
    fp64_rate = computed * FP64_PER_POINT_STEP / (float(dur.sum()) / args.steps)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    fp64_peak = n_sm * 64 * (clk.summary().get("sm_mhz") or 1965.0) * 1e6

    # ---- end to end through the public API: one e2e step is the call a
    # richlab user makes, solve_stationary(..., tol=1e-6), batched over the
    # GPU's systems: H2D of f from pinned memory, the whole device loop to
    # 1e-6 (or max_outer), D2H of the solutions into pinned memory.  Updates
    # counted are the ones actually performed (sum of inner_iterations).
    Fh = torch.from_numpy(F).pin_memory()
    Uh = torch.zeros_like(Fh).pin_memory()
    e2e_times, e2e_upd, reps = [], [], None
    for it in range(1 + args.e2e_steps if args.e2e_steps > 0 else 0):
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        res = G.solve_stationary_batched(op, Fh, scheds, P, tol=TOL, max_outer=MAX_OUTER_TOL,
                                         out=Uh)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if it >= 1:
            e2e_times.append(max_over_ranks(dt, world))
            e2e_upd.append(sum(r.inner_iterations for _, r in res) * Pn)
            reps = [r for _, r in res]
    e2e_value, ttt = None, None
    if e2e_times:
        tot_upd = sum_over_ranks(float(np.mean(e2e_upd)), world)   # all ranks' systems
        e2e_value = tot_upd / float(np.mean(e2e_times))
        ttt = {"seconds": float(np.mean(e2e_times)), "tol": TOL, "max_outer": MAX_OUTER_TOL,
               "through": "public API incl. H2D f / D2H u",
               "converged": [int(r.converged) for r in reps],
               "outer_sweeps": [int(r.iterations) for r in reps],
               "inner_iterations": [int(r.inner_iterations) for r in reps],
               "final_rel": [float(r.final_relative_residual) for r in reps]}

    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            ref = CpuReference()
            # bounded sample of ~10 s wall: a short probe sizes the real run
            k_probe = 4
            tp = ref.run(k_probe)
            k_inner = max(k_probe, int(np.ceil(k_probe * args.cpu_seconds / max(tp, 1e-3))))
            tc = ref.run(k_inner)
            cpu = {"value": ref.updates(k_inner) / tc, "unit": UNIT, "cores": ref.cores,
                   "kind": "port",
                   "sample": f"{ref.cores} processes x 1 system (1023^2) x {k_inner} inner steps "
                             f"of the oracle port, {tc:.1f} s wall"}
            ref.close()
        traffic = _ncu_traffic(avg_T)
        import bench_configs as BC
        cpu_ttt = BC.cfg3_cpu_time_to_tol(cpu, ttt["inner_iterations"] if ttt else None, Pn) \
            if world == 1 else None
        dropin = None
        if world == 1 and args.dropin:
            dropin = BC.cfg3_dropin(None, wl, N_SIDE, TOL, MAX_OUTER_TOL)
        configs = BC.run_all(ROOT) if (world == 1 and args.configs) else None
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic", "config": config_dict(), "block_T": block_T, "kernel": kernel,
               "clocks": clk.summary(),
               "e2e": None if e2e_value is None else {"value": e2e_value, "unit": UNIT,
                       "h2d_bytes_per_step": int(F.nbytes), "d2h_bytes_per_step": int(F.nbytes),
                       "step": "one full solve to 1e-6 of the GPU's 8 systems",
                       "api": "solve_stationary_batched(op, f_pinned, schedules, P, tol=1e-6, "
                              "max_outer=10000, out=u_pinned)"},
               "gpu_launches": int(e),
               "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak["value"],
                            "unit": "GB/s", "frac": achieved / peak["value"],
                            "traffic": traffic, "peak_source": peak["source"],
                            "kernel": _kernel_name(kernel, block_T, seg_rows, chunk_T),
                            "algorithmic_bytes_per_launch": alg_bytes,
                            "avg_steps_per_launch": avg_T,
                            "avg_launch_s": avg, "kernel_share_of_step": share,
                            "note": "algorithmic bytes count 24 B per point-update per inner "
                                    "step; temporal blocking fuses T steps per HBM pass, so "
                                    "frac can exceed 1 (SURVEY.md §8(d))",
                            "fp64_issue": {"achieved_Tinst_s": fp64_rate / 1e12,
                                           "peak_Tinst_s": fp64_peak / 1e12,
                                           "frac": fp64_rate / fp64_peak,
                                           "computed_point_steps_per_owned": computed / (
                                               B * Pn * float(M)),
                                           "note": "FP64 instructions issued (22 per computed "
                                                   "point-step, halo recomputation included) "
                                                   "against SMs x 64 FP64 lanes x SM clock: "
                                                   "the limiting pipe of the blocked kernel"}},
               "cpu_baseline": cpu, "time_to_tol": ttt, "cpu_time_to_tol": cpu_ttt,
               "e2e_dropin": dropin, "configs": configs}
    return out


def F_dev(op, F):
    return op.to_device(F)


def _computed_point_steps(kernel, side, T, seg_rows):
    """Point-steps one launch of T fused steps computes for ONE system
    (owned points plus the recomputed halo of the kernel's tiling)."""
    if kernel == "wave":
        W = 128                                   # csrc/wave.cuh: 32 lanes x 4 columns
        nstrip = -(-side // (W - 2 * T))
        total = 0
        for r0 in range(0, side, seg_rows):
            L = min(seg_rows, side - r0)
            total += sum(W * (L + 2 * T - 2 * t) for t in range(1, T + 1))
        return nstrip * total
    if kernel == "tile":
        tiles = (-(-side // (64 - 2 * T))) ** 2   # block_ntiles: 64 x 64 windows
        return tiles * 64 * 64 * T
    return side * side * T


def _kernel_name(kernel, T, seg_rows, chunks):
    if kernel == "wave":
        return (f"wave_kernel<double,T={T},Jacobi> (csrc/wave.cuh: 128-column strips x "
                f"{seg_rows}-row segments, chunks {sorted(set(chunks))})")
    if kernel == "tile":
        return f"block_kernel<double,plain,T~{T}> (chunks {sorted(set(chunks))})"
    return kernel


def _peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return {"value": float(json.loads(p.read_text())["hbm_gbs"]), "source": "measured"}
    except Exception:  # noqa: BLE001
        return {"value": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def _ncu_traffic(avg_T):
    """DRAM bytes per launch of the dominant kernel, from the committed ncu
    capture (profiles/ncu_wave_kernel.json: read + write of one T = 4
    launch: u and f read once, u written once, plus the strip / segment
    halos), or None."""
    p = ROOT / "profiles" / "ncu_wave_kernel.json"
    try:
        d = json.loads(p.read_text())
        return float(d["dram_bytes_per_launch"])
    except Exception:  # noqa: BLE001
        return None


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--block-T", dest="block_T", type=int, default=0)
    ap.add_argument("--e2e-steps", dest="e2e_steps", type=int, default=2)
    ap.add_argument("--no-time-to-tol", dest="time_to_tol", action="store_false")  # kept for scripts
    ap.add_argument("--no-cpu", dest="no_cpu", action="store_true")
    ap.add_argument("--no-configs", dest="configs", action="store_false",
                    help="skip the per-config lines (cfg1, cfg2, cfg4, cfg5, NAG(16) sweep)")
    ap.add_argument("--no-dropin", dest="dropin", action="store_false",
                    help="skip the cfg3 reference-signature (CSR + numpy) e2e")
    ap.add_argument("--cpu-seconds", dest="cpu_seconds", type=float, default=10.0,
                    help="wall-time target of the bounded CPU baseline sample")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    rank, world, local = dist_setup()
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        out = run_gpu(args, rank, world, local)
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

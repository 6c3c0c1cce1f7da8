"""GS / SOR / SSOR probe: device time of one
triangular-preconditioner application at 255^2 x 64 and 1023^2 x 8, an
SSOR-preconditioned NAG(3) solve to 1e-6 at 1023^2 x 8 (the paper's
NAGex(3) + SSOR family), and the oracle's (SuperLU) time for one application.

    python profiles/precond_probe.py [--no-cpu]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle as O  # noqa: E402  (CPU comparison + one-time assembly)
import paper_2412_08076_b200 as G  # noqa: E402


def ev_time(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--quick", action="store_true", help="application timings only")
    args = ap.parse_args()
    out = {}
    rng = np.random.default_rng(0)
    for n, B in ((256, 64), (1024, 8)):
        As = [O.assemble_anisotropic(10 ** rng.uniform(-4, 0), rng.uniform(0, np.pi), n)
              for _ in range(B)]
        op = G.GpuStencilOperator.stack([G.GpuStencilOperator.from_sparse(A) for A in As])
        R = torch.randn(B, op.P, dtype=torch.float64, device="cuda")
        Z, W = torch.empty_like(R), torch.empty_like(R)
        row = {}
        for kind, relax in (("sor", 1.5), ("ssor", 1.0)):
            pre = G.TriangularPreconditioner(op, kind, relax)
            passes = 1 if kind == "sor" else 2
            ms = ev_time(lambda: pre.apply_device(R, Z, W), 5)
            row[kind] = {"ms_per_apply_batch": ms, "systems": B,
                         "point_solves_per_s": passes * B * op.P / (ms * 1e-3),
                         "ns_per_wavefront_step": ms * 1e6 / (passes * (3 * (n - 1) - 2))}
        if not args.no_cpu:
            f = O.tri_precond(As[0], "ssor", 1.0)
            r0 = R[0].cpu().numpy()
            f(r0)
            t0 = time.perf_counter()
            for _ in range(3):
                f(r0)
            row["cpu_ssor_ms_per_system"] = (time.perf_counter() - t0) / 3 * 1e3
        out[f"{n - 1}^2 x {B}"] = row
    if args.quick:
        print(json.dumps({k: {m: round(v[m]["ms_per_apply_batch"], 4) for m in ("sor", "ssor")}
                          for k, v in out.items()}))
        return
    # NAG(3) + SSOR solve to 1e-6 at 1023^2 x 8 (weights for B^{-1}A in (0, 1])
    n, B = 1024, 8
    As = [O.assemble_anisotropic(10 ** rng.uniform(-2, 0), rng.uniform(0, np.pi), n)
          for _ in range(B)]
    op = G.GpuStencilOperator.stack([G.GpuStencilOperator.from_sparse(A) for A in As])
    F = rng.standard_normal((B, op.P))
    sch = G.WeightSchedule(omega=np.array([1.0, 1.0, 1.0]), alpha=np.array([0.9, 0.9, 0.9]),
                           variant="nag")
    Fd = torch.as_tensor(F, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = G.solve_stationary_batched(op, Fd, sch, P=G.Preconditioner.ssor(op, 1.0), tol=1e-6,
                                     max_outer=300)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    out["nag3_ssor_1023^2_x8"] = {
        "wall_s": wall, "iterations": [r.iterations for _, r in res],
        "converged": [bool(r.converged) for _, r in res],
        "final_rel": [float(r.final_relative_residual) for _, r in res]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

"""Tuning probe: device throughput of the cfg3 sweep for each temporal-
blocking depth T (and variant), CUDA-event timed, no host sync inside.

python profiles/sweep_bench.py [--variant plain|mom|nag] [--dtype f64|f32]
                               [--n 1024] [--batch 8] [--sweeps 20]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2412_08076_b200 as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="plain")
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--m", type=int, default=32)
    ap.add_argument("--sweeps", type=int, default=20)
    ap.add_argument("--T", default="1,2,3,4,5,6,7,8")
    a = ap.parse_args()
    dt = np.float64 if a.dtype == "f64" else np.float32
    rng = np.random.default_rng(0)
    probs = [G.AnisotropicProblem(10 ** rng.uniform(-4, 0), rng.uniform(0, np.pi), a.n)
             for _ in range(a.batch)]
    op = G.GpuStencilOperator.from_problems(probs, dtype=dt)
    F = rng.standard_normal((a.batch, op.P))
    m = a.m
    if a.variant == "plain":
        s = G.WeightSchedule(omega=np.full(m, 0.2))
    else:
        s = G.WeightSchedule(omega=np.full(m, 0.2), alpha=np.full(m, 0.3), variant=a.variant)
    P = G.JacobiScale(np.float64(0.3)) if a.variant == "plain" else None
    out = {}
    for T in [int(x) for x in a.T.split(",")]:
        S = G.StationarySolver(op, s, P, tol=1e-300, max_outer=10**7, block_T=T)
        S.begin(F)
        for _ in range(3 * m):
            S.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        steps = 0
        while steps < a.sweeps * m:
            steps += S.step()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        upd = a.batch * op.P * steps
        out[T] = upd / t / 1e9
        print(f"T={T}: {out[T]:8.1f} G upd/s  ({1e3 * t / a.sweeps:.3f} ms/sweep)", flush=True)
    print(json.dumps({"variant": a.variant, "dtype": a.dtype, "n": a.n, "batch": a.batch,
                      "G_upd_per_s": out}))


if __name__ == "__main__":
    main()

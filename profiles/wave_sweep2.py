"""In-process depth / segment sweep of the wavefront sweep (csrc/wave.cuh) on
cfg3 (8 x 1023^2, Jacobi Richardson(32), f64).  RG_WAVE / RG_WAVE_L are read
when a solver is created, so one process measures every configuration, each
three times, interleaved with the overlapped-tile kernel (RG_WAVE=0); the
iterate after 4 sweeps is compared bitwise with the tile kernel's.

python profiles/wave_sweep2.py --T 3,4 --L 32,48,64 [--out file.json]
"""
import argparse
import hashlib
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_08076_b200 as G  # noqa: E402
from paper_2412_08076_b200 import configs as CF  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", default="4")
ap.add_argument("--L", default="64")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--out", default=None)
ap.add_argument("--batch", type=int, default=8)
args = ap.parse_args()

wl = CF.cfg3(count=args.batch)
op = G.GpuStencilOperator.from_problems(wl["problems"])
P = [G.JacobiScale(np.float64(s)) for s in wl["scales"]]
Fd = op.to_device(wl["F"])


def measure(T, env):
    os.environ.update(env)
    S4 = G.StationarySolver(op, wl["schedules"], P, tol=1e-300, max_outer=4, block_T=T)
    S4.begin(Fd)
    S4.run()
    res = S4.results(like_numpy=False)
    sha = hashlib.sha256(torch.stack([u for u, _ in res]).cpu().numpy().tobytes()).hexdigest()
    S = G.StationarySolver(op, wl["schedules"], P, tol=1e-300, max_outer=10**7, block_T=T)
    S.begin(Fd)
    S.run_sweeps(4)
    out = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        S.run_sweeps(20)
        e1.record()
        torch.cuda.synchronize()
        out.append(args.batch * 1023 ** 2 * 32 * 20 / (e0.elapsed_time(e1) / 1e3) / 1e9)
    del S, S4
    return out, sha


res = {}
tile, ref = measure(5, {"RG_WAVE": "0"})
res["tile_T5"] = tile
print("tile", [round(x, 1) for x in tile], flush=True)
for T in map(int, args.T.split(",")):
    for L in map(int, args.L.split(",")):
        g, sha = measure(T, {"RG_WAVE": "1", "RG_WAVE_L": str(L)})
        res[f"wave_T{T}_L{L}"] = {"gups": g, "bitwise": sha == ref}
        print(f"T={T} L={L}", [round(x, 1) for x in g], sha == ref, flush=True)
tile2, _ = measure(5, {"RG_WAVE": "0"})
res["tile_T5_end"] = tile2
print("tile", [round(x, 1) for x in tile2], flush=True)
if args.out:
    Path(args.out).write_text(json.dumps(res, indent=1))

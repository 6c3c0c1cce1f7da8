"""Depth / segment sweep of the wavefront plain sweep (csrc/wave.cuh) on the
cfg3 workload (8 x 1023^2, Jacobi Richardson(32), f64), against the
overlapped-tile kernel (RG_WAVE=0).  Each configuration runs in its own
process (the library reads RG_WAVE / RG_WAVE_L once).  Every run's iterate
after 4 sweeps is compared bitwise with the tile kernel's.

python profiles/wave_sweep.py [--out profiles/wave_sweep_r02.json]
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CHILD = r"""
import sys, json, hashlib
sys.path.insert(0, {root!r})
import numpy as np, torch
import paper_2412_08076_b200 as G
from paper_2412_08076_b200 import configs as CF
wl = CF.cfg3()
op = G.GpuStencilOperator.from_problems(wl["problems"])
P = [G.JacobiScale(np.float64(s)) for s in wl["scales"]]
Fd = op.to_device(wl["F"])
T = {T}
S4 = G.StationarySolver(op, wl["schedules"], P, tol=1e-300, max_outer=4, block_T=T)
S4.begin(Fd)
S4.run()
res = S4.results(like_numpy=False)
sha = hashlib.sha256(torch.stack([u for u, _ in res]).cpu().numpy().tobytes()).hexdigest()
S = G.StationarySolver(op, wl["schedules"], P, tol=1e-300, max_outer=10**7, block_T=T)
S.begin(Fd)
S.run_sweeps(4)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
S.run_sweeps(2)
torch.cuda.synchronize()
e0.record()
S.run_sweeps(20)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 1e3
print(json.dumps(dict(T=T, gups=8 * 1023 ** 2 * 32 * 20 / t / 1e9, sha=sha)))
"""


def run(env, T):
    e = dict(os.environ, **env)
    p = subprocess.run([sys.executable, "-c", CHILD.format(root=str(ROOT), T=T)], env=e,
                       capture_output=True, text=True, timeout=300)
    if p.returncode != 0:
        return {"error": p.stderr[-800:]}
    return json.loads(p.stdout.strip().splitlines()[-1])


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--T", default="2,3,4,5,6")
    ap.add_argument("--L", default="32,48,64,96,128")
    args = ap.parse_args()
    out = {}
    ref = run({"RG_WAVE": "0"}, 5)
    out["tile_T5"] = ref
    for T in map(int, args.T.split(",")):
        for L in map(int, args.L.split(",")):
            r = run({"RG_WAVE": "1", "RG_WAVE_L": str(L)}, T)
            if "sha" in r:
                r["bitwise_vs_tile_after_4_sweeps"] = r.pop("sha") == ref.get("sha")
            out[f"wave_T{T}_L{L}"] = r
            print(f"T={T} L={L}: {r}", flush=True)
    print(json.dumps(out, indent=1))
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

"""Training-unroll probe: forward + reverse of the
K = 50 unroll (TrainConfig default) on 8 x 1023^2 NAG systems with Jacobi,
device time per loss+gradient evaluation, and the oracle's time for one
system.   python profiles/unroll_probe.py [--no-cpu]"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle as O  # noqa: E402
import paper_2412_08076_b200 as G  # noqa: E402
from paper_2412_08076_b200 import training as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--no-cpu", action="store_true")
args = ap.parse_args()
rng = np.random.default_rng(0)
B, n, K, m = 8, 1024, 50, 3
As = [O.assemble_anisotropic(10 ** rng.uniform(-2, 0), rng.uniform(0, np.pi), n) for _ in range(B)]
op = G.GpuStencilOperator.stack([G.GpuStencilOperator.from_sparse(A) for A in As])
F = torch.as_tensor(rng.standard_normal((B, op.P)), device="cuda")
W = rng.uniform(0.3, 0.6, (B, m))
Al = rng.uniform(0.1, 0.4, (B, m))
P = G.JacobiScale(np.asarray((2.0 / 3.0) / op._host_stencil[0, 4]))
eng = T.UnrollEngine(op, K, "nag", P)
eng.forward(F, W, Al, Al)
eng.backward()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
s.record()
for _ in range(reps):
    eng.forward(F, W, Al, Al)
mid = torch.cuda.Event(enable_timing=True)
mid.record()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    eng.backward()
e.record()
torch.cuda.synchronize()
fw = s.elapsed_time(mid) / reps
bw = mid.elapsed_time(e) / reps
# algorithmic bytes: forward 40 B/pt/step (u, v r/w, f r); adjoint 2 passes ~ 112 B/pt/step
pts = B * op.P * K
out = {"config": f"{B} x 1023^2 nag m={m} K={K} jacobi", "forward_ms": fw, "backward_ms": bw,
       "loss_grad_ms": fw + bw,
       "forward_GBs": 40 * pts / (fw * 1e-3) / 1e9,
       "backward_GBs_est": 112 * pts / (bw * 1e-3) / 1e9}
if not args.no_cpu:
    A0 = As[0]
    sc = O.jacobi_scale(A0)
    f0 = F[0].cpu().numpy()
    t0 = time.perf_counter()
    O.unroll_grad(A0, f0, W[0], Al[0], Al[0], K, "nag", sc)
    out["cpu_s_per_system"] = time.perf_counter() - t0
print(json.dumps(out))

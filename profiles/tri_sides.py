"""Wavefront preconditioner time against grid side (ns per dependent step)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle as O  # noqa: E402
import paper_2412_08076_b200 as G  # noqa: E402


def ev_time(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize(); s.record()
    for _ in range(reps):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for n, B in ((64, 8), (128, 8), (256, 8), (512, 8), (1024, 1), (1024, 8), (1024, 18), (2048, 4)):
    A = O.assemble_anisotropic(0.01, 0.5, n)
    op = G.GpuStencilOperator.from_sparse(A).broadcast(B)
    R = torch.randn(B, op.P, dtype=torch.float64, device="cuda")
    Z, W = torch.empty_like(R), torch.empty_like(R)
    pre = G.TriangularPreconditioner(op, "sor", 1.5)
    ms = ev_time(lambda: pre.apply_device(R, Z, W), 10)
    side = n - 1
    print(f"side {side:5d} batch {B:3d}: {ms*1e3:8.1f} us  {ms*1e6/(3*side):7.1f} ns per 3*side step")

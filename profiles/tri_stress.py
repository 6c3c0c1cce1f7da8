"""Stress of the cluster SOR/SSOR wavefront (DSMEM hand-off): many repeats at
full occupancy (8 and 16 systems at 1023^2, 64 systems at 255^2, both
rows-per-CTA forms via RG_TRI_RPC), identical bits every run and 1e-13
against the oracle on one system."""
import os
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle as O  # noqa: E402
import paper_2412_08076_b200 as G  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(5)
for n, B in ((1024, 8), (1024, 16), (256, 64), (2048, 2)):
    A = O.assemble_anisotropic(0.03, 1.1, n)
    op = G.GpuStencilOperator.from_sparse(A).broadcast(B)
    R = torch.as_tensor(rng.standard_normal((B, op.P))).cuda()
    for kind, relax in (("sor", 1.4), ("ssor", 1.0)):
        pre = G.TriangularPreconditioner(op, kind, relax)
        ref = pre.apply_device(R).clone()
        if n <= 1024:
            zo = O.tri_precond(A, kind, relax)(R[B - 1].cpu().numpy())
            err = np.linalg.norm(ref[B - 1].cpu().numpy() - zo) / np.linalg.norm(zo)
        else:
            err = float("nan")
        Z, W = torch.empty_like(R), torch.empty_like(R)
        bad = 0
        for _ in range(reps):
            pre.apply_device(R, Z, W)
            bad += int(not torch.equal(Z, ref))
        print(f"RPC={os.environ.get('RG_TRI_RPC', 'auto')} n={n} B={B} {kind}: rel err {err:.2e}, "
              f"{bad} of {reps} runs differ", flush=True)

"""One SOR application at 1023^2 x 8 (ncu target for tri_kernel)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle as O  # noqa: E402
import paper_2412_08076_b200 as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
A = O.assemble_anisotropic(0.01, 0.5, n)
op = G.GpuStencilOperator.from_sparse(A).broadcast(B)
R = torch.randn(B, op.P, dtype=torch.float64, device="cuda")
pre = G.TriangularPreconditioner(op, "sor", 1.5)
for _ in range(3):
    pre.apply_device(R)
torch.cuda.synchronize()
print("ok")

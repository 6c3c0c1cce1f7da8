"""cfg4 probe: a few FNS alternations on 4 x 1023^2 (for ncu launch lists)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2412_08076_b200 as G  # noqa: E402
from paper_2412_08076_b200 import configs as CF  # noqa: E402
from paper_2412_08076_b200 import fns as GF  # noqa: E402

c = CF.cfg4()
op = G.GpuStencilOperator.from_problems(c["problems"])
eng = GF.FnsEngine(op, c["schedule"], GF.SpectralCorrection(c["lam"], 1024), c["M"])
Fd = op.to_device(c["F"])
eng.u[0].zero_()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    u = eng.step(Fd)
    op.residual(u, Fd, want_r=False)
torch.cuda.synchronize()
print("ok")

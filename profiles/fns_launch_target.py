"""cfg4: 3 FNS alternations after warm-up (ncu launch-list target)."""
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
for _ in range(3):
    eng.step(Fd)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(3):
    eng.step(Fd)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()

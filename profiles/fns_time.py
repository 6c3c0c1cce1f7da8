"""cfg4: device time per FNS alternation (CUDA events), warm."""
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
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    eng.step(Fd)
e.record()
torch.cuda.synchronize()
print(f"ms per alternation: {s.elapsed_time(e) / 20:.4f}")

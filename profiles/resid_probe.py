"""Residual-norm pass (rg_residual, norm only) at 4 and 8 x 1023^2 f64."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2412_08076_b200 as G  # noqa: E402
from paper_2412_08076_b200 import configs as CF  # noqa: E402
for B in (4, 8):
    c = CF.cfg3(count=B)
    op = G.GpuStencilOperator.from_problems(c["problems"])
    F = op.to_device(c["F"])
    U = torch.randn_like(F)
    for want_r in (False, True):
        op.residual(U, F, want_r=want_r)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(50):
            op.residual(U, F, want_r=want_r)
        e.record()
        torch.cuda.synchronize()
        print(f"B {B} want_r {want_r}: {s.elapsed_time(e) / 50 * 1e3:.1f} us")

"""One FGMRES(20) cycle of cfg5 (ncu launch-list target)."""
import importlib
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle as O  # noqa: E402
import paper_2412_08076_b200 as G  # noqa: E402
from paper_2412_08076_b200 import configs as CF  # noqa: E402
from paper_2412_08076_b200 import multigrid as GM  # noqa: E402
GG = importlib.import_module("paper_2412_08076_b200.fgmres")

c = CF.cfg5()
hp = c["problem"]
A = O.assemble_helmholtz(hp.angular_frequency, hp.n)
h = GM.build_hierarchy(A, hp.n, coarsest=16, schedules=c["schedule"], batch=4)
op = G.GpuStencilOperator.from_problems([hp]).broadcast(4)
Fd = op.to_device(c["F"])
h.apply(Fd)
GG.fgmres_batched(op, Fd, precond_apply=h.apply, cfg=GG.FgmresConfig(restart=3, max_outer=1))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
GG.fgmres_batched(op, Fd, precond_apply=h.apply, cfg=GG.FgmresConfig(restart=20, max_outer=1))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()

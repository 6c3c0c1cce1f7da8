"""cfg5 probe: V-cycles on 4 x 1023^2 Helmholtz RHS (eager, for ncu launch lists)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle as O  # noqa: E402  (host CSR for the one-time hierarchy setup)
import paper_2412_08076_b200 as G  # noqa: E402
from paper_2412_08076_b200 import configs as CF  # noqa: E402
from paper_2412_08076_b200 import multigrid as GM  # noqa: E402

c = CF.cfg5()
hp = c["problem"]
A = O.assemble_helmholtz(hp.angular_frequency, hp.n)
h = GM.build_hierarchy(A, hp.n, coarsest=16, schedules=c["schedule"], batch=4)
h.use_graphs = False
op = G.GpuStencilOperator.from_problems([hp]).broadcast(4)
Fd = op.to_device(c["F"])
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    h.apply(Fd)
torch.cuda.synchronize()
print("ok")

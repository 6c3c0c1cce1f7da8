"""cfg5 V-cycle: warm device time of each level's smoothing call (16 NAG
steps, rg_sweep) and of the whole graph-replayed cycle."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle as O  # noqa: E402
import paper_2412_08076_b200 as G  # noqa: E402
from paper_2412_08076_b200 import configs as CF  # noqa: E402
from paper_2412_08076_b200 import multigrid as GM  # noqa: E402

c = CF.cfg5()
hp = c["problem"]
A = O.assemble_helmholtz(hp.angular_frequency, hp.n)
h = GM.build_hierarchy(A, hp.n, coarsest=16, schedules=c["schedule"], batch=4)
op = G.GpuStencilOperator.from_problems([hp]).broadcast(4)
Fd = op.to_device(c["F"])
h.apply(Fd)
torch.cuda.synchronize()


def ev(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


out = {"vcycle_us": ev(lambda: h.apply(Fd)), "graphs": bool(h.use_graphs)}
for k, lvl in enumerate(h.levels[:-1]):
    f = torch.randn(4, lvl.op.P, dtype=torch.complex128, device="cuda")
    u = torch.zeros_like(f)
    out[f"level{k}_side{lvl.op.side}_{['const9','diag5','var9'][lvl.op.kind - 1]}_smooth_us"] = \
        ev(lambda: h._smooth(k, f, u, 1))
print(json.dumps(out))

"""cfg5 FGMRES(20) phase timing: preconditioner, matvec, MGS, host recurrences."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle as O  # noqa: E402
import paper_2412_08076_b200 as G  # noqa: E402
from paper_2412_08076_b200 import configs as CF  # noqa: E402
import paper_2412_08076_b200.fgmres  # noqa: E402,F401  (the package attribute is the function)
GG = sys.modules["paper_2412_08076_b200.fgmres"]
from paper_2412_08076_b200 import multigrid as GM  # noqa: E402

c = CF.cfg5()
hp = c["problem"]
A = O.assemble_helmholtz(hp.angular_frequency, hp.n)
h = GM.build_hierarchy(A, hp.n, coarsest=16, schedules=c["schedule"], batch=4)
op = G.GpuStencilOperator.from_problems([hp]).broadcast(4)
Fd = op.to_device(c["F"])
T = {"precond": 0.0, "matvec": 0.0}


def timed(name, fn):
    def w(*a):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a)
        torch.cuda.synchronize()
        T[name] += time.perf_counter() - t0
        return r
    return w


h.apply(Fd)
GG.fgmres_batched(op, Fd, precond_apply=lambda R: h.apply(R),
                  cfg=GG.FgmresConfig(restart=2, tol=1e-6, max_outer=1))   # warm-up
orig_mv = GG._matvec
GG._matvec = timed("matvec", orig_mv)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = GG.fgmres_batched(op, Fd, precond_apply=timed("precond", lambda R: h.apply(R)),
                        cfg=GG.FgmresConfig(restart=20, tol=1e-6, max_outer=1))
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print(f"20 Arnoldi steps: total {1e3*tot:.1f} ms  precond {1e3*T['precond']:.1f} ms  "
      f"matvec {1e3*T['matvec']:.1f} ms  rest {1e3*(tot-T['precond']-T['matvec']):.1f} ms")

from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    GG.fgmres_batched(op, Fd, precond_apply=lambda R: h.apply(R),
                      cfg=GG.FgmresConfig(restart=6, tol=1e-6, max_outer=1))
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=14))

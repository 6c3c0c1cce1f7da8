"""Where does the end-to-end API time go?  Times each phase of
solve_stationary_batched on the cfg3 workload (host pinned in/out)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2412_08076_b200 as G  # noqa: E402
from paper_2412_08076_b200 import configs  # noqa: E402

wl = configs.cfg3(count=8)
op = G.GpuStencilOperator.from_problems(wl["problems"])
P = [G.JacobiScale(np.float64(s)) for s in wl["scales"]]
Fh = torch.from_numpy(wl["F"]).pin_memory()
Uh = [torch.zeros_like(Fh).pin_memory(), torch.zeros_like(Fh).pin_memory()]


def phase(name, fn, log):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    log.append((name, 1e3 * (time.perf_counter() - t0)))
    return r


for it in range(4):
    log = []
    S = phase("cached()", lambda: G.StationarySolver.cached(op, wl["schedules"], P, 1e-300, 1), log)
    phase("begin (H2D f,u0)", lambda: S.begin(Fh, Uh[0]), log)
    phase("run (1 sweep + poll)", lambda: S.run(), log)
    phase("results (D2H u)", lambda: S.results(like_numpy=True, out=Uh[1]), log)
    tot = sum(t for _, t in log)
    print(f"iter {it}: total {tot:.2f} ms  " + "  ".join(f"{n}={t:.2f}" for n, t in log), flush=True)

"""cfg1 time split: device time of the single-launch solve vs the API call."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2412_08076_b200 as G  # noqa: E402
from paper_2412_08076_b200 import configs  # noqa: E402

c = configs.cfg1()
op = G.GpuStencilOperator.from_problems([c["problem"]])
f = c["f"]
S = G.StationarySolver(op, c["schedule"], None, tol=1e-6, max_outer=100_000)
for it in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S.begin(f)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    S.run()
    e1.record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    u, rep = S.result(0)
    t2 = time.perf_counter()
    print(f"device solve {e0.elapsed_time(e1):.3f} ms   begin+run+poll {1e3*(t1-t0):.3f} ms   "
          f"result {1e3*(t2-t1):.3f} ms   outer={rep.iterations}", flush=True)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, rep = G.solve_stationary(op, f, c["schedule"], tol=1e-6)
    print(f"solve_stationary API {1e3*(time.perf_counter()-t0):.3f} ms", flush=True)

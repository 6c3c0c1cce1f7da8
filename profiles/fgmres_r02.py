"""cfg5 FGMRES(20) x 5 with the pipelined driver: wall time against 100
back-to-back V-cycles (the preconditioner alone), 4 right-hand sides."""
import importlib
import json
import sys
import time
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
cfg = GG.FgmresConfig(restart=20, tol=1e-6, max_outer=5)
h.apply(Fd)
GG.fgmres_batched(op, Fd, precond_apply=h.apply, cfg=GG.FgmresConfig(restart=3, max_outer=1))
out = {}
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(100):
        h.apply(Fd, check=False)
    torch.cuda.synchronize()
    tv = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = GG.fgmres_batched(op, Fd, precond_apply=h.apply, cfg=cfg)
    torch.cuda.synchronize()
    tf = time.perf_counter() - t0
    out[f"rep{rep}"] = {"vcycles_100_s": tv, "fgmres_s": tf, "ratio": tf / tv,
                        "steps": [r.iterations for _, r in res]}
    print(out[f"rep{rep}"], flush=True)
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(json.dumps(out, indent=1))

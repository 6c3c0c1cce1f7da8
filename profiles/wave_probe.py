"""A few cfg3 sweeps through the wavefront kernel (ncu target):
RG_WAVE_L / block_T select the variant.  python profiles/wave_probe.py [T]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2412_08076_b200 as G
from paper_2412_08076_b200 import configs as CF

T = int(sys.argv[1]) if len(sys.argv) > 1 else 0
wl = CF.cfg3()
op = G.GpuStencilOperator.from_problems(wl["problems"])
P = [G.JacobiScale(np.float64(s)) for s in wl["scales"]]
S = G.StationarySolver(op, wl["schedules"], P, tol=1e-300, max_outer=10**7, block_T=T)
S.begin(op.to_device(wl["F"]))
S.run_sweeps(3)
torch.cuda.synchronize()
print("ok", S.info())

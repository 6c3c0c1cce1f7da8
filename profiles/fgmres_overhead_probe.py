import importlib, sys, time
from pathlib import Path
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import oracle as O
import paper_2412_08076_b200 as G
from paper_2412_08076_b200 import configs as CF, _lib as L
GG = importlib.import_module("paper_2412_08076_b200.fgmres")
c = CF.cfg5(); hp = c["problem"]
op = G.GpuStencilOperator.from_problems([hp]).broadcast(4)
Fd = op.to_device(c["F"])
cfg = GG.FgmresConfig(restart=20, tol=1e-6, max_outer=5)
ident = lambda R: R.clone()
GG.fgmres_batched(op, Fd, precond_apply=ident, cfg=GG.FgmresConfig(restart=3, max_outer=1))
for _ in range(2):
    torch.cuda.synchronize(); t0=time.perf_counter()
    res = GG.fgmres_batched(op, Fd, precond_apply=ident, cfg=cfg)
    torch.cuda.synchronize(); print("identity precond: 100 steps", time.perf_counter()-t0, [r.iterations for _, r in res])
# MGS alone timing for k = 0..19
B, n, mr = 4, op.P, 20
V = torch.randn((B, mr+1, n), dtype=torch.complex128, device='cuda')
w = torch.randn((B, n), dtype=torch.complex128, device='cuda')
hb = torch.empty((mr+1, B), dtype=torch.complex128, device='cuda'); n2 = torch.empty(B, dtype=torch.float64, device='cuda')
lib = L.load()
for k in (0, 9, 19):
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        L.check(lib.rg_mgs_arnoldi(L.RG_C128, B, n, L.ptr(w), n, L.ptr(V), (mr+1)*n, k, L.ptr(hb), L.ptr(n2), L.stream_ptr()))
    e1.record(); torch.cuda.synchronize(); print("mgs k=", k, e0.elapsed_time(e1)/10, "ms")

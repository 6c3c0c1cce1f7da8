"""MGS orthogonalisation timing (rg_mgs_arnoldi) over batch and k: separates the
launch cost from the per-phase cost of the persistent kernel."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2412_08076_b200 import _lib as L
lib = L.load()
n, mr = 1023 * 1023, 20
for B in (1, 4):
    V = torch.randn((B, mr + 1, n), dtype=torch.complex128, device='cuda')
    w = torch.randn((B, n), dtype=torch.complex128, device='cuda')
    hb = torch.empty((mr + 1, B), dtype=torch.complex128, device='cuda')
    n2 = torch.empty(B, dtype=torch.float64, device='cuda')
    for k in (0, 1, 3, 9, 19):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            L.check(lib.rg_mgs_arnoldi(L.RG_C128, B, n, L.ptr(w), n, L.ptr(V), (mr + 1) * n, k, L.ptr(hb),
                                       L.ptr(n2), L.stream_ptr()))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        phases = B * ((k + 2) // 2 + 1)
        print(f"B {B} k {k:2d}: {ms*1e3:7.1f} us, {phases:3d} phases, {ms*1e3/phases:5.1f} us/phase, "
              f"{B*(k+1)*n*16/ms/1e9:6.2f} TB/s of v")

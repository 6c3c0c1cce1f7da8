"""One k = 19 orthogonalisation of 4 x 1023^2 c128 (ncu target)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2412_08076_b200 import _lib as L
lib = L.load()
n, mr, B, k = 1023 * 1023, 20, 4, 19
V = torch.randn((B, mr + 1, n), dtype=torch.complex128, device='cuda')
w = torch.randn((B, n), dtype=torch.complex128, device='cuda')
hb = torch.empty((mr + 1, B), dtype=torch.complex128, device='cuda')
n2 = torch.empty(B, dtype=torch.float64, device='cuda')
for _ in range(3):
    L.check(lib.rg_mgs_arnoldi(L.RG_C128, B, n, L.ptr(w), n, L.ptr(V), (mr + 1) * n, k, L.ptr(hb), L.ptr(n2),
                               L.stream_ptr()))
torch.cuda.synchronize()
print("ok")

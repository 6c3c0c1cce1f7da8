"""Small workload touching every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck; run ONE tool per gpurun call)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle as O  # noqa: E402
import paper_2412_08076_b200 as G  # noqa: E402
import paper_2412_08076_b200.fgmres  # noqa: E402,F401  (the package attribute is the function)
GG = sys.modules["paper_2412_08076_b200.fgmres"]
from paper_2412_08076_b200 import fns as GF  # noqa: E402
from paper_2412_08076_b200 import multigrid as GM  # noqa: E402

rng = np.random.default_rng(0)
A = O.assemble_anisotropic(0.05, 0.7, 80)           # 79^2: tiled block kernel + boundary tiles
f = rng.standard_normal(A.shape[0])
for variant, kw in (("plain", {}), ("mom", {"alpha": [0.3] * 6}), ("nag", {"alpha": [0.3] * 6})):
    s = G.WeightSchedule(omega=[0.2] * 6, variant=variant, **kw)
    for T in (1, 5):
        G.solve_stationary(A, f, s, P=G.JacobiScale(O.jacobi_scale(A)), tol=1e-300,
                           max_outer=2, block_T=T)
    G.solve_stationary(O.assemble_anisotropic(0.05, 0.7, 40), rng.standard_normal(39 * 39), s,
                       tol=1e-300, max_outer=2)     # single-launch small solver
    G.solve_stationary(A, f, s, tol=1e-300, max_outer=2, check="inner")
st = G.IterationState.start(A.shape[0])
G.outer_sweep(A, f, st, G.WeightSchedule(omega=[0.2, 0.3]))
op32 = G.GpuStencilOperator.from_sparse(A, dtype=np.float32)
G.solve_stationary(op32, f.astype(np.float32), G.WeightSchedule(omega=[0.2] * 4), tol=1e-300,
                   max_outer=2)
A32 = O.assemble_anisotropic(0.01, 0.3, 32)
GF.solve_fns(A32, rng.standard_normal(31 * 31), G.WeightSchedule(omega=[0.5] * 8),
             GF.SpectralCorrection(0.01 * rng.standard_normal(31 * 31), 32), 8, tol=1e-300, max_iters=2)
H = O.assemble_helmholtz(2 * np.pi * 3, 32)
h = GM.build_hierarchy(H, 32, coarsest=8, schedules=G.WeightSchedule(
    omega=[0.8 / (8 * 32 * 32)] * 4, alpha=[0.3] * 4, variant="nag"))
fh = rng.standard_normal(H.shape[0]) + 1j * rng.standard_normal(H.shape[0])
GG.fgmres(H, fh, precond_apply=lambda r: h.apply(r), cfg=GG.FgmresConfig(restart=3, max_outer=1))
torch.cuda.synchronize()
print("sanitize probe done")

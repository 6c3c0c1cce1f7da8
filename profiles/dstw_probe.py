"""Lean DST kernels (csrc/dstw.cu) against the Stockham kernels (csrc/dst.cuh)
and scipy: parity at sides 511 / 1023 / 2047, device time of a plain dst2 and
of the cfg4 FNS alternation with either path (RG_DSTW read at plan creation)."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle as O  # noqa: E402
import paper_2412_08076_b200 as G  # noqa: E402
from paper_2412_08076_b200 import configs as CF  # noqa: E402
from paper_2412_08076_b200 import fns as GF  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def timed(fn, n=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


out = {}
for lean in (1, 0):
    os.environ["RG_DSTW"] = str(lean)
    GF._PLANS.clear()
    key = "lean" if lean else "stockham"
    res = {}
    for side in (511, 1023, 2047):
        x = np.random.default_rng(side).standard_normal((2, side * side))
        y = GF.dst2(x)
        res[f"dst2_rel_vs_scipy_{side}"] = max(rel(y[b], O.dst2(x[b])) for b in range(2))
        res[f"dst2_involution_{side}"] = rel(GF.dst2(y), x)
    xd = torch.randn(4, 1023 * 1023, dtype=torch.float64, device="cuda")
    res["dst2_4x1023_ms"] = timed(lambda: GF.dst2(xd))
    c = CF.cfg4()
    op = G.GpuStencilOperator.from_problems(c["problems"])
    eng = GF.FnsEngine(op, c["schedule"], GF.SpectralCorrection(c["lam"], 1024), c["M"])
    Fd = op.to_device(c["F"])
    eng.u[0].zero_()
    eng.cur = 0
    u1 = eng.step(Fd).clone()
    res["u1"] = u1
    res["alternation_ms"] = timed(lambda: eng.step(Fd))
    eng0 = GF.FnsEngine(op, c["schedule"], GF.SpectralCorrection(c["lam"], 1024), 0)
    eng0.u[0].copy_(u1)
    res["correction_only_ms"] = timed(lambda: eng0.step(Fd))
    out[key] = res
u_l, u_s = out["lean"].pop("u1"), out["stockham"].pop("u1")
out["alternation1_rel_lean_vs_stockham"] = float(torch.linalg.norm(u_l - u_s) / torch.linalg.norm(u_s))
c = CF.cfg4()
A0 = O.assemble_anisotropic(c["problems"][0].epsilon, c["problems"][0].theta, 1024)
uo = O.fns_lite_step(A0, c["F"][0], np.zeros(A0.shape[0]), np.asarray(c["schedule"].omega), c["M"],
                     c["lam"][0].cpu().numpy())
out["alternation1_rel_lean_vs_oracle_sys0"] = rel(u_l[0].cpu().numpy(), uo)
print(json.dumps(out, indent=1))

"""Size-independent digest of a full-size iterate, shared by
make_golden_full.py (which stores it) and tests/test_gpu_full.py (which
recomputes it for the GPU result): sha256 of the bytes (bitwise paths), the
2-norm and sum, 1024 seeded sampled entries and 4 projections onto seeded
N(0,1) vectors (tolerance paths)."""
from __future__ import annotations

import hashlib

import numpy as np

N_SAMPLE = 1024
N_PROJ = 4
SEED = 20241208


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def digest(u, prefix=""):
    u = np.ascontiguousarray(u)
    rng = np.random.default_rng(SEED)
    idx = np.sort(rng.choice(u.size, size=min(N_SAMPLE, u.size), replace=False))
    proj = []
    for _ in range(N_PROJ):
        g = rng.standard_normal(u.size)
        proj.append(np.vdot(g, u))
    return {f"{prefix}sha": sha(u), f"{prefix}norm": float(np.linalg.norm(u)),
            f"{prefix}sum": complex(u.sum()) if np.iscomplexobj(u) else float(u.sum()),
            f"{prefix}idx": idx, f"{prefix}sample": u[idx], f"{prefix}proj": np.array(proj)}

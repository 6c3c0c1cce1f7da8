"""Shared fixtures.  `-m gpu` tests need a B200 (run through gpurun); every
other test runs on the CPU in a few minutes."""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path(os.environ.get("RICHLAB_SRC", "/root/reference/pkg/src"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and librichgpu.so")
    config.addinivalue_line("markers", "reference: needs the reference package importable")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))
        return cache[name]
    return load


@pytest.fixture(scope="session")
def richlab():
    """The unmodified reference, only in the dev container."""
    if not (REFERENCE_SRC / "richlab").exists():
        pytest.skip("reference package not present (GPU box)")
    sys.path.insert(0, str(REFERENCE_SRC))
    import richlab as R
    return R


def sweep_case(d, i):
    """Unpack golden sweeps.npz case i."""
    k = f"c{i}_"
    return {key[len(k):]: (v.item() if v.ndim == 0 else v) for key, v in d.items()
            if key.startswith(k)}

"""ORACLE — TEST INFRASTRUCTURE ONLY.

A NumPy/SciPy restatement of the reference's hot path (richlab,
arXiv 2412.08076; /root/reference/pkg/src/richlab), used as the checker of
the GPU path.  Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline (`cpu_baseline` leg and `--impl reference`) may import it; the
product package never does, and fails loudly without its CUDA library.

Parity pinning: tests/golden/make_golden.py runs the unmodified reference
(imported from /root/reference in the dev container) on seeded inputs and
stores its outputs in tests/golden/*.npz; tests/test_oracle.py checks this
restatement against those fixtures bitwise (iterates, counts) and, when the
reference is importable, directly against it.
"""
from .richlab_port import *  # noqa: F401,F403

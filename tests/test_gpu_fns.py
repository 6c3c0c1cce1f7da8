"""FNS-lite (cfg 4 path): GPU DST-I and hybrid step vs the reference goldens.
The DST is an FFT, not pocketfft's: tolerance 1e-12 relative."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2412_08076_b200 as G
from paper_2412_08076_b200 import fns as GF

pytestmark = pytest.mark.gpu
RTOL = 1e-12


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


def test_dst2_golden(golden):
    d = golden("fns")
    assert _rel(GF.dst2(d["x31"]), d["d31"]) <= 1e-14
    assert _rel(GF.dst2(d["x63"]), d["d63"]) <= 1e-14


@pytest.mark.parametrize("side", [3, 7, 15, 255, 1023])
def test_dst2_vs_scipy_and_involution(side):
    rng = np.random.default_rng(side)
    x = rng.standard_normal((2, side * side))
    y = GF.dst2(x)
    for b in range(2):
        assert _rel(y[b], O.dst2(x[b])) <= 1e-13
    z = GF.dst2(y)
    assert _rel(z, x) <= 1e-13                       # involutory (transforms.py:33-35)
    assert abs(np.linalg.norm(y) / np.linalg.norm(x) - 1) <= 1e-13   # orthonormal


@pytest.mark.parametrize("side", [2047, 4095])
def test_dst2_large_fft_sizes(side):
    """M = 2048 (shared twiddles, 2 lines per CTA) and M = 4096 (global
    twiddle table, one line per CTA) against scipy's dstn."""
    x = np.random.default_rng(side).standard_normal(side * side)
    y = GF.dst2(x)
    assert _rel(y, O.dst2(x)) <= 1e-13


def test_dst2_largest_fft_size_properties():
    """M = 8192 (512-thread CTAs): involutory and orthonormal (no oracle call:
    size-independent properties, transforms.py:33-35)."""
    side = 8191
    x = torch.randn(side * side, dtype=torch.float64, device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(1))
    y = GF.dst2(x)
    assert abs(float(torch.linalg.norm(y) / torch.linalg.norm(x)) - 1) <= 1e-13
    assert float(torch.linalg.norm(GF.dst2(y) - x) / torch.linalg.norm(x)) <= 1e-13


@pytest.mark.parametrize("side", [1, 2, 5, 9, 14, 99, 300])
def test_dst2_dense_path_any_size(side):
    """side + 1 not a power of two: the dense sine-matrix path (the reference's
    pocketfft dstn takes any size, transforms.py:24-30)."""
    rng = np.random.default_rng(100 + side)
    x = rng.standard_normal((3, side * side))
    y = GF.dst2(x)
    for b in range(3):
        assert _rel(y[b], O.dst2(x[b])) <= 1e-13
    assert _rel(GF.dst2(y), x) <= 1e-13


@pytest.mark.parametrize("n", [20, 48])
def test_fns_step_dense_path(n):
    """fns_lite_step (fns.py:76-84) on a grid whose DST takes the dense path."""
    rng = np.random.default_rng(n)
    A = O.assemble_anisotropic(1e-2, 0.7, n)
    f = rng.standard_normal(A.shape[0])
    lam = 0.01 * rng.standard_normal(A.shape[0])
    w = np.full(4, 0.4)
    u = GF.fns_lite_step(A, f, np.zeros(A.shape[0]), G.WeightSchedule(omega=w), 4,
                         GF.SpectralCorrection(lam, n))
    uo = O.fns_lite_step(A, f, np.zeros(A.shape[0]), w, 4, lam)
    assert _rel(u, uo) <= RTOL


def test_sine_mode_is_unit_coefficient():
    """transforms.py:38-43 / test_transforms.py analogue."""
    n = 32
    i = np.arange(1, n)
    mode = np.outer(np.sin(3 * np.pi * i / n), np.sin(5 * np.pi * i / n)).reshape(-1)
    c = GF.dst2(mode)
    k = np.argmax(np.abs(c))
    assert k == 2 * (n - 1) + 4
    assert np.allclose(np.delete(c, k), 0, atol=1e-12)


def test_fns_step_and_solve_golden(golden):
    d = golden("fns")
    n = int(d["n"])
    A = O.assemble_anisotropic(float(d["eps"]), float(d["theta"]), n)
    corr = GF.SpectralCorrection(d["lam"], n)
    sch = G.WeightSchedule(omega=np.full(8, 0.5))
    u1 = GF.fns_lite_step(A, d["f"], np.zeros(A.shape[0]), sch, 8, corr)
    assert _rel(u1, d["u1"]) <= RTOL
    u, rep = GF.solve_fns(A, d["f"], sch, corr, 8, tol=1e-300, max_iters=5)
    assert rep.iterations == 5 and rep.inner_iterations == 40
    assert _rel(u, d["u5"]) <= RTOL
    assert np.all(np.abs(rep.trace - d["trace5"]) <= RTOL * d["trace5"])


def test_exact_inverse_correction(golden):
    """test_fns.py:31-40 / acceptance criterion 6: eps=1 operator, lambda =
    1/eigenvalue, zero smoothing -> one step solves the system."""
    d = golden("fns")
    A1 = O.assemble_anisotropic(1.0, 0.0, 16)
    u = GF.fns_lite_step(A1, d["f1"], np.zeros(A1.shape[0]), G.WeightSchedule(omega=[0.0]), 0,
                         GF.SpectralCorrection(d["lam1"], 16))
    assert _rel(u, d["u_exact"]) <= RTOL
    assert np.linalg.norm(d["f1"] - A1.dot(u)) <= 1e-12 * np.linalg.norm(d["f1"])


def test_lambda_zero_is_pure_smoothing():
    """test_fns.py:18-28: lambda = 0 reduces the step to M Richardson steps."""
    A = O.assemble_anisotropic(0.1, 0.7, 32)
    f = np.random.default_rng(1).standard_normal(A.shape[0])
    u = GF.fns_lite_step(A, f, np.zeros(A.shape[0]), G.WeightSchedule(omega=[0.3, 0.5]), 5,
                         GF.SpectralCorrection(np.zeros(A.shape[0]), 32))
    ref = np.zeros(A.shape[0])
    for k in range(5):
        ref = ref + [0.3, 0.5][k % 2] * (f - A.dot(ref))
    assert np.array_equal(u, ref)      # smoothing is bitwise; correction adds exact zeros


def test_full_size_fns_alternation():
    """cfg4 size (1023^2): one hybrid step vs the oracle."""
    rng = np.random.default_rng(4)
    A = O.assemble_anisotropic(1e-3, rng.uniform(0, np.pi), 1024)
    f = rng.standard_normal(A.shape[0])
    lam = 0.01 * rng.standard_normal(A.shape[0])
    w = np.full(8, 0.5)
    u = GF.fns_lite_step(A, f, np.zeros(A.shape[0]), G.WeightSchedule(omega=w), 8,
                         GF.SpectralCorrection(lam, 1024))
    uo = O.fns_lite_step(A, f, np.zeros(A.shape[0]), w, 8, lam)
    assert _rel(u, uo) <= RTOL


def test_nonfinite_raises():
    A = O.assemble_anisotropic(0.5, 0.3, 16)
    f = np.ones(A.shape[0])
    with pytest.raises(G.DivergenceError) as e:
        GF.solve_fns(A, f, G.WeightSchedule(omega=[1e308, 1e308]), GF.SpectralCorrection(
            np.zeros(A.shape[0]), 16), 4, max_iters=3)
    assert e.value.inner_iteration == 4


def test_solve_fns_batched_matches_per_system():
    """solve_fns_batched: every system follows its own solve_fns (fns.py:87-105)
    -- same counts, traces and iterates, each stopping on its own; a zero
    right-hand side converges at once."""
    rng = np.random.default_rng(21)
    n, B = 64, 4
    probs = [(10 ** rng.uniform(-2, 0), rng.uniform(0, np.pi)) for _ in range(B)]
    As = [O.assemble_anisotropic(e, t, n) for e, t in probs]
    op = G.GpuStencilOperator.stack([G.GpuStencilOperator.from_sparse(A) for A in As])
    F = rng.standard_normal((B, As[0].shape[0]))
    F[3] = 0.0
    lam = 0.02 * rng.standard_normal((B, As[0].shape[0]))
    sch = G.WeightSchedule(omega=np.full(4, 0.35))
    res = GF.solve_fns_batched(op, F, sch, GF.SpectralCorrection(lam, n), 4, tol=0.5, max_iters=30)
    its = []
    for b in range(B):
        u1, r1 = GF.solve_fns(As[b], F[b], sch, GF.SpectralCorrection(lam[b], n), 4, tol=0.5, max_iters=30)
        ub, rb = res[b]
        assert rb.iterations == r1.iterations and rb.converged == r1.converged, b
        assert np.allclose(rb.trace, r1.trace, rtol=1e-12, atol=0)
        assert np.linalg.norm(ub - u1) <= 1e-12 * max(np.linalg.norm(u1), 1e-300)
        its.append(rb.iterations)
    assert its[3] == 0


def test_sweep_norm_is_the_input_residual_norm():
    """rg_sweep_norm: the norm the first smoothing step reduces in its fused
    epilogue is ||f - A u0||^2 of the input iterate (fns.py:99 after a
    correction), on the wavefront path (8 systems at 255^2) and on the
    fallback paths (one system; a small grid), and the sweep itself is the
    plain rg_sweep (bitwise)."""
    import ctypes as C
    from paper_2412_08076_b200 import _lib as L
    from paper_2412_08076_b200.richardson import DeviceSchedule
    rng = np.random.default_rng(31)
    for n, B in ((256, 8), (256, 1), (48, 3)):
        As = [O.assemble_anisotropic(10 ** rng.uniform(-2, 0), rng.uniform(0, np.pi), n) for _ in range(B)]
        op = G.GpuStencilOperator.stack([G.GpuStencilOperator.from_sparse(A) for A in As])
        sch = DeviceSchedule(op, G.WeightSchedule(omega=np.full(8, 0.3)), None)
        U0 = torch.as_tensor(rng.standard_normal((B, op.P))).cuda()
        F = torch.as_tensor(rng.standard_normal((B, op.P))).cuda()
        outs = []
        for with_norm in (False, True):
            u0, u1 = U0.clone(), torch.empty_like(U0)
            n2 = torch.zeros(B, dtype=torch.float64, device="cuda")
            ob = C.c_int()
            if with_norm:
                L.check(op._lib.rg_sweep_norm(op.handle, C.byref(sch.struct), 0, 8, 0, L.ptr(u0), L.ptr(u1),
                                              None, None, L.ptr(F), L.ptr(n2), C.byref(ob), L.stream_ptr()))
            else:
                L.check(op._lib.rg_sweep(op.handle, C.byref(sch.struct), 0, 8, 0, L.ptr(u0), L.ptr(u1),
                                         None, None, L.ptr(F), C.byref(ob), L.stream_ptr()))
            outs.append(((u0, u1)[ob.value].clone(), n2.cpu().numpy()))
        assert torch.equal(outs[0][0], outs[1][0]), (n, B)
        for b in range(B):
            want = np.linalg.norm(F[b].cpu().numpy() - As[b] @ U0[b].cpu().numpy()) ** 2
            assert abs(outs[1][1][b] - want) <= 1e-12 * want, (n, B, b)

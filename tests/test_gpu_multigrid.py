"""V-cycle + FGMRES (cfg 5 path) vs the reference goldens and the oracle.
Transfers and smoothers are bitwise; the coarsest solve uses a precomputed
inverse instead of lu_solve, so V-cycle outputs agree to ~1e-15 and the
FGMRES residual history to 1e-12."""
import sys

import numpy as np
import pytest
import scipy.sparse as sp
import torch

import oracle as O
import paper_2412_08076_b200 as G
from paper_2412_08076_b200 import _lib as L
import paper_2412_08076_b200.fgmres  # noqa: E402,F401  (the package attribute is the function)
GG = sys.modules["paper_2412_08076_b200.fgmres"]
from paper_2412_08076_b200 import multigrid as GM

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


@pytest.mark.parametrize("n", [4, 8, 32, 256, 1024])
@pytest.mark.parametrize("dtype", [np.float64, np.complex128])
def test_transfers_bitwise(n, dtype):
    rng = np.random.default_rng(n)
    nf, nc = (n - 1) ** 2, (n // 2 - 1) ** 2
    x = rng.standard_normal((3, nf)).astype(dtype)
    e = rng.standard_normal((3, nc)).astype(dtype)
    u = rng.standard_normal((3, nf)).astype(dtype)
    if dtype == np.complex128:
        x += 1j * rng.standard_normal((3, nf))
        e += 1j * rng.standard_normal((3, nc))
    lib = L.load()
    code = L.RG_F64 if dtype == np.float64 else L.RG_C128
    td = torch.float64 if dtype == np.float64 else torch.complex128
    xd = torch.as_tensor(x).cuda()
    cd = torch.empty((3, nc), dtype=td, device="cuda")
    L.check(lib.rg_restrict(code, 3, n, L.ptr(xd), L.ptr(cd), L.stream_ptr()))
    R, P = O.restriction(n), O.prolongation(n)
    got = cd.cpu().numpy()
    for b in range(3):
        assert np.array_equal(got[b], R.dot(x[b]))
    ud = torch.as_tensor(u).cuda()
    L.check(lib.rg_prolong_add(code, 3, n, L.ptr(torch.as_tensor(e).cuda()), L.ptr(ud),
                               L.stream_ptr()))
    got = ud.cpu().numpy()
    for b in range(3):
        assert np.array_equal(got[b], u[b] + P.dot(e[b]))


def _sched(n):
    return G.WeightSchedule(omega=np.full(4, 0.8 / (8 * n * n)), alpha=np.full(4, 0.3),
                            variant="nag")


def test_vcycle_golden(golden):
    d = golden("multigrid")
    n = int(d["n"])
    A = O.assemble_helmholtz(float(d["omega_phys"]), n)
    h = GM.build_hierarchy(A, n, coarsest=8, schedules=_sched(n))
    assert h.depth == d["depth"]
    assert h.levels[0].op.kind == L.RG_DIAG5 and h.levels[1].op.kind == L.RG_VAR9
    u = GM.v_cycle(h, d["f"])
    assert _rel(u, d["u"]) <= 1e-13


def test_fgmres_vcycle_golden(golden):
    d = golden("multigrid")
    n = int(d["n"])
    A = O.assemble_helmholtz(float(d["omega_phys"]), n)
    h = GM.build_hierarchy(A, n, coarsest=8, schedules=_sched(n))
    op = G.GpuStencilOperator.from_sparse(A)
    u, rep = GG.fgmres(op, d["f"], precond_apply=lambda r: h.apply(r),
                       cfg=GG.FgmresConfig(restart=5, tol=1e-6, max_outer=4))
    assert rep.iterations == d["fg_iterations"]
    assert rep.converged == bool(d["fg_converged"]) and rep.stagnated == bool(d["fg_stagnated"])
    assert np.all(np.abs(rep.trace - d["fg_trace"]) <= 1e-12 * np.abs(d["fg_trace"]) + 1e-15)
    assert _rel(u, d["fg_u"]) <= 1e-11


def test_vcycle_vs_oracle_larger_and_batched():
    """n = 128 Helmholtz, depth 4, two right-hand sides through one shared
    hierarchy; each equals the oracle's single-system V-cycle."""
    n = 128
    A = O.assemble_helmholtz(2 * np.pi * n / 10, n)
    sched = _sched(n)
    h = GM.build_hierarchy(A, n, coarsest=16, schedules=sched, batch=2)
    levels, lu = O.build_hierarchy(A, n, coarsest=16)
    rng = np.random.default_rng(7)
    F = rng.standard_normal((2, A.shape[0])) + 1j * rng.standard_normal((2, A.shape[0]))
    U = h.apply(torch.as_tensor(F).cuda()).cpu().numpy()
    sd = dict(omega=sched.omega, alpha=sched.alpha, alpha_tilde=sched.alpha_tilde, variant="nag")
    for b in range(2):
        assert _rel(U[b], O.v_cycle(levels, lu, F[b], sd)) <= 1e-13


def test_vcycle_vs_oracle_every_smoother_kind():
    """n = 512 Helmholtz, depth 6: the blocked Galerkin smoother on 511^2 and
    255^2, the resident cluster sweeps on 127^2 (operator rows in shared
    memory), 63^2 and 31^2; equals the oracle's V-cycle."""
    n = 512
    A = O.assemble_helmholtz(2 * np.pi * n / 10, n)
    sched = _sched(n)
    h = GM.build_hierarchy(A, n, coarsest=16, schedules=sched, batch=1)
    levels, lu = O.build_hierarchy(A, n, coarsest=16)
    rng = np.random.default_rng(9)
    f = rng.standard_normal(A.shape[0]) + 1j * rng.standard_normal(A.shape[0])
    u = h.apply(torch.as_tensor(f[None]).cuda()).cpu().numpy()[0]
    sd = dict(omega=sched.omega, alpha=sched.alpha, alpha_tilde=sched.alpha_tilde, variant="nag")
    assert _rel(u, O.v_cycle(levels, lu, f, sd)) <= 1e-13


def test_fgmres_plain_matches_oracle():
    """Unpreconditioned restarted FGMRES(10) on a real anisotropic system, 188
    Arnoldi steps: the dot products are not BLAS-bitwise, and the restarted
    recurrence amplifies last-bit differences to ~1e-9 by the end."""
    A = O.assemble_anisotropic(0.1, 0.4, 24)
    f = np.random.default_rng(3).standard_normal(A.shape[0])
    u, rep = GG.fgmres(A, f, cfg=GG.FgmresConfig(restart=10, tol=1e-8, max_outer=20))
    uo, ro = O.fgmres(A, f, lambda r: r, restart=10, tol=1e-8, max_outer=20)
    assert rep.iterations == ro["iterations"]
    assert np.allclose(rep.trace, ro["trace"], rtol=1e-7, atol=0)
    assert _rel(u, uo) <= 1e-7


def _csweep(op, variant, n_steps, block_T, f, u0, v0, seed=0, P=None, lam=None):
    """rg_sweep on a stencil operator, returns (u, v) on the host."""
    import ctypes as C
    m = 4
    rng = np.random.default_rng(seed)
    lam = 8.0 * op.side ** 2 if lam is None else lam
    w = rng.uniform(0.2, 0.9, m) / lam
    kw = {} if variant == "plain" else {"alpha": np.full(m, 0.35)}
    from paper_2412_08076_b200.richardson import DeviceSchedule
    sch = DeviceSchedule(op, G.WeightSchedule(omega=w, variant=variant, **kw), P)
    dev = op.device
    t = lambda a: torch.as_tensor(a).to(dev).clone()
    u = [t(u0), torch.empty_like(t(u0))]
    v = [t(v0), torch.empty_like(t(v0))]
    fd = t(f)
    outb = C.c_int()
    L.check(L.load().rg_sweep(op.handle, C.byref(sch.struct), 0, n_steps, block_T,
                             L.ptr(u[0]), L.ptr(u[1]), L.ptr(v[0]), L.ptr(v[1]), L.ptr(fd),
                             C.byref(outb), L.stream_ptr()))
    torch.cuda.synchronize()
    return u[outb.value].cpu().numpy(), v[outb.value].cpu().numpy()


@pytest.mark.parametrize("n", [9, 101, 258])
@pytest.mark.parametrize("variant", ["plain", "mom", "nag"])
def test_complex_blocked_sweep_bitwise(n, variant):
    """The temporally blocked complex 5-point sweep (cblock.cuh, the V-cycle
    fine-level smoother) gives the one-step kernel's bits at every depth."""
    A = O.assemble_helmholtz(12.0, n)
    B = 3
    op = G.GpuStencilOperator.from_sparse(A).broadcast(B)
    rng = np.random.default_rng(n)
    P = A.shape[0]
    cplx = lambda: rng.standard_normal((B, P)) + 1j * rng.standard_normal((B, P))
    f, u0 = cplx(), cplx()
    v0 = cplx() if variant != "plain" else np.zeros((B, P), complex)
    ref = _csweep(op, variant, 11, 1, f, u0, v0)
    for T in (0, 2, 3, 4):
        got = _csweep(op, variant, 11, T, f, u0, v0)
        assert np.array_equal(got[0], ref[0]), (T, np.abs(got[0] - ref[0]).max())
        if variant != "plain":
            assert np.array_equal(got[1], ref[1])
    # and the one-step path is the CSR loop of the reference (system 1)
    s = G.WeightSchedule(omega=np.random.default_rng(0).uniform(0.2, 0.9, 4) / (8.0 * op.side ** 2),
                         variant=variant, **({} if variant == "plain" else {"alpha": np.full(4, 0.35)}))
    if variant != "plain":
        return
    x = u0[1].copy()
    for k in range(11):
        x = x + s.omega[k % 4] * (f[1] - A @ x)
    assert np.array_equal(ref[0][1], x)


@pytest.mark.parametrize("n", [64, 256])
@pytest.mark.parametrize("variant", ["plain", "mom", "nag"])
def test_complex_galerkin_blocked_sweep_bitwise(n, variant):
    """The blocked 9-point complex sweep of the Galerkin levels (repeated
    stencil + band planes, cblock9_kernel) gives the one-step kernel's bits."""
    H = O.assemble_helmholtz(2 * np.pi * n / 10, n)
    levels, _ = O.build_hierarchy(H, n, coarsest=8)
    Ac = levels[1]["A"]
    B = 3
    op = G.GpuStencilOperator.from_sparse(Ac).broadcast(B)
    assert op.kind == 3
    rng = np.random.default_rng(n + 1)
    P = Ac.shape[0]
    cplx = lambda: rng.standard_normal((B, P)) + 1j * rng.standard_normal((B, P))  # noqa: E731
    f, u0 = cplx(), cplx()
    v0 = cplx() if variant != "plain" else np.zeros((B, P), complex)
    ref = _csweep(op, variant, 9, 1, f, u0, v0)
    for T in (0, 2, 3, 4):
        got = _csweep(op, variant, 9, T, f, u0, v0)
        assert np.array_equal(got[0], ref[0]), (T, np.abs(got[0] - ref[0]).max())
        if variant != "plain":
            assert np.array_equal(got[1], ref[1])



@pytest.mark.parametrize("variant", ["plain", "mom", "nag"])
@pytest.mark.parametrize("pre", [None, "field"])
def test_small_grid_resident_sweep_bitwise(variant, pre):
    """Small grids run every step in one cluster-resident launch
    (psweep_kernel): same bits as the one-step kernel, real VAR9 and DIAG5
    operators, with and without a per-node Jacobi scale."""
    import scipy.sparse as sp
    rng = np.random.default_rng(17)
    A = O.assemble_anisotropic(0.1, 0.7, 24)
    A9 = (sp.diags(rng.uniform(0.5, 1.5, A.shape[0])) @ A).tocsr()        # VAR9
    H = O.assemble_helmholtz(20.0, 40)
    A5 = sp.csr_matrix((H.data.real.copy(), H.indices, H.indptr), shape=H.shape)   # real DIAG5
    for M in (A9, A5):
        B = 2
        op = G.GpuStencilOperator.from_sparse(M).broadcast(B)
        P = None
        if pre == "field":
            P = G.JacobiScale((2.0 / 3.0) / M.diagonal())
        n = M.shape[0]
        f, u0 = rng.standard_normal((B, n)), rng.standard_normal((B, n))
        v0 = rng.standard_normal((B, n)) if variant != "plain" else np.zeros((B, n))
        lam = np.abs(M.diagonal()).max() * 2.5
        ref = _csweep(op, variant, 7, 1, f, u0, v0, P=P, lam=lam)
        got = _csweep(op, variant, 7, 0, f, u0, v0, P=P, lam=lam)
        assert np.array_equal(got[0], ref[0])
        if variant != "plain":
            assert np.array_equal(got[1], ref[1])

"""Gauss-Seidel / SOR / SSOR on the device (precond.py:79-118, SURVEY.md
§8(f) item 1) vs the reference's outputs (tests/golden/precond.npz) and the
oracle.  The wavefront substitutions round differently from SuperLU's
(which stores L pre-divided by the diagonal), so the bar is the reference's
own for these maps: 1e-13 relative (test_precond.py:33-62); preconditioned
solves then match iteration counts exactly, iterates to 1e-10 and traces
to 1e-10 relative (1e-12 of trace[0] near the residual's rounding floor)."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2412_08076_b200 as G
from paper_2412_08076_b200.errors import DivergenceError

pytestmark = pytest.mark.gpu

KINDS = {"gs": ("gauss-seidel", 1.0), "sor14": ("sor", 1.4), "ssor10": ("ssor", 1.0),
         "ssor13": ("ssor", 1.3)}


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _close_trace(got, want):
    """Relative residuals agree to 1e-10 relative, or 1e-12 of trace[0] once
    they approach the rounding floor of the residual itself."""
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape
    assert np.all(np.abs(got - want) <= 1e-10 * want + 1e-12 * want[0]), \
        np.max(np.abs(got - want) / want)


def _gpu_pre(A, kind, relax):
    return {"gauss-seidel": lambda: G.Preconditioner.gauss_seidel(A),
            "sor": lambda: G.Preconditioner.sor(A, relax),
            "ssor": lambda: G.Preconditioner.ssor(A, relax)}[kind]()


class _RefLike:
    """Duck-typed stand-in for a richlab Preconditioner (kind, relax, apply)."""

    def __init__(self, A, kind, relax):
        self.kind, self.relax = kind, (None if kind == "gauss-seidel" else relax)
        self._f = O.tri_precond(A, kind, relax)

    def apply(self, r):
        return self._f(r)


def test_apply_matches_reference(golden):
    d = golden("precond")
    for k in range(int(d["n_apply"])):
        A = O.assemble_anisotropic(float(d[f"a{k}_eps"]), float(d[f"a{k}_theta"]),
                                   int(d[f"a{k}_n"]))
        for name, (kind, relax) in KINDS.items():
            z = _gpu_pre(A, kind, relax).apply(d[f"a{k}_r"])
            assert _rel(z, d[f"a{k}_{name}"]) <= 1e-13, (k, name, _rel(z, d[f"a{k}_{name}"]))


def test_apply_dense_oracle():
    """The reference's own known answers (test_precond.py:33-62) on a grid."""
    rng = np.random.default_rng(3)
    A = O.assemble_anisotropic(0.3, 0.7, 8)
    Ad = A.toarray()
    D = np.diag(np.diag(Ad))
    Lo, Up = -np.tril(Ad, -1), -np.triu(Ad, 1)
    r = rng.standard_normal(A.shape[0])
    a = 1.3
    ref = {"gs": np.linalg.solve(D - Lo, r), "sor14": 1.4 * np.linalg.solve(D - 1.4 * Lo, r),
           "ssor13": a * (2 - a) * np.linalg.solve(D - a * Up, D @ np.linalg.solve(D - a * Lo, r))}
    for name, want in ref.items():
        kind, relax = KINDS[name]
        assert _rel(_gpu_pre(A, kind, relax).apply(r), want) <= 1e-13


@pytest.mark.parametrize("n", [64, 256, 1024, 1500])
def test_apply_large_vs_oracle(n):
    """Full-size grids (one pass of 1023 rows; 1499 rows = two passes)."""
    rng = np.random.default_rng(n)
    A = O.assemble_anisotropic(10 ** rng.uniform(-3, 0), rng.uniform(0, np.pi), n)
    r = rng.standard_normal(A.shape[0])
    for kind, relax in (("sor", 1.7), ("ssor", 1.0)):
        z = _gpu_pre(A, kind, relax).apply(r)
        zo = O.tri_precond(A, kind, relax)(r)
        assert _rel(z, zo) <= 1e-13, (kind, _rel(z, zo))


def test_apply_batched_and_f32():
    rng = np.random.default_rng(7)
    As = [O.assemble_anisotropic(10 ** rng.uniform(-3, 0), rng.uniform(0, np.pi), 40)
          for _ in range(3)]
    op = G.GpuStencilOperator.stack([G.GpuStencilOperator.from_sparse(A) for A in As])
    R = rng.standard_normal((3, As[0].shape[0]))
    Z = G.TriangularPreconditioner(op, "ssor", 1.2).apply(R)
    for b in range(3):
        assert _rel(Z[b], O.tri_precond(As[b], "ssor", 1.2)(R[b])) <= 1e-13
    op32 = G.GpuStencilOperator.from_sparse(As[0], dtype=np.float32)
    z32 = G.TriangularPreconditioner(op32, "sor", 1.4).apply(R[0].astype(np.float32))
    assert z32.dtype == np.float32
    assert _rel(z32, O.tri_precond(As[0], "sor", 1.4)(R[0])) <= 1e-5


def test_solves_match_reference(golden):
    d = golden("precond")
    for k in range(int(d["n_solve"])):
        g = lambda key: d[f"s{k}_{key}"]  # noqa: E731
        A = O.assemble_anisotropic(float(g("eps")), float(g("theta")), int(g("n")))
        sch = G.WeightSchedule(omega=g("omega"), alpha=g("alpha"), alpha_tilde=g("alpha_tilde"),
                               variant=str(g("variant")))
        for P in (_gpu_pre(A, str(g("kind")), float(g("relax"))),
                  _RefLike(A, str(g("kind")), float(g("relax")))):
            if int(g("diverged")) >= 0:
                with pytest.raises(DivergenceError) as e:
                    G.solve_stationary(A, g("f"), sch, P=P, tol=float(g("tol")), max_outer=60)
                assert e.value.inner_iteration == int(g("diverged"))
                continue
            u, rep = G.solve_stationary(A, g("f"), sch, P=P, tol=float(g("tol")), max_outer=60)
            assert rep.iterations == int(g("iterations")), k
            assert rep.inner_iterations == int(g("inner"))
            assert rep.converged == bool(g("converged"))
            _close_trace(rep.trace, g("trace"))
            assert _rel(u, g("u")) <= 1e-10


def test_inner_check_batched_and_sweeps():
    rng = np.random.default_rng(9)
    As = [O.assemble_anisotropic(10 ** rng.uniform(-2, 0), rng.uniform(0, np.pi), 20)
          for _ in range(3)]
    F = rng.standard_normal((3, As[0].shape[0]))
    w = np.array([0.9, 1.2, 1.0])
    sch = G.WeightSchedule(omega=w, alpha=np.full(3, 0.3), variant="nag")
    op = G.GpuStencilOperator.stack([G.GpuStencilOperator.from_sparse(A) for A in As])
    res = G.solve_stationary_batched(op, F, sch, P=_RefLike(As[0], "ssor", 1.1), tol=1e-9,
                                     max_outer=400, check="inner")
    for b in range(3):
        pre = O.tri_precond(As[b], "ssor", 1.1)
        uo, ro = O.solve_stationary(As[b], F[b], w, sch.alpha, sch.alpha_tilde, "nag", scale=pre,
                                    tol=1e-9, max_outer=400, check="inner")
        u, rep = res[b]
        assert rep.iterations == ro["iterations"] and rep.inner_iterations == ro["inner_iterations"]
        assert rep.converged == ro["converged"]
        assert _rel(u, uo) <= 1e-10
        _close_trace(rep.trace, ro["trace"])
    # outer_sweep / inner_update with the same map
    A, f = As[0], F[0]
    P = G.Preconditioner.ssor(A, 1.1)
    st = G.IterationState.start(A.shape[0])
    G.outer_sweep(A, f, st, sch, P=P)
    uo, vo, nr = O.outer_sweep(A, f, np.zeros(A.shape[0]), np.zeros(A.shape[0]), w, sch.alpha,
                               sch.alpha_tilde, "nag", scale=O.tri_precond(A, "ssor", 1.1))
    assert _rel(st.u, uo) <= 1e-12 and _rel(st.v, vo) <= 1e-12
    assert abs(st.residual_history[-1] - nr) <= 1e-12 * nr


def test_device_tensors_and_errors():
    A = O.assemble_anisotropic(0.1, 0.3, 16)
    P = G.Preconditioner.sor(A, 1.5)
    r = torch.randn(A.shape[0], dtype=torch.float64, device="cuda")
    z = P.apply(r)
    assert z.is_cuda and _rel(z.cpu().numpy(), O.tri_precond(A, "sor", 1.5)(r.cpu().numpy())) <= 1e-13
    with pytest.raises(ValueError):
        G.Preconditioner.sor(A, 2.0)
    with pytest.raises(ValueError):
        G.Preconditioner.ssor(A, 0.0)
    # a zero diagonal entry is refused (precond.py:83-84 ZeroDiagonalError)
    import scipy.sparse as sp
    Z = sp.csr_matrix(O.assemble_anisotropic(0.3, 0.2, 8)).tolil()
    Z[5, 5] = 0.0
    with pytest.raises(ValueError):
        G.Preconditioner.ssor(sp.csr_matrix(Z))


def test_apply_transpose_matches_dense_transpose():
    """B^{-T} on a non-symmetric constant stencil (anisotropic + a constant
    convection term) equals the transpose of the assembled B^{-1}
    (test_precond.py:66-72: 1e-12)."""
    import scipy.sparse as sp
    n = 10
    A = O.assemble_anisotropic(0.2, 0.6, n).tolil()
    s = n - 1
    for i in range(s):
        for j in range(s):
            k = i * s + j
            if j + 1 < s:
                A[k, k + 1] += 0.3
            if j > 0:
                A[k, k - 1] -= 0.3
    A = sp.csr_matrix(A)
    op = G.GpuStencilOperator.from_sparse(A)
    assert op.kind == 1
    for P in (G.Preconditioner.sor(op, 1.2), G.Preconditioner.ssor(op, 0.9),
              G.Preconditioner.gauss_seidel(op)):
        E = np.eye(A.shape[0])
        Bm = np.column_stack([P.apply(e) for e in E])
        Bt = np.column_stack([P.apply_transpose(e) for e in E])
        assert np.abs(Bt - Bm.T).max() <= 1e-12
        kind = "gauss-seidel" if P.kind == "gauss-seidel" else P.kind
        ref = np.column_stack([O.tri_precond(A, kind, P._relax)(e) for e in E])
        assert np.abs(Bm - ref).max() <= 1e-13


def _variable_real(n, seed, amp=0.3):
    """Non-symmetric real 9-point operator with per-node coefficients."""
    import scipy.sparse as sp
    rng = np.random.default_rng(seed)
    A = O.assemble_anisotropic(0.2, 0.6, n).tocsr().astype(np.float64)
    A.data = A.data * (1.0 + amp * rng.random(A.nnz))
    return sp.csr_matrix(A)


def _general_cases():
    H = O.assemble_helmholtz(2 * np.pi * 16 / 10, 16)                  # DIAG5 complex128
    levels, _ = O.build_hierarchy(O.assemble_helmholtz(2 * np.pi * 32 / 10, 32), 32, coarsest=8)
    return {"var9_real": (_variable_real(14, 1), 3), "diag5_c128": (H.tocsr(), 2),
            "var9_c128": (levels[1]["A"].tocsr(), 3)}


@pytest.mark.parametrize("case", ["var9_real", "diag5_c128", "var9_c128"])
def test_general_operators_match_oracle_and_transpose(case):
    """precond.py:86-118 builds GS/SOR/SSOR for any SparseMatrix: per-node
    coefficients and complex scalars (csrc/trigen.cuh) against the oracle's
    SuperLU substitutions (1e-13) and the transposed maps against the
    assembled B^{-1} (test_precond.py:66-72)."""
    A, kind_id = _general_cases()[case]
    op = G.GpuStencilOperator.from_sparse(A)
    assert op.kind == kind_id
    rng = np.random.default_rng(5)
    N = A.shape[0]
    r = rng.standard_normal(N)
    if np.iscomplexobj(A.data):
        r = r + 1j * rng.standard_normal(N)
    for kind, relax in (("gauss-seidel", 1.0), ("sor", 1.4), ("ssor", 1.0), ("ssor", 0.8)):
        P = _gpu_pre(op, kind, relax)
        assert _rel(P.apply(r), O.tri_precond(A, kind, relax)(r)) <= 1e-13, (case, kind)
    if N <= 400:
        for P in (G.Preconditioner.sor(op, 1.2), G.Preconditioner.ssor(op, 0.9)):
            E = np.eye(N, dtype=A.dtype)
            Bm = np.column_stack([P.apply(e) for e in E])
            Bt = np.column_stack([P.apply_transpose(e) for e in E])
            assert np.abs(Bt - Bm.T).max() <= 1e-12 * np.abs(Bm).max()


def test_general_operator_large_and_solve():
    """A 1023^2 Galerkin-type variable operator (two passes need side > 1024:
    1500 cells) and an SSOR-preconditioned solve on a variable operator with
    the oracle's counts."""
    A = _variable_real(1501, 2)
    op = G.GpuStencilOperator.from_sparse(A)
    assert op.kind == 3
    r = np.random.default_rng(3).standard_normal(A.shape[0])
    for kind, relax in (("sor", 1.5), ("ssor", 1.1)):
        assert _rel(_gpu_pre(op, kind, relax).apply(r), O.tri_precond(A, kind, relax)(r)) <= 1e-13
    A2 = _variable_real(24, 4, amp=0.1)
    f = np.random.default_rng(6).standard_normal(A2.shape[0])
    sch = G.WeightSchedule(omega=np.array([1.0, 0.9]))
    u, rep = G.solve_stationary(A2, f, sch, P=G.Preconditioner.ssor(A2, 1.0), tol=1e-8, max_outer=400)
    uo, ro = O.solve_stationary(A2, f, sch.omega, scale=O.tri_precond(A2, "ssor", 1.0), tol=1e-8,
                                max_outer=400)
    assert rep.iterations == ro["iterations"] and rep.converged
    assert _rel(u, uo) <= 1e-10


@pytest.mark.parametrize("n", [2, 3, 4, 5, 17, 32, 33, 34, 64, 65, 66, 97, 128, 129, 130, 193, 257])
def test_apply_small_and_boundary_sizes(n):
    """Grid sides around every warp / CTA / cluster boundary of the wavefront
    kernel (1 .. 256 rows: 1 to 4 CTAs of 64 rows, partial warps, one-row
    grids), SOR / SSOR and the transposed maps, two systems."""
    rng = np.random.default_rng(100 + n)
    As = [O.assemble_anisotropic(10 ** rng.uniform(-2, 0), rng.uniform(0, np.pi), n) for _ in range(2)]
    op = G.GpuStencilOperator.stack([G.GpuStencilOperator.from_sparse(A) for A in As])
    R = rng.standard_normal((2, As[0].shape[0]))
    for kind, relax in (("sor", 1.6), ("ssor", 0.9)):
        P = G.TriangularPreconditioner(op, kind, relax)
        Z = P.apply(R)
        Zt = P.apply_transpose(R)
        for b in range(2):
            f = O.tri_precond(As[b], kind, relax)
            assert _rel(Z[b], f(R[b])) <= 1e-13, (n, kind, b)
            if As[b].shape[0] > 1200:
                continue
            # B^{-T} r from dense transposed solves (small grids only)
            Ad = As[b].toarray()
            D = np.diag(np.diag(Ad))
            Lo, Up = np.tril(Ad, -1), np.triu(Ad, 1)
            if kind == "sor":
                want = relax * np.linalg.solve((D + relax * Lo).T, R[b])
            else:
                c = relax * (2 - relax)
                want = c * np.linalg.solve((D + relax * Lo).T, D @ np.linalg.solve((D + relax * Up).T, R[b]))
            assert _rel(Zt[b], want) <= 1e-12, (n, kind, b, "transpose")

"""GpuStencilOperator: the structured-grid matrix the solve loop applies.

Duck-types the reference SparseMatrix (sparse.py:13-133) as the solvers see
it -- `matvec`, `rmatvec`, `diagonal`, `ncols`, `nrows`, `shape`, `dtype`
(richardson.py:92-93,105,119,124; precond.py:73) -- but holds only stencil
data on the GPU:

  CONST9  9 coefficients per system   (anisotropic FEM, problems.py:121-154)
  DIAG5   4 off-diagonals + diagonal  (damped Helmholtz, problems.py:174-200)
  VAR9    9 coefficient planes        (Galerkin coarse levels, multigrid.py:62-68)

`from_sparse` extracts and validates the stencil from an assembled CSR
matrix (values copied bit for bit); `from_problems`
builds it directly from problem specs without assembling a CSR.
A batched operator holds B independent systems of the same side and kind.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib as L
from .errors import DimensionMismatch, UnsupportedOperator, ZeroDiagonalError
from .problems import (OFFSETS9, AnisotropicProblem, HelmholtzProblem, anisotropic_stencil,
                       helmholtz_stencil)

_DTYPES = {
    np.dtype(np.float32): (L.RG_F32, torch.float32),
    np.dtype(np.float64): (L.RG_F64, torch.float64),
    np.dtype(np.complex128): (L.RG_C128, torch.complex128),
}
_KIND_NAMES = {L.RG_CONST9: "const9", L.RG_DIAG5: "diag5", L.RG_VAR9: "var9"}


def default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2412_08076_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _csr_arrays(A):
    """(nrows, ncols, indptr, indices, data) of a richlab SparseMatrix or any
    scipy sparse matrix."""
    if hasattr(A, "row_starts") and hasattr(A, "col_indices"):
        return A.nrows, A.ncols, np.asarray(A.row_starts), np.asarray(A.col_indices), np.asarray(A.values)
    import scipy.sparse as sp
    csr = sp.csr_matrix(A)
    return csr.shape[0], csr.shape[1], csr.indptr, csr.indices, csr.data


def extract_planes(A):
    """Scatter a CSR matrix on an s x s interior grid into 9 coefficient
    planes [9, s*s] (CSR column order), zero where the CSR has no entry.
    Raises UnsupportedOperator if an entry lies outside the 3x3
    neighbourhood or the matrix is not square on a square grid."""
    nrows, ncols, indptr, indices, data = _csr_arrays(A)
    if nrows != ncols:
        raise UnsupportedOperator(f"matrix is {nrows}x{ncols}, not square")
    s = math.isqrt(nrows)
    if s * s != nrows:
        raise UnsupportedOperator(f"{nrows} unknowns is not a square interior grid")
    rows = np.repeat(np.arange(nrows, dtype=np.int64), np.diff(indptr))
    ix, iy = np.divmod(rows, s)
    jx, jy = np.divmod(np.asarray(indices, dtype=np.int64), s)
    dx, dy = jx - ix, jy - iy
    if np.any(np.abs(dx) > 1) or np.any(np.abs(dy) > 1):
        raise UnsupportedOperator("entries outside the 3x3 grid neighbourhood")
    q = (dx + 1) * 3 + (dy + 1)
    planes = np.zeros((9, nrows), dtype=data.dtype)
    planes[q, rows] = data
    present = np.zeros((9, nrows), dtype=bool)
    present[q, rows] = True
    return s, planes, present


def _neighbour_mask(s):
    """mask[q, i]: neighbour q of node i lies inside the s x s interior."""
    i = np.arange(s * s)
    x, y = np.divmod(i, s)
    m = np.zeros((9, s * s), dtype=bool)
    for q, (dx, dy) in enumerate(OFFSETS9):
        m[q] = (x + dx >= 0) & (x + dx < s) & (y + dy >= 0) & (y + dy < s)
    return m


def classify(s, planes, present):
    """Pick the cheapest exact representation: ('const9', c[9]),
    ('diag5', (off[4], diag[P])) or ('var9', planes)."""
    inside = _neighbour_mask(s)
    if np.any(present & ~inside):
        raise UnsupportedOperator("entry couples to a node outside the grid")
    # constant stencil: every in-grid neighbour carries the same value
    c = np.zeros(9, dtype=planes.dtype)
    for q in range(9):
        vals = planes[q][inside[q]]
        if vals.size:
            c[q] = vals[0]
    expect = np.where(inside, c[:, None], 0)
    if np.array_equal(planes, expect) and np.array_equal(
            np.signbit(planes.real), np.signbit(np.asarray(expect).real)):
        return "const9", c
    five = [1, 3, 5, 7]
    corners = [0, 2, 6, 8]
    if not np.any(present[corners]):
        off = c[five]
        expect5 = np.where(inside[five], off[:, None], 0)
        if np.array_equal(planes[five], expect5):
            return "diag5", (off, planes[4].copy())
    return "var9", planes


class JacobiScale:
    """Weighted-Jacobi map r -> scale * r (precond.py:71-77), scale = relax / diag."""

    def __init__(self, scale):
        self.scale = np.asarray(scale)

    @classmethod
    def weighted_jacobi(cls, A, relax=2.0 / 3.0):
        """precond.py:71-77.  For a batched GpuStencilOperator whose systems
        carry their own coefficients this returns one JacobiScale per system
        (a list, accepted as `P` by every batched entry point): system b is
        scaled by its own diagonal, never system 0's."""
        if isinstance(A, GpuStencilOperator) and A.batch > 1 and not A.shared:
            return [cls._from_diag(A.diagonal(b), relax) for b in range(A.batch)]
        return cls._from_diag(A.diagonal(), relax)

    @classmethod
    def _from_diag(cls, diag, relax):
        diag = np.asarray(diag)
        zero = np.nonzero(diag == 0)[0]
        if len(zero):
            raise ZeroDiagonalError(int(zero[0]))
        return cls(relax / diag)

    def apply(self, r):
        return self.scale * np.asarray(r)


_SCALE_MEMO = {}


def precond_scale(P, n):
    """Jacobi scale of a preconditioner (ours or richlab's): a 0-d array when
    it is one constant, else a length-n array; None for P=None.  richlab
    hides the scale in a closure; P.apply(ones) returns it exactly
    (scale * 1.0 == scale).  Results are memoised per preconditioner object."""
    if P is None:
        return None
    key = (id(P), n)
    hit = _SCALE_MEMO.get(key)
    if hit is not None and hit[0] is P:
        return hit[1]
    if isinstance(P, JacobiScale):
        s = P.scale
    elif getattr(P, "kind", None) in ("weighted-jacobi", "identity"):
        s = np.asarray(P.apply(np.ones(n)))
    else:
        raise UnsupportedOperator(
            f"preconditioner kind {getattr(P, 'kind', None)!r} has no GPU path (weighted "
            "Jacobi only; GS/SOR/SSOR are SURVEY.md §8(f) next items)")
    if s.ndim == 1 and s.size and np.all(s == s[0]):
        s = np.asarray(s[0])
    if len(_SCALE_MEMO) > 256:
        _SCALE_MEMO.clear()
    _SCALE_MEMO[key] = (P, s)
    return s


def as_numpy_dtype(dt):
    if isinstance(dt, torch.dtype):
        return {torch.float32: np.dtype(np.float32), torch.float64: np.dtype(np.float64),
                torch.complex128: np.dtype(np.complex128)}[dt]
    return np.dtype(dt)


class GpuStencilOperator:
    """A batch of B structured-grid operators resident on the GPU."""

    def __init__(self, kind, side, stencil, diag=None, dtype=np.float64, device=None, batch=None):
        """stencil/diag hold one coefficient set per system ([B, ...]); with
        `batch` > len(stencil) == 1 the single set is shared by `batch`
        systems (several right-hand sides of one operator)."""
        self.device = torch.device(device) if device is not None else default_device()
        self.np_dtype = as_numpy_dtype(dtype)
        if self.np_dtype not in _DTYPES:
            raise ValueError(f"unsupported dtype {self.np_dtype}")
        self.rg_dtype, self.torch_dtype = _DTYPES[self.np_dtype]
        self.kind = {"const9": L.RG_CONST9, "diag5": L.RG_DIAG5, "var9": L.RG_VAR9}[kind]
        self.side = int(side)
        self.P = self.side * self.side
        st = np.asarray(stencil)
        self.nsets = st.shape[0]
        self.batch = int(batch) if batch is not None else self.nsets
        self.shared = self.nsets == 1 and self.batch > 1
        if self.nsets != self.batch and not self.shared:
            raise DimensionMismatch(f"{self.nsets} coefficient sets for {self.batch} systems")
        # coefficients are float64 (complex128) even for float32 vectors: the
        # f32 mode stores vectors in f32 but computes in f64 (csrc/common.cuh)
        self.coef_np_dtype = np.dtype(np.complex128 if np.iscomplexobj(np.zeros(0, self.np_dtype))
                                      else np.float64)
        self.coef_torch_dtype = _DTYPES[self.coef_np_dtype][1]
        self._host_stencil = st.astype(self.coef_np_dtype)
        self._host_diag = None if diag is None else np.asarray(diag).astype(self.coef_np_dtype)
        self.stencil = torch.as_tensor(np.ascontiguousarray(self._host_stencil)).to(self.device)
        self.diag = None if diag is None else torch.as_tensor(
            np.ascontiguousarray(self._host_diag)).to(self.device)
        lib = L.load()
        d = L.rg_op_desc(self.rg_dtype, self.kind, self.batch, self.side,
                         self.stencil.data_ptr(),
                         self.diag.data_ptr() if self.diag is not None else None,
                         1 if self.shared else 0)
        h = C.c_void_p()
        L.check(lib.rg_op_create(C.byref(h), C.byref(d)))
        self._h = h
        self._lib = lib

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.rg_op_destroy(h)
            self._h = None

    # ---- construction ----------------------------------------------------
    @classmethod
    def from_sparse(cls, A, dtype=None, device=None):
        """Single-system operator from an assembled CSR (richlab SparseMatrix
        or scipy sparse).  dtype defaults to the matrix dtype (float64 or
        complex128); float32 may be requested for real operators."""
        s, planes, present = extract_planes(A)
        kind, data = classify(s, planes, present)
        dt = np.dtype(dtype) if dtype is not None else planes.dtype
        if np.iscomplexobj(planes) and dt != np.complex128:
            raise ValueError("complex operator needs dtype complex128")
        if kind == "const9":
            return cls("const9", s, data[None, :], None, dt, device)
        if kind == "diag5":
            off, dg = data
            return cls("diag5", s, off[None, :], dg[None, :], dt, device)
        return cls("var9", s, planes[None, :, :], None, dt, device)

    @classmethod
    def from_problems(cls, problems, dtype=np.float64, device=None):
        """Batched operator straight from problem specs (no CSR assembly)."""
        problems = list(problems) if isinstance(problems, (list, tuple)) else [problems]
        sides = {p.n - 1 for p in problems}
        if len(sides) != 1:
            raise DimensionMismatch("all systems of a batch must share the grid size")
        s = sides.pop()
        if all(isinstance(p, AnisotropicProblem) for p in problems):
            st = np.stack([anisotropic_stencil(p) for p in problems])
            return cls("const9", s, st, None, dtype, device)
        if all(isinstance(p, HelmholtzProblem) for p in problems):
            offs, diags = zip(*(helmholtz_stencil(p) for p in problems))
            return cls("diag5", s, np.stack(offs), np.stack(diags), np.complex128, device)
        raise UnsupportedOperator("mixed or unknown problem kinds in one batch")

    @classmethod
    def stack(cls, ops):
        """Concatenate single operators of equal kind/side/dtype into a batch."""
        ops = list(ops)
        k, s, dt = ops[0].kind, ops[0].side, ops[0].np_dtype
        if any(o.kind != k or o.side != s or o.np_dtype != dt for o in ops):
            raise DimensionMismatch("stacked operators must share kind, side and dtype")
        st = np.concatenate([o._host_stencil for o in ops])
        dg = None if ops[0]._host_diag is None else np.concatenate([o._host_diag for o in ops])
        return cls(_KIND_NAMES[k], s, st, dg, dt, ops[0].device)

    def broadcast(self, batch):
        """The same operator applied to `batch` systems (shared coefficients)."""
        if self.nsets != 1:
            raise DimensionMismatch("only a single-system operator can be broadcast")
        return GpuStencilOperator(_KIND_NAMES[self.kind], self.side, self._host_stencil,
                                  self._host_diag, self.np_dtype, self.device, batch=batch)

    # ---- reference duck-typing -------------------------------------------
    @property
    def nrows(self):
        return self.P

    @property
    def ncols(self):
        return self.P

    @property
    def shape(self):
        return (self.P, self.P)

    @property
    def dtype(self):
        return self.np_dtype

    @property
    def handle(self):
        return self._h

    def diagonal(self, b=0):
        """Main diagonal of system b as a host array (sparse.py:116-117)."""
        b = 0 if self.shared else b
        if self.kind == L.RG_CONST9:
            c = self._host_stencil[b, 4]
            return np.full(self.P, c, dtype=self.coef_np_dtype)
        if self.kind == L.RG_DIAG5:
            return self._host_diag[b].copy()
        return self._host_stencil[b, 4].copy()

    def to_device(self, x, batched=None):
        """Host/torch vector(s) -> contiguous device tensor [B, P] of the op dtype."""
        t = torch.as_tensor(x) if not isinstance(x, torch.Tensor) else x
        t = t.to(device=self.device, dtype=self.torch_dtype)
        if t.numel() != self.batch * self.P:
            raise DimensionMismatch(
                f"operator has {self.batch} x {self.P} unknowns but vector has shape {tuple(t.shape)}")
        return t.reshape(self.batch, self.P).contiguous()

    def matvec(self, x):
        """y = A x (batched); numpy in -> numpy out, torch in -> torch out."""
        xt = self.to_device(x)
        y = torch.empty_like(xt)
        L.check(self._lib.rg_matvec(self._h, L.ptr(xt), L.ptr(y), L.stream_ptr()))
        return _like(y, x, self.batch)

    def rmatvec(self, x):
        """A^T x (unconjugated, sparse.py:108-114) via the transposed stencil."""
        return self.transpose().matvec(x)

    def transpose(self):
        if self.kind == L.RG_CONST9:
            return GpuStencilOperator("const9", self.side, self._host_stencil[:, ::-1].copy(),
                                      None, self.np_dtype, self.device, batch=self.batch)
        planes = self._full_planes()
        s = self.side
        t = np.zeros_like(planes)
        x, y = np.divmod(np.arange(self.P), s)
        for q, (dx, dy) in enumerate(OFFSETS9):
            # (A^T)[i, i+d] = A[i+d, i]: row i+d of A at offset -d (plane 8-q)
            ok = (x + dx >= 0) & (x + dx < s) & (y + dy >= 0) & (y + dy < s)
            src = np.nonzero(ok)[0]
            nb = (x[src] + dx) * s + (y[src] + dy)
            t[:, q, src] = planes[:, 8 - q, nb]
        return GpuStencilOperator("var9", s, t, None, self.np_dtype, self.device, batch=self.batch)

    def _full_planes(self):
        if self.kind == L.RG_VAR9:
            return self._host_stencil
        planes = np.zeros((self.nsets, 9, self.P), dtype=self.coef_np_dtype)
        inside = _neighbour_mask(self.side)
        for b in range(self.nsets):
            if self.kind == L.RG_CONST9:
                planes[b] = np.where(inside, self._host_stencil[b][:, None], 0)
            else:
                for j, q in enumerate((1, 3, 5, 7)):
                    planes[b, q] = np.where(inside[q], self._host_stencil[b, j], 0)
                planes[b, 4] = self._host_diag[b]
        return planes

    def residual(self, u, f, want_r=True):
        """(r = f - A u, ||r||^2 per system) on the device."""
        ut, ft = self.to_device(u), self.to_device(f)
        r = torch.empty_like(ut) if want_r else None
        n2 = torch.empty(self.batch, dtype=torch.float64, device=self.device)
        L.check(self._lib.rg_residual(self._h, L.ptr(ut), L.ptr(ft), L.ptr(r), L.ptr(n2),
                                      L.stream_ptr()))
        return r, n2

    def __repr__(self):
        return (f"GpuStencilOperator({_KIND_NAMES[self.kind]}, batch={self.batch}, shared={self.shared}, "
                f"side={self.side}, dtype={self.np_dtype})")


def _like(t, ref, batch):
    """Return device tensor t shaped/typed like the caller's input `ref`."""
    if isinstance(ref, torch.Tensor):
        return t.reshape(ref.shape) if ref.numel() == t.numel() else t
    out = t.cpu().numpy()
    shp = np.shape(ref)
    return out.reshape(shp) if int(np.prod(shp)) == out.size else out


class _OperatorMemo:
    """CSR matrix -> GpuStencilOperator, built once per matrix object.

    The reference's SparseMatrix is immutable (sparse.py:13-19), so the
    stencil extracted from it stays valid for the matrix's lifetime: repeated
    drop-in calls (`solve_stationary(A_csr, ...)` in a loop, `_smooth`-style
    reuse) then pay the host CSR scan and the coefficient upload only once,
    and the solver cache (keyed on the operator) hits.  Entries are keyed on
    id(A) and validated by a weak reference to A (falling back to a strong
    reference for objects that cannot be weakly referenced) plus the identity
    of the CSR value/index arrays, so a SciPy matrix whose arrays were
    replaced is re-extracted.  In-place edits of a SciPy matrix's arrays after
    a solve are not detected (the same contract as a cached factorisation)."""

    MAX = 16

    def __init__(self):
        self._d = {}

    @staticmethod
    def _arrays(A):
        if hasattr(A, "row_starts") and hasattr(A, "col_indices"):
            return (A.row_starts, A.col_indices, A.values)
        return tuple(getattr(A, k, None) for k in ("indptr", "indices", "data"))

    def get(self, A, dtype, device):
        import weakref
        key = (id(A), None if dtype is None else np.dtype(dtype).str, str(device))
        hit = self._d.get(key)
        if hit is not None:
            ref, arrs, op = hit
            if ref() is A and all(x is y for x, y in zip(arrs, self._arrays(A))):
                return op
            del self._d[key]
        op = GpuStencilOperator.from_sparse(A, dtype=dtype, device=device)
        try:
            ref = weakref.ref(A)
        except TypeError:
            ref = (lambda obj: (lambda: obj))(A)      # strong reference keeps id(A) unique
        if len(self._d) >= self.MAX:
            self._d.pop(next(iter(self._d)))
        self._d[key] = (ref, self._arrays(A), op)
        return op

    def clear(self):
        self._d.clear()


OPERATOR_MEMO = _OperatorMemo()


def operator_for_matrix(A, dtype=None, device=None):
    """Memoised GpuStencilOperator.from_sparse (see _OperatorMemo)."""
    return OPERATOR_MEMO.get(A, dtype, device)


def as_operator(A, dtype=None):
    """GpuStencilOperator for A (already one, or an assembled CSR)."""
    if isinstance(A, GpuStencilOperator):
        if dtype is not None and np.dtype(dtype) != A.np_dtype:
            raise ValueError("operator dtype differs from the requested dtype")
        return A
    return operator_for_matrix(A, dtype=dtype)

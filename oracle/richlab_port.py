"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

CPU restatement of the richlab hot path.  Each function cites the reference
lines it follows (paths relative to /root/reference/pkg/src/richlab/).  The
arithmetic goes through the same third-party kernels the reference uses --
SciPy CSR matvec, NumPy ufuncs, np.linalg.norm, scipy.fft.dstn,
scipy.linalg LU -- in the same order, so results are bitwise the
reference's on the same machine.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.fft
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla

DIVERGENCE_FACTOR = 1e12  # richardson.py:17


class OracleDivergence(RuntimeError):
    """richardson.py:20-23 DivergenceError."""

    def __init__(self, message, inner_iteration):
        super().__init__(message)
        self.inner_iteration = inner_iteration


# ----------------------------------------------------------- problems.py
def diffusion_tensor(eps, theta):
    """problems.py:95-99."""
    c, s = np.cos(theta), np.sin(theta)
    Q = np.array([[c, -s], [s, c]])
    return Q @ np.diag([1.0, eps]) @ Q.T


def element_matrix(C):
    """problems.py:17-23,102-118: 2x2 Gauss, symmetrised."""
    g = 0.5 / np.sqrt(3.0)
    Ke = np.zeros((4, 4))
    for xi, eta in ((0.5 - g, 0.5 - g), (0.5 + g, 0.5 - g), (0.5 + g, 0.5 + g), (0.5 - g, 0.5 + g)):
        G = np.array([[-(1 - eta), (1 - eta), eta, -eta],
                      [-(1 - xi), -xi, xi, (1 - xi)]])
        Ke += 0.25 * G.T @ C @ G
    return 0.5 * (Ke + Ke.T)


def _csr_from_triplets(N, rows, cols, vals, drop_tol=0.0):
    """sparse.py:67-81 SparseMatrix.from_triplets."""
    csr = sp.coo_matrix((vals, (rows, cols)), shape=(N, N)).tocsr()
    csr.sum_duplicates()
    if drop_tol != 0.0:
        csr.data[np.abs(csr.data) <= drop_tol] = 0.0
    csr.eliminate_zeros()
    csr.sort_indices()
    return csr


def assemble_anisotropic(eps, theta, n):
    """problems.py:121-154: Q1 FEM on the (n-1)^2 interior, unscaled."""
    Ke = element_matrix(diffusion_tensor(eps, theta))
    node = -np.ones((n + 1, n + 1), dtype=np.int64)
    gx, gy = np.meshgrid(np.arange(1, n), np.arange(1, n), indexing="ij")
    node[1:n, 1:n] = (gx - 1) * (n - 1) + (gy - 1)
    ex, ey = [a.reshape(-1) for a in np.meshgrid(np.arange(n), np.arange(n), indexing="ij")]
    corners = np.stack([node[ex, ey], node[ex + 1, ey], node[ex + 1, ey + 1], node[ex, ey + 1]], 1)
    R, Cc, V = [], [], []
    for a in range(4):
        for b in range(4):
            keep = (corners[:, a] >= 0) & (corners[:, b] >= 0)
            R.append(corners[keep, a])
            Cc.append(corners[keep, b])
            V.append(np.full(int(keep.sum()), Ke[a, b]))
    return _csr_from_triplets((n - 1) ** 2, np.concatenate(R), np.concatenate(Cc),
                              np.concatenate(V), drop_tol=1e-14 * np.abs(Ke).max())


def sponge_gamma(omega, n, width=None, c=1.0):
    """problems.py:157-171."""
    if width is None:
        width = max(1, int(round(2.0 * np.pi * c / (omega * (1.0 / n)))))
    i = np.arange(1, n)
    edge = np.minimum(i, n - i)
    dist = np.minimum(edge[:, None], edge[None, :])
    depth = np.clip(width - dist, 0, width) / width
    return (omega * depth ** 2).reshape(-1)


def assemble_helmholtz(omega, n, c=1.0, width=None):
    """problems.py:174-200: 5-point damped Helmholtz, complex symmetric."""
    h = 1.0 / n
    m = n - 1
    k = omega / c
    diag = (4.0 - k ** 2 * h ** 2) / h ** 2 + 1j * sponge_gamma(omega, n, width, c) * (omega / c ** 2)
    off = -1.0 / h ** 2
    idx = np.arange(m * m).reshape(m, m)
    R, Cc, V = [idx.reshape(-1)], [idx.reshape(-1)], [diag]
    for ra, ca in ((idx[:-1, :], idx[1:, :]), (idx[1:, :], idx[:-1, :]),
                   (idx[:, :-1], idx[:, 1:]), (idx[:, 1:], idx[:, :-1])):
        R.append(ra.reshape(-1))
        Cc.append(ca.reshape(-1))
        V.append(np.full(ra.size, off, dtype=np.complex128))
    return _csr_from_triplets(m * m, np.concatenate(R), np.concatenate(Cc), np.concatenate(V))


# ----------------------------------------------------------- schedules.py
def chebyshev_weights(lmax, lmin, m):
    """schedules.py:57-67."""
    x = np.cos((2 * np.arange(1, m + 1) - 1) * np.pi / (2 * m))
    return 2.0 / (lmax + lmin + (lmax - lmin) * x)


def jacobi_scale(A, relax=2.0 / 3.0):
    """precond.py:71-77: scale = relax / diag."""
    return relax / A.diagonal()


def _tri_solver(T):
    """precond.py:36-45: SuperLU of a triangular matrix in natural order
    without pivoting (the factor is the matrix itself), used as a
    substitution routine."""
    lu = spla.splu(T.tocsc(), permc_spec="NATURAL", diag_pivot_thresh=0.0,
                   options={"SymmetricMode": True})
    return lu.solve


def tri_precond(A, kind, relax=1.0):
    """precond.py:79-118: r -> B^{-1} r for kind 'gauss-seidel' (relax 1),
    'sor' or 'ssor'.  A: scipy CSR."""
    if kind == "gauss-seidel":
        relax = 1.0
    if not 0.0 < relax < 2.0:
        raise ValueError(f"relaxation must be in (0, 2), got {relax}")
    diag = A.diagonal()
    if np.any(diag == 0):
        raise ValueError(f"zero diagonal entry in row {int(np.nonzero(diag == 0)[0][0])}")
    DL = (sp.diags(diag) + relax * sp.tril(A, k=-1)).tocsr()
    dl = _tri_solver(DL)
    if kind in ("sor", "gauss-seidel"):
        return lambda r: relax * dl(r)
    DU = (sp.diags(diag) + relax * sp.triu(A, k=1)).tocsr()
    du = _tri_solver(DU)
    c = relax * (2.0 - relax)
    return lambda r: c * du(diag * dl(r))


def _precond(scale, r):
    """apply_preconditioner (precond.py:125-129): None, a Jacobi scale
    array, or a callable map."""
    if scale is None:
        return r
    return scale(r) if callable(scale) else scale * r


def _norm(x):
    return float(np.linalg.norm(x))


# ----------------------------------------------------------- richardson.py
def inner_update(A, f, u, v, w, a, at, variant, scale=None):
    """richardson.py:49-59 for one inner index."""
    if variant in ("plain", "mom"):
        r = f - A.dot(u)
    else:
        r = f - A.dot(u + at * v)
    p = _precond(scale, r)
    v = a * v + w * p
    return u + v, v


def solve_stationary(A, f, omega, alpha=None, alpha_tilde=None, variant="plain", scale=None,
                     tol=1e-6, max_outer=100_000, u0=None, check="outer"):
    """richardson.py:77-141.  Returns (u, report dict); raises OracleDivergence."""
    m = len(omega)
    alpha = np.zeros(m) if alpha is None else np.asarray(alpha, dtype=float)
    alpha_tilde = (alpha if variant == "nag" else np.zeros(m)) if alpha_tilde is None else \
        np.asarray(alpha_tilde, dtype=float)
    dtype = np.promote_types(A.dtype, np.asarray(f).dtype)
    n = A.shape[1]
    u = np.zeros(n, dtype=dtype) if u0 is None else np.array(u0, dtype=dtype)
    v = np.zeros(n, dtype=dtype)
    fnorm = _norm(f)
    if fnorm == 0.0:
        return u, dict(iterations=0, inner_iterations=0, converged=True,
                       final_relative_residual=0.0, trace=np.array([0.0]))
    reuse = variant in ("plain", "mom")
    r = f - A.dot(u)
    rel = _norm(r) / fnorm
    trace = [rel]
    inner = outer = 0
    converged = rel <= tol
    while not converged and outer < max_outer:
        for i in range(m):
            w, a, at = omega[i], alpha[i], alpha_tilde[i]
            step_r = r if reuse else f - A.dot(u + at * v)
            p = _precond(scale, step_r)
            v = a * v + w * p
            u = u + v
            inner += 1
            if reuse or check == "inner" or i == m - 1:
                r = f - A.dot(u)
                rel = _norm(r) / fnorm
                if not np.isfinite(rel) or rel > DIVERGENCE_FACTOR * max(trace[0], 1.0):
                    raise OracleDivergence(
                        f"residual blew up to {rel:.3g} at inner iteration {inner}", inner)
            if check == "inner" and rel <= tol:
                converged = True
                break
        outer += 1
        trace.append(rel)
        converged = converged or rel <= tol
    return u, dict(iterations=outer, inner_iterations=inner, converged=converged,
                   final_relative_residual=rel, trace=np.array(trace))


def outer_sweep(A, f, u, v, omega, alpha=None, alpha_tilde=None, variant="plain",
                scale=None, outer_count=0):
    """richardson.py:62-74.  Returns (u, v, ||f - A u||)."""
    m = len(omega)
    alpha = np.zeros(m) if alpha is None else np.asarray(alpha, dtype=float)
    alpha_tilde = (alpha if variant == "nag" else np.zeros(m)) if alpha_tilde is None else \
        np.asarray(alpha_tilde, dtype=float)
    for i in range(m):
        u, v = inner_update(A, f, u, v, omega[i], alpha[i], alpha_tilde[i], variant, scale)
        if not (np.all(np.isfinite(u.view(float))) and np.all(np.isfinite(v.view(float)))):
            raise OracleDivergence(
                f"non-finite iterate in inner step {i + 1} of outer sweep {outer_count + 1}",
                outer_count * m + i + 1)
    return u, v, _norm(f - A.dot(u))


# ----------------------------------------------------------- transforms.py / fns.py
def dst2(x):
    """transforms.py:24-35: orthonormal 2D DST-I (involutory)."""
    x = np.asarray(x)
    s = math.isqrt(x.size)
    return scipy.fft.dstn(x.reshape(s, s), type=1, norm="ortho").reshape(-1)


def fns_lite_step(A, f, u, omega, M, lam):
    """fns.py:76-84."""
    m = len(omega)
    for k in range(M):
        u = u + omega[k % m] * (f - A.dot(u))
    u = u + dst2(lam * dst2(f - A.dot(u)))
    if not np.all(np.isfinite(u)):
        raise OracleDivergence("hybrid step produced a non-finite iterate", M)
    return u


def solve_fns(A, f, omega, lam, M, tol=1e-6, max_iters=10_000):
    """fns.py:87-105."""
    u = np.zeros(A.shape[1])
    fnorm = np.linalg.norm(f)
    rel, trace, it = 1.0, [1.0], 0
    converged = fnorm == 0.0
    while not converged and it < max_iters:
        u = fns_lite_step(A, f, u, omega, M, lam)
        it += 1
        rel = float(np.linalg.norm(f - A.dot(u))) / fnorm
        trace.append(rel)
        converged = rel <= tol
    return u, dict(iterations=it, inner_iterations=it * M, converged=converged,
                   final_relative_residual=rel, trace=np.array(trace))


# ----------------------------------------------------------- multigrid.py
def _fw1d(n):
    """multigrid.py:24-36: 1D full weighting (1/4)[1,2,1], (n-1) -> (n/2-1)."""
    nc = n // 2
    r = np.repeat(np.arange(nc - 1), 3)
    c = (2 * np.arange(nc - 1)[:, None] + np.arange(3)[None, :]).reshape(-1)
    v = np.tile([0.25, 0.5, 0.25], nc - 1)
    return sp.csr_matrix((v, (r, c)), shape=(nc - 1, n - 1))


def _canon(M):
    M = sp.csr_matrix(M)
    M.sum_duplicates()
    M.sort_indices()
    M.eliminate_zeros()
    return M


def restriction(n):
    """multigrid.py:39-42."""
    r1 = _fw1d(n)
    return _canon(sp.kron(r1, r1, format="csr"))


def prolongation(n):
    """multigrid.py:45-49: P = 4 R^T (bilinear)."""
    p1 = (2.0 * _fw1d(n).T).tocsr()
    return _canon(sp.kron(p1, p1, format="csr"))


def build_hierarchy(A, n, coarsest=8):
    """multigrid.py:90-123 (schedules attached by the caller)."""
    levels, side, Al = [], n, _canon(A)
    while side > coarsest:
        R, P = restriction(side), prolongation(side)
        levels.append(dict(n=side, A=Al, R=R, P=P))
        Al = _canon((R @ Al @ P).tocsr())
        side //= 2
    levels.append(dict(n=side, A=Al))
    lu = scipy.linalg.lu_factor(Al.toarray())
    return levels, lu


def smooth(A, f, u, count, omega, alpha, alpha_tilde, variant):
    """multigrid.py:126-138: fresh v, no preconditioner."""
    if count == 0:
        return u
    v = np.zeros_like(u)
    for _ in range(count):
        for i in range(len(omega)):
            u, v = inner_update(A, f, u, v, omega[i], alpha[i], alpha_tilde[i], variant)
    if not np.all(np.isfinite(u.view(float))):
        raise OracleDivergence("smoother produced a non-finite iterate", count * len(omega))
    return u


def v_cycle(levels, lu, f, sched, u=None, pre=1, post=1):
    """multigrid.py:141-163 (one schedule dict shared by all levels)."""
    A0 = levels[0]["A"]
    dtype = np.promote_types(A0.dtype, np.asarray(f).dtype)
    u = np.zeros(A0.shape[1], dtype=dtype) if u is None else np.asarray(u, dtype=dtype)

    def level(k, f, u):
        if k == len(levels) - 1:
            return scipy.linalg.lu_solve(lu, f)
        L = levels[k]
        u = smooth(L["A"], f, u, pre, **sched)
        r = f - L["A"].dot(u)
        ec = level(k + 1, L["R"].dot(r), np.zeros(L["R"].shape[0], dtype=r.dtype))
        u = u + L["P"].dot(ec)
        return smooth(L["A"], f, u, post, **sched)

    return level(0, np.asarray(f, dtype=dtype), u)


# ----------------------------------------------------------- fgmres.py
def fgmres(A, f, precond, restart=20, tol=1e-6, max_outer=100):
    """fgmres.py:31-131 (real or complex, MGS + Givens, flexible)."""
    n = A.shape[1]
    dtype = np.promote_types(A.dtype, np.asarray(f).dtype)
    u = np.zeros(n, dtype=dtype)
    fnorm = float(np.linalg.norm(f))
    if fnorm == 0.0:
        return u, dict(iterations=0, converged=True, final_relative_residual=0.0,
                       trace=np.array([0.0]), stagnated=False)
    r = f - A.dot(u)
    beta = float(np.linalg.norm(r))
    rel = beta / fnorm
    trace, total, outer = [rel], 0, 0
    converged, stagnated = rel <= tol, False
    while not converged and not stagnated and outer < max_outer:
        start_rel = rel
        V = np.zeros((n, restart + 1), dtype=dtype)
        Z = np.zeros((n, restart), dtype=dtype)
        H = np.zeros((restart + 1, restart), dtype=dtype)
        cs = np.zeros(restart, dtype=dtype)
        sn = np.zeros(restart, dtype=dtype)
        g = np.zeros(restart + 1, dtype=dtype)
        V[:, 0] = r / beta
        g[0] = beta
        k = 0
        while k < restart:
            z = np.asarray(precond(V[:, k]), dtype=dtype)
            Z[:, k] = z
            w = A.dot(z)
            for i in range(k + 1):
                H[i, k] = np.vdot(V[:, i], w)
                w = w - H[i, k] * V[:, i]
            hk1 = np.linalg.norm(w)
            H[k + 1, k] = hk1
            for i in range(k):
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -np.conj(sn[i]) * H[i, k] + np.conj(cs[i]) * H[i + 1, k]
                H[i, k] = t
            den = np.sqrt(np.abs(H[k, k]) ** 2 + np.abs(hk1) ** 2)
            if den == 0.0:
                cs[k], sn[k] = 1.0, 0.0
            else:
                cs[k], sn[k] = np.conj(H[k, k]) / den, np.conj(H[k + 1, k]) / den
            H[k, k] = cs[k] * H[k, k] + sn[k] * H[k + 1, k]
            H[k + 1, k] = 0.0
            g[k + 1] = -np.conj(sn[k]) * g[k]
            g[k] = cs[k] * g[k]
            total += 1
            rel = float(np.abs(g[k + 1])) / fnorm
            trace.append(rel)
            happy = hk1 <= 1e-14 * max(1.0, float(np.abs(H[k, k])))
            k += 1
            if rel <= tol or happy:
                converged = True
                break
            if hk1 > 0:
                V[:, k] = w / hk1
        Hk = np.triu(H[:k, :k])
        if k == 0:
            y = np.zeros(0, dtype=dtype)
        else:
            try:
                y = np.linalg.solve(Hk, g[:k])
            except np.linalg.LinAlgError:
                y = np.linalg.lstsq(Hk, g[:k], rcond=None)[0]
        u = u + Z[:, :k] @ y
        r = f - A.dot(u)
        beta = float(np.linalg.norm(r))
        rel = beta / fnorm
        converged = rel <= tol
        if not converged and rel >= start_rel:
            stagnated = True
        outer += 1
    return u, dict(iterations=total, converged=converged, final_relative_residual=rel,
                   trace=np.array(trace), stagnated=stagnated)




# ----------------------------------------------------------- training.py (unroll)
def unroll_forward(A, f, omega, alpha, alpha_t, K, variant, scale=None):
    """training.py:61-81: K inner updates from u = v = 0; returns (loss,
    histories us, vs, ps) with p_k = P r_k."""
    n = A.shape[1]
    u, v = np.zeros(n), np.zeros(n)
    us, vs, ps = [u], [v], []
    m = len(omega)
    for k in range(K):
        i = k % m
        y = u if variant in ("plain", "mom") else u + alpha_t[i] * v
        r = f - A.dot(y)
        p = _precond(scale, r)
        v = (alpha[i] * v + omega[i] * p) if variant != "plain" else omega[i] * p
        u = u + v
        us.append(u)
        vs.append(v)
        ps.append(p)
    return float(np.linalg.norm(f - A.dot(u)) / np.linalg.norm(f)), us, vs, ps


def unroll_grad(A, f, omega, alpha, alpha_t, K, variant, scale=None):
    """Reverse pass of _unroll_tape (training.py:84-104) as the tape performs
    it (tape.py:28-42, vjps of tape.py:93-133,191-199): returns (loss,
    d_omega, d_alpha, d_alpha_t).  `scale`: Jacobi scale (P^T = P)."""
    m = len(omega)
    loss, us, vs, ps = unroll_forward(A, f, omega, alpha, alpha_t, K, variant, scale)
    fnorm = float(np.linalg.norm(f))
    r = f - A.dot(us[K])
    nr = np.linalg.norm(r)
    g = (1.0 / fnorm) * (r / nr)
    ubar = -(A.T.dot(g))
    vbar = np.zeros_like(ubar)
    dw, da, dat = np.zeros(m), np.zeros(m), np.zeros(m)
    nag = variant in ("nag", "nagex")
    for k in range(K - 1, -1, -1):
        i = k % m
        vt = vbar + ubar
        if variant != "plain":
            da[i] += np.sum(vt * vs[k])
        dw[i] += np.sum(vt * ps[k])
        pbar = omega[i] * vt
        rbar = pbar if scale is None else scale * pbar
        ybar = -(A.T.dot(rbar))
        ubar = ubar + ybar
        vbar = alpha[i] * vt if variant != "plain" else np.zeros_like(vt)
        if nag:
            vbar = vbar + alpha_t[i] * ybar
            dat[i] += np.sum(ybar * vs[k])
    return loss, dw, da, dat


__all__ = [n for n in dir() if not n.startswith("_")]

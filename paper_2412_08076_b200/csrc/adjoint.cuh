// adjoint.cuh — reverse-mode pass of the K-step training unroll
// (training.py:84-104 _unroll_tape, differentiated by tape.py:191-199;
// SURVEY.md §8(f) item 3).
//
// Forward (per k, i = k mod m), recorded as histories u_k, v_k:
//     y_k = u_k (+ at_i v_k for nag/nagex);  r_k = f - A y_k;  p_k = P r_k
//     v_{k+1} = a_i v_k + w_i p_k;  u_{k+1} = u_k + v_{k+1}
//     L = ||f - A u_K|| / ||f||
// Reverse, with vt = vbar_{k+1} + ubar_{k+1} (adjoint of v_{k+1}):
//     dL/da_i  += <vt, v_k>      dL/dw_i += <vt, p_k>
//     rbar = P^T (w_i vt);  ybar = -A^T rbar
//     ubar_k = ubar_{k+1} + ybar;  vbar_k = a_i vt (+ at_i ybar)
//     dL/dat_i += <ybar, v_k>    (nag/nagex)
// Two kernels per step (the second needs rbar at the neighbours); the three
// inner products are per-CTA partials summed in a fixed order (deterministic,
// not BLAS-bitwise).  Real float64 operators; P = identity or Jacobi inline,
// GS / SOR / SSOR through the two-phase entry (adj_a_ext_kernel, then the
// host's transposed triangular solve, then adj_b_kernel).
#pragma once
#include "step.cuh"

namespace rg {

struct AdjArgs {
    OpView<double> A;       // forward operator
    OpView<double> At;      // its transpose (A^T x = matvec of At)
    const double* f;
    const double* u;        // u_k  [B][P]
    const double* v;        // v_k
    double* ubar;           // in: ubar_{k+1}; out: ubar_k (in place)
    double* vbar;           // in: vbar_{k+1}; out: vbar_k (in place)
    double* rbar;           // work [B][P]
    const double* omega;
    const double* alpha;    // may be null (plain)
    const double* atil;     // may be null unless nag/nagex
    const double* scale;    // Jacobi: [B] (JSCALAR) or [B][P] (JFIELD)
    const double* pk;       // external preconditioner: p_k history [B][P] (EXT pass)
    double* rbar_pre;       // external preconditioner: w vt, before P^T (EXT pass)
    int precond;
    int m, i;
    int nag;
    double* part;           // [3][B][ncta]
};

// pass 1 with an external (GS/SOR/SSOR) preconditioner: p_k from the forward
// history, rbar_pre = w vt (the host applies P^T with rg_tri_apply)
__global__ void __launch_bounds__(STEP_NT) adj_a_ext_kernel(AdjArgs a) {
    const int b = blockIdx.z;
    const int side = a.A.side;
    const int cta = blockIdx.x + gridDim.x * blockIdx.y;
    const int ncta = gridDim.x * gridDim.y;
    const int j = blockIdx.x * STEP_BX + threadIdx.x;
    const int i = blockIdx.y * STEP_BY + threadIdx.y;
    const size_t base = (size_t)b * a.A.P;
    const int si = b * a.m + a.i;
    double d1 = 0.0, d2 = 0.0;
    if (i < side && j < side) {
        const size_t q = base + (size_t)i * side + j;
        const double vt = a.vbar[q] + a.ubar[q];
        d1 = vt * a.v[q];
        d2 = vt * a.pk[q];
        a.rbar_pre[q] = a.omega[si] * vt;
    }
    write_partial<STEP_NT>(a.part + ((size_t)0 * gridDim.z + b) * ncta, cta, d1);
    write_partial<STEP_NT>(a.part + ((size_t)1 * gridDim.z + b) * ncta, cta, d2);
}

// pass 1: p_k at the point (stencil of y_k), vt, rbar; partials <vt,v_k>, <vt,p_k>
template <int KIND>
__global__ void __launch_bounds__(STEP_NT) adj_a_kernel(AdjArgs a) {
    const int b = blockIdx.z;
    const int side = a.A.side;
    const int cta = blockIdx.x + gridDim.x * blockIdx.y;
    const int ncta = gridDim.x * gridDim.y;
    const int j = blockIdx.x * STEP_BX + threadIdx.x;
    const int i = blockIdx.y * STEP_BY + threadIdx.y;
    const size_t base = (size_t)b * a.A.P;
    const int si = b * a.m + a.i;
    double d1 = 0.0, d2 = 0.0;
    if (i < side && j < side) {
        const size_t idx = (size_t)i * side + j;
        const double at = a.nag ? a.atil[si] : 0.0;
        const double* u = a.u + base;
        const double* v = a.v + base;
        auto Y = [&](int di, int dj) -> double {
            const int ii = i + di, jj = j + dj;
            if (ii < 0 || ii >= side || jj < 0 || jj >= side) return 0.0;
            const size_t q = idx + (ptrdiff_t)di * side + dj;
            return a.nag ? u[q] + at * v[q] : u[q];
        };
        const double r = a.f[base + idx] - apply_op<double, KIND>(a.A, b, idx, Y);
        double sc = 1.0;
        if (a.precond == P_JSCALAR) sc = a.scale[b];
        else if (a.precond == P_JFIELD) sc = a.scale[base + idx];
        const double p = a.precond == P_NONE ? r : sc * r;
        const double vt = a.vbar[base + idx] + a.ubar[base + idx];
        d1 = vt * v[idx];
        d2 = vt * p;
        const double pb = a.omega[si] * vt;
        a.rbar[base + idx] = a.precond == P_NONE ? pb : sc * pb;
    }
    write_partial<STEP_NT>(a.part + ((size_t)0 * gridDim.z + b) * ncta, cta, d1);
    write_partial<STEP_NT>(a.part + ((size_t)1 * gridDim.z + b) * ncta, cta, d2);
}

// pass 2: ybar = -A^T rbar; ubar_k, vbar_k in place; partial <ybar, v_k>
template <int KIND>
__global__ void __launch_bounds__(STEP_NT) adj_b_kernel(AdjArgs a) {
    const int b = blockIdx.z;
    const int side = a.A.side;
    const int cta = blockIdx.x + gridDim.x * blockIdx.y;
    const int ncta = gridDim.x * gridDim.y;
    const int j = blockIdx.x * STEP_BX + threadIdx.x;
    const int i = blockIdx.y * STEP_BY + threadIdx.y;
    const size_t base = (size_t)b * a.A.P;
    const int si = b * a.m + a.i;
    double d3 = 0.0;
    if (i < side && j < side) {
        const size_t idx = (size_t)i * side + j;
        const double* rb = a.rbar + base;
        auto X = [&](int di, int dj) -> double {
            const int ii = i + di, jj = j + dj;
            if (ii < 0 || ii >= side || jj < 0 || jj >= side) return 0.0;
            return rb[idx + (ptrdiff_t)di * side + dj];
        };
        const double yb = -apply_op<double, KIND>(a.At, b, idx, X);
        const double ub = a.ubar[base + idx];
        const double vt = a.vbar[base + idx] + ub;
        const double al = a.alpha ? a.alpha[si] : 0.0;
        a.ubar[base + idx] = ub + yb;
        double vb = al * vt;
        if (a.nag) {
            vb = vb + a.atil[si] * yb;
            d3 = yb * a.v[base + idx];
        }
        a.vbar[base + idx] = vb;
    }
    write_partial<STEP_NT>(a.part + ((size_t)2 * gridDim.z + b) * ncta, cta, d3);
}

// seed: r = f - A u_K with partial sums of r^2 and f^2
template <int KIND>
__global__ void __launch_bounds__(STEP_NT) adj_seed_a_kernel(OpView<double> A, const double* u,
                                                            const double* f, double* r,
                                                            double* part) {
    const int b = blockIdx.z;
    const int side = A.side;
    const int cta = blockIdx.x + gridDim.x * blockIdx.y;
    const int ncta = gridDim.x * gridDim.y;
    const int j = blockIdx.x * STEP_BX + threadIdx.x;
    const int i = blockIdx.y * STEP_BY + threadIdx.y;
    const size_t base = (size_t)b * A.P;
    double rr = 0.0, ff = 0.0;
    if (i < side && j < side) {
        const size_t idx = (size_t)i * side + j;
        const double* ub = u + base;
        auto X = [&](int di, int dj) -> double {
            const int ii = i + di, jj = j + dj;
            if (ii < 0 || ii >= side || jj < 0 || jj >= side) return 0.0;
            return ub[idx + (ptrdiff_t)di * side + dj];
        };
        const double fi = f[base + idx];
        const double ri = fi - apply_op<double, KIND>(A, b, idx, X);
        r[base + idx] = ri;
        rr = ri * ri;
        ff = fi * fi;
    }
    write_partial<STEP_NT>(part + ((size_t)0 * gridDim.z + b) * ncta, cta, rr);
    write_partial<STEP_NT>(part + ((size_t)1 * gridDim.z + b) * ncta, cta, ff);
}

// loss = ||r|| / ||f||;  rbar = r (1/||f||) / ||r||  (tape.py norm2 / mul vjps)
__global__ void adj_seed_scale_kernel(int B, int P, const double* sums, double* r, double* loss) {
    const int b = blockIdx.y;
    const double n = sqrt(sums[b]);
    const double fn = sqrt(sums[B + b]);
    if (blockIdx.x == 0 && threadIdx.x == 0) loss[b] = n * (1.0 / fn);
    const double c = n > 0.0 ? (1.0 / fn) / n : 0.0;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < P; q += gridDim.x * blockDim.x)
        r[(size_t)b * P + q] = n > 0.0 ? r[(size_t)b * P + q] * c : 0.0;
}

// ubar_K = -A^T rbar, vbar_K = 0
template <int KIND>
__global__ void __launch_bounds__(STEP_NT) adj_seed_b_kernel(OpView<double> At, const double* rbar,
                                                            double* ubar, double* vbar) {
    const int b = blockIdx.z;
    const int side = At.side;
    const int j = blockIdx.x * STEP_BX + threadIdx.x;
    const int i = blockIdx.y * STEP_BY + threadIdx.y;
    if (i >= side || j >= side) return;
    const size_t base = (size_t)b * At.P;
    const size_t idx = (size_t)i * side + j;
    const double* rb = rbar + base;
    auto X = [&](int di, int dj) -> double {
        const int ii = i + di, jj = j + dj;
        if (ii < 0 || ii >= side || jj < 0 || jj >= side) return 0.0;
        return rb[idx + (ptrdiff_t)di * side + dj];
    };
    ubar[base + idx] = -apply_op<double, KIND>(At, b, idx, X);
    vbar[base + idx] = 0.0;
}

}  // namespace rg

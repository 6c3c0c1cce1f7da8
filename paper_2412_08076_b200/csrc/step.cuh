// step.cuh — one-inner-step kernels for every operator kind and dtype.
//
// These cover the general cases (complex Helmholtz / Galerkin operators,
// check="inner", outer_sweep, V-cycle smoothing, rg_residual/rg_matvec).
// The anisotropic CONST9 real sweeps of solve_stationary go through the
// temporally blocked kernel in block.cuh instead.
//
// One thread per grid point, neighbours through L1; all operands are
// streamed once from HBM per step, so the kernel is HBM-bound.
#pragma once
#include "reduce.cuh"

namespace rg {

template <typename S>
struct OpView {
    const CT<S>* stencil;  // CONST9 [B][9] | DIAG5 [B][4] | VAR9 [B][9][P] (arithmetic type)
    const CT<S>* diag;     // DIAG5 [B][P]
    int side;
    int P;
    int shared;        // one coefficient set applied to every system of the batch
};

// y = A x at interior point (i, j) of system b, CSR column order, no FMA.
// X(di, dj) returns the stencil input at (i+di, j+dj), zero outside.
// Zero-padded terms add +-0 to an accumulator that is never -0, which is an
// exact no-op, so boundary rows (fewer CSR entries) are reproduced bitwise.
template <typename S, int KIND, class F>
__device__ __forceinline__ CT<S> apply_op(const OpView<S>& A, int bv, size_t idx, F X) {
    typedef CT<S> C;
    const int b = A.shared ? 0 : bv;   // coefficient set of vector system bv
    if (KIND == K_CONST9) {
        const C* c = A.stencil + (size_t)b * 9;
        C s = mul(c[0], X(-1, -1));
        s = add(s, mul(c[1], X(-1, 0)));
        s = add(s, mul(c[2], X(-1, 1)));
        s = add(s, mul(c[3], X(0, -1)));
        s = add(s, mul(c[4], X(0, 0)));
        s = add(s, mul(c[5], X(0, 1)));
        s = add(s, mul(c[6], X(1, -1)));
        s = add(s, mul(c[7], X(1, 0)));
        s = add(s, mul(c[8], X(1, 1)));
        return s;
    } else if (KIND == K_DIAG5) {
        const C* c = A.stencil + (size_t)b * 4;
        C s = mul(c[0], X(-1, 0));
        s = add(s, mul(c[1], X(0, -1)));
        s = add(s, mul(A.diag[(size_t)b * A.P + idx], X(0, 0)));
        s = add(s, mul(c[2], X(0, 1)));
        s = add(s, mul(c[3], X(1, 0)));
        return s;
    } else {  // K_VAR9: planes [b][d][P]
        const C* c = A.stencil + (size_t)b * 9 * A.P + idx;
        const size_t P = A.P;
        C s = mul(c[0], X(-1, -1));
        s = add(s, mul(c[1 * P], X(-1, 0)));
        s = add(s, mul(c[2 * P], X(-1, 1)));
        s = add(s, mul(c[3 * P], X(0, -1)));
        s = add(s, mul(c[4 * P], X(0, 0)));
        s = add(s, mul(c[5 * P], X(0, 1)));
        s = add(s, mul(c[6 * P], X(1, -1)));
        s = add(s, mul(c[7 * P], X(1, 0)));
        s = add(s, mul(c[8 * P], X(1, 1)));
        return s;
    }
}

template <typename S>
struct StepArgs {
    OpView<S> A;
    const S* u_in;
    const S* v_in;     // may be null (treated as 0)
    S* u_out;
    S* v_out;          // may be null
    const S* f;
    S* r_out;          // residual output (rg_residual), may be null
    const double* omega;
    const double* alpha;
    const double* atil;
    const CT<S>* scale;  // Jacobi scale (P_JSCALAR: [B], P_JFIELD: [B][P])
    int m;
    int i;             // schedule index of this inner step
    int variant;       // V_*
    int precond;       // P_*
    int update;        // apply the Richardson update
    int norm_u;        // accumulate ||f - A u||^2 (slot 0)
    int use_status;    // skip systems whose SysState is not ACTIVE
    int* nonfinite_at; // outer_sweep finite check (may be null)
    int tag;
    double* partials;  // plain partial mode (rg_residual): [B][ncta], may be null
    EpiArgs epi;       // fused decision mode when epi.st != null
};

constexpr int STEP_BX = 32, STEP_BY = 8, STEP_NT = STEP_BX * STEP_BY;
// rows per thread of step1_kernel (rows i, i + STEP_BY, ...); 2 measured
// slower than 1 on the complex V-cycle smoother (5.87 vs 5.45 ms per cycle)
constexpr int STEP_RPT = 1;

template <typename S, int KIND>
__global__ void __launch_bounds__(STEP_NT) step1_kernel(StepArgs<S> a) {
    const int b = blockIdx.z;
    const int side = a.A.side;
    const int cta = blockIdx.x + gridDim.x * blockIdx.y;
    const int ncta = gridDim.x * gridDim.y;
    if (a.use_status && a.epi.st[b].status != ST_ACTIVE) return;  // uniform per CTA

    const int j = blockIdx.x * STEP_BX + threadIdx.x;
    const size_t base = (size_t)b * a.A.P;
    const bool nag = a.variant >= V_NAG;
    const int si = b * a.m + a.i;
    typedef CT<S> C;
    double acc[1] = {0.0};
    double facc = 0.0;
    const S* u = a.u_in + base;
    const S* v = a.v_in ? a.v_in + base : nullptr;
#pragma unroll
    for (int rr = 0; rr < STEP_RPT; ++rr) {
        const int i = (blockIdx.y * STEP_RPT + rr) * STEP_BY + threadIdx.y;
        if (i >= side || j >= side) continue;
        const size_t idx = (size_t)i * side + j;
        auto Xu = [&](int di, int dj) -> C {
            const int ii = i + di, jj = j + dj;
            if (ii < 0 || ii >= side || jj < 0 || jj >= side) return szero<C>();
            return to_c(u[idx + (ptrdiff_t)di * side + dj]);
        };
        const C fi = a.f ? to_c(a.f[base + idx]) : szero<C>();
        C r = szero<C>();
        if (!nag || !a.update) {
            // plain / mom: the step residual is the residual at u (:116-117)
            const C s = apply_op<S, KIND>(a.A, b, idx, Xu);
            r = sub(fi, s);
            if (a.norm_u) acc[0] = sqacc(acc[0], r);
        } else {
            // nag / nagex: residual at the look-ahead u + at*v (:118-119)
            const double at = a.atil[si];
            auto Xy = [&](int di, int dj) -> C {
                const int ii = i + di, jj = j + dj;
                if (ii < 0 || ii >= side || jj < 0 || jj >= side) return szero<C>();
                const size_t q = idx + (ptrdiff_t)di * side + dj;
                C x = to_c(u[q]);
                if (v) x = add(x, rmul(at, to_c(v[q])));
                return x;
            };
            const C s = apply_op<S, KIND>(a.A, b, idx, Xy);
            r = sub(fi, s);
            if (a.norm_u) {  // convergence residual at u itself (:124-125)
                const C su = apply_op<S, KIND>(a.A, b, idx, Xu);
                acc[0] = sqacc(acc[0], sub(fi, su));
            }
        }
        if (a.r_out) a.r_out[base + idx] = to_s<S>(r);
        if (a.update) {
            C p = r;  // precond.py:125-129
            if (a.precond == P_JSCALAR) p = mul(a.scale[b], r);
            else if (a.precond == P_JFIELD) p = mul(a.scale[base + idx], r);
            const double w = a.omega[si];
            const C ui = to_c(u[idx]);
            C vn;
            if (a.variant == V_PLAIN) {
                vn = rmul(w, p);  // 0*v + w*p == w*p for finite v
            } else {
                const C vi = v ? to_c(v[idx]) : szero<C>();
                vn = add(rmul(a.alpha[si], vi), rmul(w, p));  // :120 / :58
            }
            const S vs = to_s<S>(vn);
            const S us = to_s<S>(add(ui, vn));  // :121 / :59 (u + v from the unrounded v)
            a.u_out[base + idx] = us;
            if (a.v_out) a.v_out[base + idx] = vs;
            if (a.nonfinite_at && !(finite(us) && finite(vs))) atomicMin(&a.nonfinite_at[b], a.tag);
        }
        if (a.epi.with_f) facc = sqacc(facc, fi);
    }
    if (a.partials) {
        write_partial<STEP_NT>(a.partials + (size_t)b * ncta, cta, acc[0]);
    } else if (a.epi.st && (a.epi.nslots > 0 || a.epi.with_f)) {
        epilogue<STEP_NT, 1>(a.epi, b, cta, ncta, acc, facc);
    }
}

// y = A x (sparse.py:101-106), batched.
template <typename S, int KIND>
__global__ void __launch_bounds__(STEP_NT) matvec_kernel(OpView<S> A, const S* x, S* y) {
    typedef CT<S> C;
    const int b = blockIdx.z;
    const int side = A.side;
    const int j = blockIdx.x * STEP_BX + threadIdx.x;
    const int i = blockIdx.y * STEP_BY + threadIdx.y;
    if (i >= side || j >= side) return;
    const size_t base = (size_t)b * A.P;
    const size_t idx = (size_t)i * side + j;
    const S* xs = x + base;
    auto X = [&](int di, int dj) -> C {
        const int ii = i + di, jj = j + dj;
        if (ii < 0 || ii >= side || jj < 0 || jj >= side) return szero<C>();
        return to_c(xs[idx + (ptrdiff_t)di * side + dj]);
    };
    y[base + idx] = to_s<S>(apply_op<S, KIND>(A, b, idx, X));
}

}  // namespace rg

// tri.cuh — Gauss-Seidel / SOR / SSOR preconditioners on the device
// (precond.py:79-118).
//
//   SOR (GS = SOR with relax 1):  z = relax * (D + relax L)^{-1} r
//   SSOR:  z = c * (D + relax U)^{-1} (D * ((D + relax L)^{-1} r)),
//          c = relax (2 - relax)
// with L / U the strict lower / upper parts of A in the lexicographic order
// of the grid (x the first axis, precond.py:10-12).  The reference factors
// the triangular matrices with SuperLU in natural order and substitutes; the
// lower stencil of a 9-point operator couples (i, j) to (i-1, j-1..j+1) and
// (i, j-1), so the substitution is a slope-2 wavefront: point (i, j) can be
// computed at step s = j + 2 i.
//
// One CTA per system.  Thread t owns grid row p0 + t of the current pass
// (rows are processed in passes of blockDim.x), walks its row left to right
// one point per step, and receives the row above through a warp shuffle
// (lane - 1 computed x(i-1, j+1) in the previous step), through a two-slot
// shared-memory mailbox across warps, and through `edge` (the last row of
// the previous pass).  One __syncthreads per step.  The right-hand side is
// prefetched PF points ahead.  Contributions are subtracted in the column
// order of a column-oriented substitution and divided by the diagonal, as
// the reference's triangular solves do; SuperLU stores the lower factor
// pre-divided by the diagonal, so results agree to rounding (~1e-15), the
// reference's own bar for these maps is 1e-13 (test_precond.py:33-62).
// The backward (upper) solve is the same walk in reversed index order.
#pragma once
#include "common.cuh"

namespace rg {

enum { TRI_SOR = 1, TRI_SSOR = 2 };
constexpr int TRI_PF = 8;

template <typename S>
struct TriArgs {
    const double* stencil;  // CONST9 [B or 1][9]
    int shared;
    int side, P;
    double relax;
    const S* r;
    S* z;
    S* work;                // SSOR: forward result [B][P]
};

// One substitution sweep: dst = oscale * x where M x = rhs, M lower
// triangular in traversal order (reversed index order when REV).
// rhs = src, or d * src when MULD (SSOR's D * y).  Coefficients in
// traversal order: l0 (i-1, j-1), l1 (i-1, j), l2 (i-1, j+1), l3 (i, j-1).
//
// Every step ends in a block barrier, so the step time is the slowest
// warp's body: the body is branch-free (predicated stores/loads, pointers
// advanced per step) and warps whose rows have not started or are finished
// skip whole windows of TRI_PF steps (barrier only).  x = t * (1/d): one rounding more than a
// division, inside the 1e-13 bar.
template <bool REV, bool MULD, bool SCALE, typename SI, typename SO>
__device__ __forceinline__ void tri_sweep(const SI* __restrict__ src, SO* __restrict__ dst, int side,
                                          int P, double oscale, double l0, double l1, double l2,
                                          double l3, double d, double* edge, double (*xfer)[2]) {
    const int t = threadIdx.x, NT = blockDim.x, lane = t & 31, wp = t >> 5;
    const int nw = NT >> 5;
    const double rd = 1.0 / d;
    for (int p0 = 0; p0 < side; p0 += NT) {
        const int ip = p0 + t;
        const bool row_ok = ip < side;
        const int nrows = min(NT, side - p0);
        const int nsteps = side + 2 * (nrows - 1);
        if (t < nw) xfer[t][0] = xfer[t][1] = 0.0;
        __syncthreads();
        const long long rbase = (long long)ip * side;
        // element jp of this thread's row (traversal order); clamped in-row
        auto gptr = [&](int jp) -> long long {
            const long long g = rbase + jp;
            return REV ? (long long)P - 1 - g : g;
        };
        auto ld = [&](int jp) -> double {
            if (!row_ok || jp < 0 || jp >= side) return 0.0;
            return (double)src[gptr(jp)];
        };
        double rq[TRI_PF];
#pragma unroll
        for (int q = 0; q < TRI_PF; ++q) rq[q] = ld(q - 2 * t);
        double left = 0.0, nm1 = 0.0, n0 = 0.0, pub = 0.0;
        // thread 0 starts at column 0 with no warm-up steps: x(i-1, 0) of the
        // previous pass's last row seeds its window (zero for the first pass)
        if (t == 0 && p0 > 0) n0 = edge[0];
        // warp's rows: lane 0 starts at step a0, lane 31 is done at a0 + 62 + side
        const int a0 = 2 * 32 * wp;
        for (int s0 = 0; s0 < nsteps; s0 += TRI_PF) {
            // idle before lane 0's warm-up step a0 - 1, and after lane 31
            // relayed its trailing zero (step a0 + 62 + side)
            const bool idle = (s0 + TRI_PF <= a0 - 1) || (s0 > a0 + 62 + side);
            if (idle) {
#pragma unroll
                for (int q = 0; q < TRI_PF; ++q) {
                    rq[q] = ld(s0 + TRI_PF + q - 2 * t);   // next window's rhs
                    __syncthreads();
                }
                continue;
            }
            // one predicated body: pointers advance by one element per step
            // whether or not the row is inside its column range
            const int jp0 = s0 - 2 * t;
            SO* out = dst + gptr(jp0);
            const SI* in = src + gptr(jp0 + TRI_PF);
#pragma unroll
            for (int q = 0; q < TRI_PF; ++q) {
                const int s = s0 + q;
                const int jp = jp0 + q;
                const bool act = row_ok && (unsigned)jp < (unsigned)side;
                double nb = __shfl_up_sync(0xffffffffu, pub, 1);
                if (lane == 0)
                    nb = wp > 0 ? xfer[wp][(s + 1) & 1]
                                : ((p0 > 0 && (unsigned)(jp + 1) < (unsigned)side) ? edge[jp + 1]
                                                                                  : 0.0);
                double tt = MULD ? d * rq[q] : rq[q];
                tt = tt - l0 * nm1;
                tt = tt - l1 * n0;
                tt = tt - l2 * nb;
                tt = tt - l3 * left;
                const double x = act ? tt * rd : 0.0;
                if (act) {
                    out[REV ? -q : q] = (SO)(SCALE ? oscale * x : x);
                    if (t == NT - 1) edge[jp] = x;
                }
                nm1 = n0;
                n0 = nb;
                left = x;
                pub = x;
                if (lane == 31 && wp + 1 < nw) xfer[wp + 1][s & 1] = x;
                const bool nact = row_ok && (unsigned)(jp + TRI_PF) < (unsigned)side;
                rq[q] = nact ? (double)in[REV ? -q : q] : 0.0;
                __syncthreads();
            }
        }
        __syncthreads();
    }
}

template <typename S, int MODE>
__global__ void __launch_bounds__(1024, 1) tri_kernel(const TriArgs<S> a) {
    extern __shared__ double edge[];
    __shared__ double xfer[32][2];
    const int b = blockIdx.x;
    const double* c = a.stencil + (size_t)(a.shared ? 0 : b) * 9;
    const double w = a.relax;
    // DL = diag + relax * tril(A, -1), DU = diag + relax * triu(A, 1) (precond.py:91,104-105)
    const double d = c[4];
    const double lo0 = w * c[0], lo1 = w * c[1], lo2 = w * c[2], lo3 = w * c[3];
    const double up0 = w * c[8], up1 = w * c[7], up2 = w * c[6], up3 = w * c[5];
    const size_t base = (size_t)b * a.P;
    if (MODE == TRI_SOR) {
        // relax * solve(r)  (precond.py:93)
        tri_sweep<false, false, true, S, S>(a.r + base, a.z + base, a.side, a.P, w, lo0, lo1, lo2,
                                            lo3, d, edge, xfer);
    } else {
        // c * du(diag * dl(r))  (precond.py:109-110)
        const double cc = w * (2.0 - w);
        tri_sweep<false, false, false, S, S>(a.r + base, a.work + base, a.side, a.P, 1.0, lo0, lo1,
                                             lo2, lo3, d, edge, xfer);
        __syncthreads();
        tri_sweep<true, true, true, S, S>(a.work + base, a.z + base, a.side, a.P, cc, up0, up1, up2,
                                          up3, d, edge, xfer);
    }
}

template <typename S, int MODE>
cudaError_t launch_tri_m(const TriArgs<S>& a, int batch, cudaStream_t st) {
    int nt = (a.side + 31) / 32 * 32;
    if (nt > 1024) nt = 1024;
    const size_t smem = (size_t)a.side * sizeof(double);
    auto k = tri_kernel<S, MODE>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k<<<batch, nt, smem, st>>>(a);
    return cudaGetLastError();
}

template <typename S>
cudaError_t launch_tri(const TriArgs<S>& a, int mode, int batch, cudaStream_t st) {
    return mode == TRI_SOR ? launch_tri_m<S, TRI_SOR>(a, batch, st)
                           : launch_tri_m<S, TRI_SSOR>(a, batch, st);
}

// Richardson update from an externally preconditioned residual z
// (richardson.py:120-121 / :58-59):  v = a_i v + w_i z ;  u = u + v, and
// the next look-ahead point y = u + at_{i+1} v for nag/nagex.  z == NULL:
// only y = u + at_i v (the first look-ahead of a solve).
template <typename S>
__global__ void pupdate_kernel(int B, int P, const S* z, S* u, S* v, S* y, const double* omega,
                               const double* alpha, const double* atil, int m, int i, int variant) {
    const size_t n = (size_t)B * P;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
         q += (size_t)gridDim.x * blockDim.x) {
        const int b = (int)(q / P);
        const double ui = to_c(u[q]);
        const double vi = v ? to_c(v[q]) : 0.0;
        if (!z) {
            y[q] = to_s<S>(ui + atil[b * m + i] * vi);
            continue;
        }
        const int si = b * m + i;
        const double zi = to_c(z[q]);
        const double vn = variant == V_PLAIN ? omega[si] * zi : alpha[si] * vi + omega[si] * zi;
        const S vs = to_s<S>(vn);
        const S us = to_s<S>(ui + vn);
        u[q] = us;
        if (v) v[q] = vs;
        if (y) y[q] = to_s<S>(to_c(us) + atil[b * m + (i + 1) % m] * to_c(vs));
    }
}

}  // namespace rg

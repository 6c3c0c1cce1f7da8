// resid.cuh — r = f - A u and ||r||^2 for the constant 9-point real operator
// (richardson.py:105-106,124-125; fns.py:80,99; multigrid.py:151): the
// residual pass every driver calls between sweeps.  step1_kernel does this
// one point per thread through L1 (45 us for 4 x 1023^2, 1.5 TB/s); here a
// CTA stages a 32 x 128 tile of u with its one-cell halo in shared memory
// (coalesced row loads, zeros outside the grid), every thread takes 4
// columns of 4 rows, and f / r stream straight between global memory and
// registers.  Same arithmetic per point as step1_kernel: the CSR-order
// unfused stencil sum (apply_op<K_CONST9>), r = f - s, and the norm
// accumulated with fma; the per-CTA partials are summed in a fixed order by
// sum_partials_kernel (deterministic; the summation order differs from
// step1_kernel's, so norms agree to rounding, r bitwise).
#pragma once
#include "step.cuh"

namespace rg {

constexpr int RS_TR = 32, RS_TC = 128, RS_NT = 256;
constexpr int RS_LD = RS_TC + 4;          // staged row stride (u columns -1 .. 128, padded)

template <typename S>
struct ResidArgs {
    const double* stencil;   // [B or 1][9]
    int shared;
    int side, P;
    const S* u;
    const S* f;
    S* r;                    // may be null
    double* partials;        // [B][ncta], may be null
};

template <typename S>
__global__ void __launch_bounds__(RS_NT) resid9_kernel(const ResidArgs<S> a) {
    __shared__ double su[(RS_TR + 2) * RS_LD];
    const int b = blockIdx.z, side = a.side;
    const int i0 = blockIdx.y * RS_TR, j0 = blockIdx.x * RS_TC;
    const size_t base = (size_t)b * a.P;
    const S* u = a.u + base;
    // stage rows i0-1 .. i0+32, columns j0-1 .. j0+128: warp w takes rows
    // w, w + 8, ..., its lanes consecutive columns (all loads issued before
    // the first store)
    {
        const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
        constexpr int NR = (RS_TR + 2 + 7) / 8, NC = (RS_TC + 2 + 31) / 32;
        double t[NR][NC];
#pragma unroll
        for (int ri = 0; ri < NR; ++ri) {
            const int rr = wp + 8 * ri, i = i0 - 1 + rr;
#pragma unroll
            for (int ci = 0; ci < NC; ++ci) {
                const int cc = lane + 32 * ci, j = j0 - 1 + cc;
                const bool in = rr < RS_TR + 2 && cc < RS_TC + 2 && (unsigned)i < (unsigned)side &&
                                (unsigned)j < (unsigned)side;
                t[ri][ci] = in ? to_c(u[(size_t)i * side + j]) : 0.0;
            }
        }
#pragma unroll
        for (int ri = 0; ri < NR; ++ri) {
            const int rr = wp + 8 * ri;
#pragma unroll
            for (int ci = 0; ci < NC; ++ci) {
                const int cc = lane + 32 * ci;
                if (rr < RS_TR + 2 && cc < RS_TC + 2) su[rr * RS_LD + cc] = t[ri][ci];
            }
        }
    }
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;     // 32 x 8
    // this thread's f values, requested before the barrier
    double fv[RS_TR / 8][4];
#pragma unroll
    for (int it = 0; it < RS_TR / 8; ++it) {
        const int i = i0 + ty + 8 * it;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
            const int j = j0 + tx + 32 * cc;
            fv[it][cc] = (i < side && j < side) ? to_c(a.f[base + (size_t)i * side + j]) : 0.0;
        }
    }
    __syncthreads();
    const double* c = a.stencil + (size_t)(a.shared ? 0 : b) * 9;
    double cf[9];
#pragma unroll
    for (int d = 0; d < 9; ++d) cf[d] = c[d];
    double acc = 0.0;
#pragma unroll
    for (int it = 0; it < RS_TR / 8; ++it) {
        const int li = ty + 8 * it, i = i0 + li;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
            const int lj = tx + 32 * cc, j = j0 + lj;            // lanes on consecutive columns
            if (i < side && j < side) {
                const double* p = su + (li + 1) * RS_LD + (lj + 1);
                // CSR column order, unfused (apply_op<K_CONST9>)
                double s = cf[0] * p[-RS_LD - 1];
                s = s + cf[1] * p[-RS_LD];
                s = s + cf[2] * p[-RS_LD + 1];
                s = s + cf[3] * p[-1];
                s = s + cf[4] * p[0];
                s = s + cf[5] * p[1];
                s = s + cf[6] * p[RS_LD - 1];
                s = s + cf[7] * p[RS_LD];
                s = s + cf[8] * p[RS_LD + 1];
                const size_t idx = (size_t)i * side + j;
                const double rv = fv[it][cc] - s;
                if (a.r) a.r[base + idx] = to_s<S>(rv);
                acc = fma(rv, rv, acc);
            }
        }
    }
    if (a.partials) {
        const int cta = blockIdx.x + gridDim.x * blockIdx.y;
        write_partial<RS_NT>(a.partials + (size_t)b * gridDim.x * gridDim.y, cta, acc);
    }
}

}  // namespace rg

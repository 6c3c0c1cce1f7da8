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

enum { TRI_SOR = 1, TRI_SSOR = 2, TRI_SOR_T = 3, TRI_SSOR_T = 4 };
// Transposed maps (P.apply_transpose, precond.py:93-94,112-113; the training
// adjoint): (D + wL)^T has row i coupled to rows below at the mirrored
// lower coefficients, so relax (D + wL)^{-T} r is the reverse-order sweep
// with the lower coefficients, and (D + wU)^{-T} the forward sweep with the
// upper ones.
constexpr int TRI_PF = 8;
// rows per pass (threads per CTA); a grid taller than this runs in passes
#ifndef RG_TRI_NT_MAX
#define RG_TRI_NT_MAX 1024
#endif

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
// Memory: at step s every thread touches a different grid row, so direct
// loads/stores cost one L1 line per thread per step (measured ~340 ns per
// wavefront step at 1023 rows).  Instead the steps run in windows of
// TRI_PF: the rhs of window k+1 is fetched into shared memory with
// cp.async while window k computes (each warp copies its own 32 rows, 8
// lanes per row segment, coalesced), every step replaces its rhs slot with
// the result, and the window is written back with coalesced stores.  The
// step body itself touches only registers and shared memory.  Warps whose
// rows have not started or are finished skip the compute (barriers only).
// Arithmetic: x = rhs/d - (l0/d) nm1 - ... with FMAs (the kernel is
// compiled without contraction; these are explicit): a different rounding
// from SuperLU's, agreement ~1e-15, inside the reference's 1e-13 bar.
constexpr int TRI_WS = TRI_PF + 1;   // padded row stride of the staging buffers


template <bool REV, bool MULD, bool SCALE, typename SI, typename SO>
__device__ __forceinline__ void tri_sweep(const SI* __restrict__ src, SO* __restrict__ dst, int side,
                                          int P, double oscale, double l0, double l1, double l2,
                                          double l3, double d, double* edge, double (*xfer)[2],
                                          double* stage) {
    static_assert(sizeof(SI) == 8 || sizeof(SI) == 4, "element size");
    const int t = threadIdx.x, NT = blockDim.x, lane = t & 31, wp = t >> 5;
    const int nw = NT >> 5;
    const double rd = 1.0 / d;
    l0 *= rd;
    l1 *= rd;
    l2 *= rd;
    l3 *= rd;
    // staging: [2][NT][TRI_WS] doubles (f32 inputs are staged as raw 4-byte
    // words in the low half of each slot and widened on use)
    for (int p0 = 0; p0 < side; p0 += NT) {
        const int ip = p0 + t;
        const bool row_ok = ip < side;
        const int nrows = min(NT, side - p0);
        const int nsteps = side + 2 * (nrows - 1);
        const int nwin = (nsteps + TRI_PF - 1) / TRI_PF;
        const int a0 = 2 * 32 * wp;   // lane 0 starts at a0; lane 31 done at a0 + 62 + side
        if (t < nw) xfer[t][0] = xfer[t][1] = 0.0;
        auto gidx = [&](int row, int c) -> long long {   // row: index within the pass
            const long long g = (long long)(p0 + row) * side + c;
            return REV ? (long long)P - 1 - g : g;
        };
        auto idle_win = [&](int k) {
            const int s0 = k * TRI_PF;
            return (s0 + TRI_PF <= a0 - 1) || (s0 > a0 + 62 + side);
        };
        // warp-cooperative window copies: lane -> (row 32 wp + lane/8 + 4 it, slot lane%8)
        auto load_win = [&](int k) {
            double* b = stage + (size_t)(k & 1) * NT * TRI_WS;
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int row = wp * 32 + (lane >> 3) + 4 * it;
                const int c = k * TRI_PF + (lane & 7) - 2 * row;
                const bool ok = p0 + row < side && c >= 0 && c < side;
                cp_async_el<sizeof(SI)>(&b[row * TRI_WS + (lane & 7)], src + (ok ? gidx(row, c) : 0), ok);
            }
            cp_async_commit();
        };
        auto store_win = [&](int k) {
            const double* b = stage + (size_t)(k & 1) * NT * TRI_WS;
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int row = wp * 32 + (lane >> 3) + 4 * it;
                const int c = k * TRI_PF + (lane & 7) - 2 * row;
                if (p0 + row < side && c >= 0 && c < side)
                    dst[gidx(row, c)] = (SO)b[row * TRI_WS + (lane & 7)];
            }
        };
        auto rhs_at = [&](const double* slot) -> double {
            if (sizeof(SI) == 8) return *slot;
            return (double)*reinterpret_cast<const float*>(slot);
        };
        if (!idle_win(0)) load_win(0);
        double left = 0.0, nm1 = 0.0, n0 = 0.0, pub = 0.0;
        // thread 0 starts at column 0 with no warm-up steps: x(i-1, 0) of the
        // previous pass's last row seeds its window (zero for the first pass)
        if (t == 0 && p0 > 0) n0 = edge[0];
        for (int k = 0; k < nwin; ++k) {
            const bool idle = idle_win(k);
            cp_async_wait_all();          // window k's rhs (issued one window ago)
            __syncwarp();
            if (k + 1 < nwin && !idle_win(k + 1)) load_win(k + 1);
            __syncthreads();
            if (idle) {
#pragma unroll
                for (int q = 0; q < TRI_PF - 1; ++q) __syncthreads();
                continue;
            }
            double* b = stage + ((size_t)(k & 1) * NT + t) * TRI_WS;
            const int s0 = k * TRI_PF;
#pragma unroll
            for (int q = 0; q < TRI_PF; ++q) {
                const int s = s0 + q;
                const int jp = s - 2 * t;
                const bool act = row_ok && (unsigned)jp < (unsigned)side;
                // x(i-1, j+1): lane - 1 (shuffle), the previous warp's lane 31
                // (mailbox) or the previous pass's last row (edge); selects
                // instead of a divergent branch
                const double sh = __shfl_up_sync(0xffffffffu, pub, 1);
                const double mb = xfer[wp][(s + 1) & 1];
                const int ce = min(max(jp + 1, 0), side - 1);
                const double ev = (p0 > 0 && (unsigned)(jp + 1) < (unsigned)side) ? edge[ce] : 0.0;
                const double nb = lane != 0 ? sh : (wp > 0 ? mb : ev);
                // x = (rhs - l0 nm1 - l1 n0 - l2 nb - l3 left) / d, as
                // rhs/d - (l/d) x with FMAs: two dependent FMAs per step
                // after the neighbour value arrives
                const double rv = rhs_at(&b[q]);
                double u = MULD ? rv : rv * rd;          // (d y) / d = y for SSOR's D y
                u = __fma_rn(-l0, nm1, u);
                u = __fma_rn(-l1, n0, u);
                u = __fma_rn(-l2, nb, u);
                const double x = act ? __fma_rn(-l3, left, u) : 0.0;
                b[q] = SCALE ? oscale * x : x;
                if (act && t == NT - 1) edge[jp] = x;
                nm1 = n0;
                n0 = nb;
                left = x;
                pub = x;
                if (lane == 31 && wp + 1 < nw) xfer[wp + 1][s & 1] = x;
                if (q + 1 < TRI_PF) __syncthreads();
            }
            __syncwarp();
            store_win(k);
        }
        cp_async_wait_all();
        __syncthreads();
    }
}

template <typename S, int MODE>
__global__ void __launch_bounds__(1024, 1) tri_kernel(const TriArgs<S> a) {
    extern __shared__ double tri_smem[];
    double* stage = tri_smem;                                        // [2][NT][TRI_WS]
    double* edge = tri_smem + 2 * (size_t)blockDim.x * TRI_WS;        // [side]
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
                                            lo3, d, edge, xfer, stage);
    } else if (MODE == TRI_SOR_T) {
        // relax * solve_t(r)  (precond.py:94)
        tri_sweep<true, false, true, S, S>(a.r + base, a.z + base, a.side, a.P, w, lo0, lo1, lo2,
                                           lo3, d, edge, xfer, stage);
    } else if (MODE == TRI_SSOR_T) {
        // c * dlt(diag * dut(r))  (precond.py:112-113)
        const double cc = w * (2.0 - w);
        tri_sweep<false, false, false, S, S>(a.r + base, a.work + base, a.side, a.P, 1.0, up0, up1,
                                             up2, up3, d, edge, xfer, stage);
        __syncthreads();
        tri_sweep<true, true, true, S, S>(a.work + base, a.z + base, a.side, a.P, cc, lo0, lo1, lo2,
                                          lo3, d, edge, xfer, stage);
    } else {
        // c * du(diag * dl(r))  (precond.py:109-110)
        const double cc = w * (2.0 - w);
        tri_sweep<false, false, false, S, S>(a.r + base, a.work + base, a.side, a.P, 1.0, lo0, lo1,
                                             lo2, lo3, d, edge, xfer, stage);
        __syncthreads();
        tri_sweep<true, true, true, S, S>(a.work + base, a.z + base, a.side, a.P, cc, up0, up1, up2,
                                          up3, d, edge, xfer, stage);
    }
}

template <typename S, int MODE>
cudaError_t launch_tri_m(const TriArgs<S>& a, int batch, cudaStream_t st) {
    int nt = (a.side + 31) / 32 * 32;
    if (nt > RG_TRI_NT_MAX) nt = RG_TRI_NT_MAX;
    const size_t smem = (2 * (size_t)nt * TRI_WS + a.side) * sizeof(double);
    auto k = tri_kernel<S, MODE>;
    {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k<<<batch, nt, smem, st>>>(a);
    return cudaGetLastError();
}

template <typename S>
cudaError_t launch_tri(const TriArgs<S>& a, int mode, int batch, cudaStream_t st) {
    switch (mode) {
        case TRI_SOR: return launch_tri_m<S, TRI_SOR>(a, batch, st);
        case TRI_SOR_T: return launch_tri_m<S, TRI_SOR_T>(a, batch, st);
        case TRI_SSOR_T: return launch_tri_m<S, TRI_SSOR_T>(a, batch, st);
        default: return launch_tri_m<S, TRI_SSOR>(a, batch, st);
    }
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

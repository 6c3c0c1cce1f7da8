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
// A thread-block cluster of up to 8 (16) CTAs per system.  A pass covers
// (CTAs x RPC) grid rows, RPC = 128 or 64; compute thread t of CTA c owns row
// p0 + c RPC + t and walks it left to right one point per step.  Inside
// a warp the rows are skewed by two steps (lane l is at column sigma - 2 l
// of the warp's local step sigma) and the row above arrives by warp
// shuffle.  Warps are decoupled: global warp g runs TRI_D = 64 + TRI_PF
// steps behind warp g - 1, TRI_PF more than the dependency needs, so what
// lane 0 of a warp reads from the row above (the last row of the previous
// warp) during a window of TRI_PF steps was produced before that window
// began, and ONE __syncthreads per window (not per step) orders producer
// and consumer.
//
// A lone warp issues in order, so every instruction between two steps of
// the recurrence lengthens it (measured: the bare shuffle + select + 2 DFMA
// step runs at 41 cycles, profiles/micro/fp64_chain.cu).  The compute warps
// therefore do nothing but the recurrence: per window they load their rows'
// TRI_PF right-hand sides and the TRI_PF look-ahead values of the row above
// from shared memory, run TRI_PF steps in registers, and store the TRI_PF
// unscaled results back over the right-hand sides.  Everything else belongs
// to two mover warps per compute warp (a CTA is RPC compute threads,
// RPC write-back threads and RPC fetch threads):
//   * fetch warp: cp.async of the right-hand sides TRI_NBUF - 3 windows
//     ahead (TRI_PF lanes per row segment, coalesced);
//   * write-back warp: coalesced stores of the previous window's results,
//     with the output scale applied on the way;
//   * the hand-off between CTAs: the write-back warp of a CTA's last compute
//     warp copies that warp's last row of the previous window into the
//     boundary buffer of the next CTA (DSMEM, plain 8-byte stores over a
//     sentinel), and the fetch warp of the next CTA's first compute warp
//     polls the columns of the coming window until they have landed.  No
//     cluster barrier, flag or fence is on the path (a release store costs
//     a MEMBAR.ALL.GPU that waits for the warp's outstanding global
//     traffic), and a CTA only ever waits for its predecessor.
// Inside a CTA the row above warp w is simply the staged last row of warp
// w - 1 (windows k - 2 and k - 1, kept alive that long).
//
// A system's ~3.5 side dependent steps thus run on up to 8 (16) SMs with 4 (2)
// compute warps each: SOR at 8 x 1023^2 takes 0.22 ms; the single-CTA,
// barrier-per-step form took 0.80 ms (profiles/ncu_tri_r01.json).  The
// CTAs of a system are chained window by window, so the time is (windows
// of a pass) x (window time of an active CTA): ~1950 cycles per 16-step
// window against ~700 for the bare recurrence; what is left is the movers'
// burst after each barrier (the compute warps' first steps of a window run
// at ~130 cycles while it lasts) and the per-window barrier and loop.
// Contributions are subtracted with FMAs from rhs/d; SuperLU stores the
// lower factor pre-divided by the diagonal and substitutes column by
// column, so results agree to rounding (~1e-15); the reference's own bar
// for these maps is 1e-13 (test_precond.py:33-62).  The backward (upper)
// solve is the same walk in reversed index order.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

namespace rg {
namespace cg = cooperative_groups;

enum { TRI_SOR = 1, TRI_SSOR = 2, TRI_SOR_T = 3, TRI_SSOR_T = 4 };
// Transposed maps (P.apply_transpose, precond.py:93-94,112-113; the training
// adjoint): (D + wL)^T has row i coupled to rows below at the mirrored
// lower coefficients, so relax (D + wL)^{-T} r is the reverse-order sweep
// with the lower coefficients, and (D + wU)^{-T} the forward sweep with the
// upper ones.
#ifndef RG_TRI_SKIP
#define RG_TRI_SKIP 0  // timing experiments only: bit 0 no fetch, bit 1 no write-back, bit 2 no CTA hand-off, bit 3 no compute
#endif
#ifndef RG_TRI_PF
#define RG_TRI_PF 16
#endif
#ifndef RG_TRI_L2PF
#define RG_TRI_L2PF 0                   // windows of L2 prefetch distance beyond the cp.async depth (0: none; measured no gain)
#endif
#ifndef RG_TRI_NBUF
#define RG_TRI_NBUF 8                   // staging buffers (power of two): cp.async runs NBUF - 3 windows ahead
#endif
constexpr int TRI_NBUF = RG_TRI_NBUF;
constexpr int TRI_AHEAD = TRI_NBUF - 3; // a buffer is refilled two windows after its write-back
constexpr int TRI_PF = RG_TRI_PF;       // steps per window (8 or 16)
constexpr int TRI_WS = TRI_PF + 2;      // staged row stride: 16-byte aligned rows, conflict-free 128-bit access
constexpr int TRI_D = 64 + TRI_PF;      // steps a warp lags its predecessor
// rows (compute threads) per CTA are a template parameter RPC: 128 (clusters
// of up to 8 CTAs) or 64 (up to 16 CTAs, the non-portable cluster size: half
// the movers' burst per SM; chosen when the device can hold all the batch's
// clusters at once, cudaOccupancyMaxActiveClusters)
static_assert(TRI_NBUF >= 4 && (TRI_NBUF & (TRI_NBUF - 1)) == 0, "staging depth");

template <typename S>
struct TriArgs {
    const double* stencil;  // CONST9 [B or 1][9]
    int shared;
    int side, P;
    double relax;
    const S* r;
    S* z;
    S* work;                // SSOR: forward result [B][P]
    int nc;                 // CTAs per cluster
};

template <typename SI>
__device__ __forceinline__ double tri_rhs(double slot) {
    if (sizeof(SI) == 8) return slot;
    return (double)__int_as_float(__double2loint(slot));   // f32 staged raw in the low word
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// Sentinel of the cross-CTA hand-off: a quiet NaN with a payload no
// arithmetic produces.  The consumer CTA arms its boundary buffer with it,
// the producer overwrites it with plain 8-byte DSMEM stores (single-copy
// atomic), and the consumer re-reads a column until it is no longer the
// sentinel.  Should an input carry this very NaN, the bounded spin accepts
// it (the result is NaN either way).
constexpr unsigned long long TRI_SENT = 0xFFF8B200DEAD0001ULL;
constexpr int TRI_SPIN_MAX = 1 << 22;
__device__ __forceinline__ double ld_volatile_shared(const double* p) {
    double v;
    asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ bool tri_is_sent(double v) {
    return (unsigned long long)__double_as_longlong(v) == TRI_SENT;
}
__device__ __forceinline__ void tri_arm(double* bnd, int side) {
    for (int i = threadIdx.x; i < side; i += blockDim.x) bnd[i] = __longlong_as_double((long long)TRI_SENT);
}

// boundary index of column col: shifted by one so that the TRI_PF look-ahead
// columns of a window are 16-byte aligned
__device__ __forceinline__ int tri_bnd_idx(int col, int side) { return col ? col - 1 : side - 1; }

struct TriShared {
    double* stage;   // [TRI_NBUF][RPC][TRI_WS]: right-hand sides, then unscaled results
    double* bnd;     // [side]: the row above this CTA's first row (previous CTA / previous pass)
};

// One substitution sweep: dst = oscale * x where M x = rhs, M lower
// triangular in traversal order (reversed index order when REV).
// rhs = src, or d * src when MULD (SSOR's D * y).  Coefficients in
// traversal order: l0 (i-1, j-1), l1 (i-1, j), l2 (i-1, j+1), l3 (i, j-1).
// Windows in which all 32 lanes of a warp are inside the grid run
// predicate-free.
template <int RPC, bool REV, bool MULD, bool SCALE, typename SI, typename SO>
__device__ __forceinline__ void tri_sweep(cg::cluster_group& cl, const SI* __restrict__ src,
                                          SO* __restrict__ dst, int side, int P, double oscale,
                                          double l0, double l1, double l2, double l3, double d,
                                          const TriShared& sm, int nc) {
    static_assert(sizeof(SI) == 8 || sizeof(SI) == 4, "element size");
    constexpr int NCW = RPC / 32;            // compute warps per CTA
    const int crank = (int)cl.block_rank();
    const int lane = threadIdx.x & 31;
    const int role = threadIdx.x / RPC;                      // 0 compute, 1 write-back, 2 fetch
    const bool mover = role > 0, storer = role == 1, loader = role == 2;
    const int wp = (threadIdx.x >> 5) - role * NCW;          // compute warp (owned or served)
    const int t = wp * 32 + lane;                                // row within the CTA
    const int gw = crank * NCW + wp;                         // global warp of the pass
    const int RPP = nc * RPC;                                // rows per pass
    const double rd = 1.0 / d;
    const double m0 = -(l0 * rd), m1 = -(l1 * rd), m2 = -(l2 * rd), m3 = -(l3 * rd);
    const int a0 = TRI_D * gw;              // lane 0 is at column s - a0 at step s
    const int shift = a0 + 2 * lane;        // this row: column s - shift
    // movers: element (row 32 wp + r8 + RPI it, slot) of window k is column
    // c0 - 2 RPI it + TRI_PF k
    constexpr int LPR = TRI_PF;              // lanes per row segment
    constexpr int RPI = 32 / LPR;            // rows per copy instruction
    constexpr int NIT = 32 / RPI;            // copy instructions per window
    const int r8 = lane / LPR, slot = lane % LPR;
    const int c0 = slot - a0 - 2 * r8;
    const long long gstride = (long long)RPI * side - 2 * RPI;
    const long long gs = REV ? -gstride : gstride;
    const int dk = REV ? -TRI_PF : TRI_PF;
    double* stage = sm.stage;
    auto buf = [&](int k) { return stage + (size_t)(k & (TRI_NBUF - 1)) * RPC * TRI_WS; };
    const bool cta_first = wp == 0, cta_last = wp == NCW - 1;
    double* bnd_next = cl.map_shared_rank(sm.bnd, crank + 1 < nc ? crank + 1 : 0);
    for (int p0 = 0; p0 < side; p0 += RPP) {
        const int row = p0 + crank * RPC + t;                  // traversal-order grid row
        const int wrow0 = row - lane;                              // first row of the warp
        const bool row_ok = row < side;
        const int nrows = min(RPP, side - p0);
        const int last = nrows - 1;
        const int nsteps = side + TRI_D * (last >> 5) + 2 * (last & 31);
        const int nwin = (nsteps + TRI_PF - 1) / TRI_PF;
        // the warp's last row goes to the next CTA, or (last CTA) to CTA 0 for the next pass
        const bool pushes = cta_last && wrow0 + 31 < side &&
                            (crank + 1 < nc ? wrow0 + 32 < side : p0 + RPP < side);
        const bool polls = cta_first && crank > 0;                 // row above comes from the previous CTA
        const bool has_above = wp > 0 || crank > 0 || p0 > 0;
        const long long g0 = (long long)(wrow0 + r8) * side + c0;
        const SI* sp = src + (REV ? (long long)P - 1 - g0 : g0);
        SO* dp = dst + (REV ? (long long)P - 1 - g0 : g0);
        // window k of this warp: idle (nothing of the warp inside the grid,
        // not even lane 0's warm-up step), or interior (every lane inside
        // for all TRI_PF steps, and lane 0's look-ahead column too)
        // (as window ranges, so that the per-window tests are two compares:
        //  idle: s0 + PF <= -1 or s0 > 62 + side - 1 with s0 = k PF - a0;
        //  interior: s0 >= 62 and s0 + PF <= side - 1, all 32 rows inside)
        int k_first = max(0, (a0 - TRI_PF) / TRI_PF);
        while (k_first * TRI_PF - a0 + TRI_PF <= -1) ++k_first;
        int k_last = min(nwin - 1, (a0 + 61 + side) / TRI_PF);
        if (wrow0 >= side) k_last = -1;
        int i_first = (a0 + 62 + TRI_PF - 1) / TRI_PF;
        int i_last = (a0 + side - 1 - TRI_PF) / TRI_PF;
        if (wrow0 + 31 >= side || a0 + side - 1 - TRI_PF < 0) i_last = -1;
        auto idle_win = [&](int k) { return k < k_first || k > k_last; };
        auto interior = [&](int k) { return k >= i_first && k <= i_last; };
        auto load_win = [&](int k) {     // rhs of window k -> its staging buffer
            double* b = buf(k) + (size_t)(wp * 32 + r8) * TRI_WS + slot;
            const SI* s = sp + (long long)k * dk;
            if (interior(k)) {
#pragma unroll
                for (int it = 0; it < NIT; ++it)
                    cp_async_el<sizeof(SI)>(b + it * RPI * TRI_WS, s + it * gs, true);
            } else {
#pragma unroll
                for (int it = 0; it < NIT; ++it) {
                    const int c = c0 - 2 * RPI * it + k * TRI_PF;
                    const bool ok = wrow0 + r8 + RPI * it < side && (unsigned)c < (unsigned)side;
                    cp_async_el<sizeof(SI)>(b + it * RPI * TRI_WS, ok ? s + it * gs : src, ok);
                }
            }
        };
        auto store_win = [&](int k) {    // results of window k -> dst
            const double* b = buf(k) + (size_t)(wp * 32 + r8) * TRI_WS + slot;
            SO* o = dp + (long long)k * dk;
            if (interior(k)) {
                double x[NIT];
#pragma unroll
                for (int it = 0; it < NIT; ++it) x[it] = b[it * RPI * TRI_WS];
#pragma unroll
                for (int it = 0; it < NIT; ++it) o[it * gs] = (SO)(SCALE ? oscale * x[it] : x[it]);
            } else {
#pragma unroll
                for (int it = 0; it < NIT; ++it) {
                    const int c = c0 - 2 * RPI * it + k * TRI_PF;
                    if (wrow0 + r8 + RPI * it < side && (unsigned)c < (unsigned)side) {
                        const double x = b[it * RPI * TRI_WS];
                        o[it * gs] = (SO)(SCALE ? oscale * x : x);
                    }
                }
            }
        };
        auto prefetch_win = [&](int k) { // one lane per row: window k's segment -> L2
            int c = k * TRI_PF - shift;
            if (!row_ok || c + TRI_PF <= 0 || c >= side) return;
            c = max(c, 0);
            const long long g = (long long)row * side + c;
            prefetch_l2(src + (REV ? (long long)P - 1 - g : g));
        };
        auto push_win = [&](int k) {     // last row of window k -> the next CTA's boundary buffer
            if (lane < TRI_PF) {
                const int col = k * TRI_PF + lane - a0 - 62;
                if ((unsigned)col < (unsigned)side)
                    bnd_next[tri_bnd_idx(col, side)] = buf(k)[(size_t)(wp * 32 + 31) * TRI_WS + lane];
            }

        };
        auto poll_win = [&](int k) {     // look-ahead columns of window k have landed
            if (lane < TRI_PF) {
                const int col = k * TRI_PF + lane - a0 + 1;
                if ((unsigned)col < (unsigned)side) {
                    const double* q = sm.bnd + tri_bnd_idx(col, side);
                    for (int spin = 0; spin < TRI_SPIN_MAX; ++spin)
                        if (!tri_is_sent(ld_volatile_shared(q))) break;
                }
            }
            __syncwarp();
        };
        double left = 0.0, nm1 = 0.0, n0 = 0.0, pub = 0.0;
        if (loader) {
            for (int k = 0; k < TRI_AHEAD; ++k) {
                if (!idle_win(k)) load_win(k);
                cp_async_commit();
            }
            if (polls && !idle_win(0)) poll_win(0);
        } else if (storer) {
        } else if (t == 0 && crank == 0 && p0 > 0) {
            // the pass's first row starts at column 0 with no warm-up step:
            // x(i-1, 0) of the previous pass's last row seeds its window
            n0 = sm.bnd[tri_bnd_idx(0, side)];
        }
        // window k: [barrier] the movers hand on and write back window k-1
        // and fetch window k + AHEAD (into the buffer window k-3 left) while
        // the owners compute window k; one extra round drains
        for (int k = 0; k <= nwin; ++k) {
            if (loader) cp_async_wait_group<TRI_AHEAD - 1>();  // window k's rhs has landed
            __syncthreads();                                   // + results of window k-1 visible
            if (mover) {
                if ((RG_TRI_SKIP & 1) && loader) continue;
                if (storer) {
                    if (!idle_win(k - 1)) {
                        if (pushes && !(RG_TRI_SKIP & 4)) push_win(k - 1);
                        if (!(RG_TRI_SKIP & 2)) store_win(k - 1);
                    }
                } else {
                    if (!idle_win(k + TRI_AHEAD)) load_win(k + TRI_AHEAD);
                    cp_async_commit();
                    if (RG_TRI_L2PF > 0) prefetch_win(k + TRI_AHEAD + RG_TRI_L2PF);
                    if (polls && !idle_win(k + 1) && !(RG_TRI_SKIP & 4)) poll_win(k + 1);
                }
                continue;
            }
            if (RG_TRI_SKIP & 8) continue;
            if (idle_win(k)) continue;
            const int s0 = k * TRI_PF;
            double2* b2 = reinterpret_cast<double2*>(buf(k) + (size_t)t * TRI_WS);
            double raw[TRI_PF], rb[TRI_PF];
#pragma unroll
            for (int q = 0; q < TRI_PF; q += 2) {
                const double2 v = b2[q >> 1];
                raw[q] = v.x;
                raw[q + 1] = v.y;
            }
            if (interior(k)) {
                // x(i-1, j+1) for lane 0 over the window: columns
                // s0 - a0 + 1 + q of the row above
                if (wp > 0) {
                    // previous warp's last row: its lane 31 computed column
                    // s0 - a0 + 1 + q at step s0 + q - 1 - TRI_PF, i.e. the last
                    // slot of window k - 2 for q = 0, slot q - 1 of window k - 1
                    // after that
                    const double* pr2 = buf(k - 2) + (size_t)(wp * 32 - 1) * TRI_WS;
                    const double* pr1 = buf(k - 1) + (size_t)(wp * 32 - 1) * TRI_WS;
                    rb[0] = pr2[TRI_PF - 1];
#pragma unroll
                    for (int q = 1; q + 1 < TRI_PF; q += 2) {
                        const double2 v = *reinterpret_cast<const double2*>(pr1 + q - 1);
                        rb[q] = v.x;
                        rb[q + 1] = v.y;
                    }
                    rb[TRI_PF - 1] = pr1[TRI_PF - 2];
                } else if (has_above) {
                    const double2* r2 = reinterpret_cast<const double2*>(sm.bnd + (s0 - a0));
#pragma unroll
                    for (int q = 0; q < TRI_PF; q += 2) {
                        const double2 v = r2[q >> 1];
                        rb[q] = v.x;
                        rb[q + 1] = v.y;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < TRI_PF; ++q) rb[q] = 0.0;
                }
#pragma unroll
                for (int q = 0; q < TRI_PF; ++q) {
                    const double sh = __shfl_up_sync(0xffffffffu, pub, 1);
                    const double nb = lane != 0 ? sh : rb[q];
                    const double rv = tri_rhs<SI>(raw[q]);
                    double u = MULD ? rv : rv * rd;          // (d y) / d = y for SSOR's D y
                    u = __fma_rn(m0, nm1, u);
                    u = __fma_rn(m1, n0, u);
                    u = __fma_rn(m3, left, u);
                    const double x = __fma_rn(m2, nb, u);   // the value that arrives last goes last
                    raw[q] = x;
                    nm1 = n0;
                    n0 = nb;
                    left = x;
                    pub = x;
                }
            } else {
                if (wp > 0) {
                    // same slots as above; columns outside the grid were not
                    // computed by the row above (stale slots): masked to zero
                    const double* pr2 = buf(k - 2) + (size_t)(wp * 32 - 1) * TRI_WS;
                    const double* pr1 = buf(k - 1) + (size_t)(wp * 32 - 1) * TRI_WS;
                    rb[0] = pr2[TRI_PF - 1];
#pragma unroll
                    for (int q = 1; q + 1 < TRI_PF; q += 2) {
                        const double2 v = *reinterpret_cast<const double2*>(pr1 + q - 1);
                        rb[q] = v.x;
                        rb[q + 1] = v.y;
                    }
                    rb[TRI_PF - 1] = pr1[TRI_PF - 2];
#pragma unroll
                    for (int q = 0; q < TRI_PF; ++q)
                        if ((unsigned)(s0 + q - a0 + 1) >= (unsigned)side) rb[q] = 0.0;
                } else {
#pragma unroll
                    for (int q = 0; q < TRI_PF; ++q) {
                        const int col = s0 + q - a0 + 1;
                        rb[q] = 0.0;
                        if (has_above && (unsigned)col < (unsigned)side) rb[q] = sm.bnd[tri_bnd_idx(col, side)];
                    }
                }
#pragma unroll
                for (int q = 0; q < TRI_PF; ++q) {
                    const int jp = s0 + q - shift;
                    const bool act = row_ok && (unsigned)jp < (unsigned)side;
                    const double sh = __shfl_up_sync(0xffffffffu, pub, 1);
                    const double nb = lane != 0 ? sh : rb[q];
                    const double rv = tri_rhs<SI>(raw[q]);
                    double u = MULD ? rv : rv * rd;
                    u = __fma_rn(m0, nm1, u);
                    u = __fma_rn(m1, n0, u);
                    u = __fma_rn(m3, left, u);
                    const double x = act ? __fma_rn(m2, nb, u) : 0.0;
                    raw[q] = x;
                    nm1 = n0;
                    n0 = nb;
                    left = x;
                    pub = x;
                }
            }
#pragma unroll
            for (int q = 0; q < TRI_PF; q += 2) b2[q >> 1] = make_double2(raw[q], raw[q + 1]);
        }
        if (loader) cp_async_wait_all();
        // passes and sweeps: boundary rows handed to CTA 0 and global results
        // must be complete before anyone starts the next one, and the
        // boundary buffers of CTAs >= 1 (fully consumed by now) are armed
        // again before their producers restart
        if (nc > 1) {
            __syncthreads();
            if (crank > 0) tri_arm(sm.bnd, side);
            cl.sync();
        } else {
            __syncthreads();
        }
    }
}

template <typename S, int MODE, int RPC>
__global__ void __launch_bounds__(3 * RPC, 1) tri_kernel(const TriArgs<S> a) {
    extern __shared__ double tri_smem[];
    cg::cluster_group cl = cg::this_cluster();
    TriShared sm;
    sm.stage = tri_smem;                                          // [TRI_NBUF][RPC][TRI_WS]
    sm.bnd = sm.stage + (size_t)TRI_NBUF * RPC * TRI_WS;      // [side + 1]
    if (a.nc > 1) {
        if (cl.block_rank() > 0) tri_arm(sm.bnd, a.side);
        cl.sync();                                                // armed before any producer store lands
    }
    const int b = blockIdx.x / a.nc;
    const double* c = a.stencil + (size_t)(a.shared ? 0 : b) * 9;
    const double w = a.relax;
    // DL = diag + relax * tril(A, -1), DU = diag + relax * triu(A, 1) (precond.py:91,104-105)
    const double d = c[4];
    const double lo0 = w * c[0], lo1 = w * c[1], lo2 = w * c[2], lo3 = w * c[3];
    const double up0 = w * c[8], up1 = w * c[7], up2 = w * c[6], up3 = w * c[5];
    const size_t base = (size_t)b * a.P;
    if (MODE == TRI_SOR) {
        // relax * solve(r)  (precond.py:93)
        tri_sweep<RPC, false, false, true, S, S>(cl, a.r + base, a.z + base, a.side, a.P, w, lo0, lo1, lo2,
                                            lo3, d, sm, a.nc);
    } else if (MODE == TRI_SOR_T) {
        // relax * solve_t(r)  (precond.py:94)
        tri_sweep<RPC, true, false, true, S, S>(cl, a.r + base, a.z + base, a.side, a.P, w, lo0, lo1, lo2,
                                           lo3, d, sm, a.nc);
    } else if (MODE == TRI_SSOR_T) {
        // c * dlt(diag * dut(r))  (precond.py:112-113)
        const double cc = w * (2.0 - w);
        tri_sweep<RPC, false, false, false, S, S>(cl, a.r + base, a.work + base, a.side, a.P, 1.0, up0, up1,
                                             up2, up3, d, sm, a.nc);
        tri_sweep<RPC, true, true, true, S, S>(cl, a.work + base, a.z + base, a.side, a.P, cc, lo0, lo1, lo2,
                                          lo3, d, sm, a.nc);
    } else {
        // c * du(diag * dl(r))  (precond.py:109-110)
        const double cc = w * (2.0 - w);
        tri_sweep<RPC, false, false, false, S, S>(cl, a.r + base, a.work + base, a.side, a.P, 1.0, lo0, lo1,
                                             lo2, lo3, d, sm, a.nc);
        tri_sweep<RPC, true, true, true, S, S>(cl, a.work + base, a.z + base, a.side, a.P, cc, up0, up1, up2,
                                          up3, d, sm, a.nc);
    }
}

template <typename S, int MODE, int RPC>
cudaError_t launch_tri_r(TriArgs<S> a, int batch, cudaStream_t st, bool probe_only, int* max_clusters) {
    constexpr int MAXC = RPC == 64 ? 16 : 8;
    a.nc = (a.side + RPC - 1) / RPC;
    if (a.nc > MAXC) a.nc = MAXC;
    const size_t smem = ((size_t)TRI_NBUF * RPC * TRI_WS + a.side + 1) * sizeof(double);
    auto k = tri_kernel<S, MODE, RPC>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (a.nc > 8) {
        e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(batch * a.nc, 1, 1);
    cfg.blockDim = dim3(3 * RPC, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.nc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (probe_only) return cudaOccupancyMaxActiveClusters(max_clusters, k, &cfg);
    return cudaLaunchKernelEx(&cfg, k, a);
}

// 64 rows per CTA when every cluster of the batch is resident at once (the
// chained CTAs of a system then carry half the data movement each: SOR at
// 1 x 1023^2 219 -> 180 us, 8 x 1023^2 221 -> 213 us, 4 x 2047^2 561 ->
// 441 us); otherwise 128 rows per CTA, half as many CTAs per system.
template <typename S, int MODE>
cudaError_t launch_tri_m(const TriArgs<S>& a, int batch, cudaStream_t st) {
    static const int force = [] { const char* e = getenv("RG_TRI_RPC"); return e ? atoi(e) : 0; }();
    if (force != 128 && a.side > 32) {
        int fit = 0;
        if (force == 64 ||
            (launch_tri_r<S, MODE, 64>(a, batch, st, true, &fit) == cudaSuccess && fit >= batch))
            return launch_tri_r<S, MODE, 64>(a, batch, st, false, nullptr);
        cudaGetLastError();
    }
    return launch_tri_r<S, MODE, 128>(a, batch, st, false, nullptr);
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

// instantiated in tri.cu (parallel build)
extern template cudaError_t launch_tri<double>(const TriArgs<double>&, int, int, cudaStream_t);
extern template cudaError_t launch_tri<float>(const TriArgs<float>&, int, int, cudaStream_t);

}  // namespace rg

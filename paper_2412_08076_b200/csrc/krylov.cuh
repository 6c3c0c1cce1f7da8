// krylov.cuh — fused modified Gram-Schmidt step for the FGMRES driver
// (fgmres.py:76-78).
//
// One launch per orthogonalisation index i applies the previous projection
// and takes the next inner product in a single pass over w:
//     w <- w - h_{i-1} v_{i-1}        (numpy: w - H[i-1,k] * V[:, i-1])
//     h_i = vdot(v_i, w)              (conj(v_i) . w)
// plus, on the last call, ||w||^2.  4 vectors of traffic per index instead
// of the ~10 of separate vdot / mul / sub.  Per-CTA partials are summed in
// a fixed order by a second tiny kernel (deterministic; not BLAS-bitwise).
#pragma once
#include "reduce.cuh"

namespace rg {

constexpr int MGS_NT = 256;

__device__ __forceinline__ double2 conj_mul(double2 a, double2 b) {   // conj(a) * b
    return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double conj_mul(double a, double b) { return a * b; }
__device__ __forceinline__ double2 acc_add(double2 s, double2 t) { return make_double2(s.x + t.x, s.y + t.y); }
__device__ __forceinline__ double acc_add(double s, double t) { return s + t; }

template <typename S>
struct MgsArgs {
    S* w; long long ldw;
    const S* v; long long ldv;     // previous basis vector (null: no projection)
    const S* h;                    // [B] previous coefficient
    const S* vn; long long ldvn;   // next basis vector (null: no dot)
    double* part;                  // [B][ncta][3]: dot (re, im), ||w||^2
    int n;
    int want_norm;
    int* counter;                  // [B] last-CTA tickets (null: separate finish kernel)
    S* hn;                         // fused finish outputs (with counter)
    double* wnorm2;
};

template <typename S>
__global__ void __launch_bounds__(MGS_NT) mgs_kernel(MgsArgs<S> a) {
    __shared__ double red[MGS_NT / 32];
    __shared__ int is_last;
    const int b = blockIdx.y;
    S* w = a.w + b * a.ldw;
    const S* v = a.v ? a.v + b * a.ldv : nullptr;
    const S* vn = a.vn ? a.vn + b * a.ldvn : nullptr;
    const S hb = a.v ? a.h[b] : szero<S>();
    S dot = szero<S>();
    double nn = 0.0;
    for (int j = blockIdx.x * MGS_NT + threadIdx.x; j < a.n; j += gridDim.x * MGS_NT) {
        S x = w[j];
        if (v) {
            x = sub(x, mul(hb, v[j]));
            w[j] = x;
        }
        if (vn) dot = acc_add(dot, conj_mul(vn[j], x));
        if (a.want_norm) nn = sqacc(nn, x);
    }
    double* part = a.part + ((size_t)b * gridDim.x + blockIdx.x) * 3;
    double re, im = 0.0;
    if constexpr (sizeof(S) == 16) { re = dot.x; im = dot.y; } else { re = dot; }
    const double r0 = block_sum<MGS_NT>(re, red);
    const double r1 = block_sum<MGS_NT>(im, red);
    const double r2 = block_sum<MGS_NT>(nn, red);
    if (threadIdx.x == 0) { part[0] = r0; part[1] = r1; part[2] = r2; }
    if (!a.counter) return;
    // fused finish: the last CTA of system b sums the partials in a fixed
    // order (deterministic whichever CTA arrives last)
    if (threadIdx.x == 0) {
        __threadfence();
        is_last = atomicAdd(&a.counter[b], 1) == (int)gridDim.x - 1;
        if (is_last) __threadfence();
    }
    __syncthreads();
    if (!is_last) return;
    const double* pb = a.part + (size_t)b * gridDim.x * 3;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int c = threadIdx.x; c < (int)gridDim.x; c += MGS_NT) {
        s0 += __ldcg(&pb[c * 3]); s1 += __ldcg(&pb[c * 3 + 1]); s2 += __ldcg(&pb[c * 3 + 2]);
    }
    s0 = block_sum<MGS_NT>(s0, red);
    s1 = block_sum<MGS_NT>(s1, red);
    s2 = block_sum<MGS_NT>(s2, red);
    if (threadIdx.x == 0) {
        if (a.hn) {
            if constexpr (sizeof(S) == 16) a.hn[b] = make_double2(s0, s1);
            else a.hn[b] = s0;
        }
        if (a.wnorm2) a.wnorm2[b] = s2;
        a.counter[b] = 0;
        __threadfence();
    }
}

template <typename S>
__global__ void __launch_bounds__(MGS_NT) mgs_finish_kernel(const double* part, int ncta, S* hn,
                                                            double* wnorm2) {
    __shared__ double red[MGS_NT / 32];
    const int b = blockIdx.x;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int c = threadIdx.x; c < ncta; c += MGS_NT) {
        const double* p = part + ((size_t)b * ncta + c) * 3;
        s0 += p[0]; s1 += p[1]; s2 += p[2];
    }
    s0 = block_sum<MGS_NT>(s0, red);
    s1 = block_sum<MGS_NT>(s1, red);
    s2 = block_sum<MGS_NT>(s2, red);
    if (threadIdx.x == 0) {
        if (hn) {
            if constexpr (sizeof(S) == 16) hn[b] = make_double2(s0, s1);
            else hn[b] = s0;
        }
        if (wnorm2) wnorm2[b] = s2;
    }
}

// ---- persistent MGS: one cooperative launch per Arnoldi orthogonalisation.
// Each CTA (one per SM) keeps its slice of w AND of the current basis vector
// in shared memory for all k + 2 passes of a system, so a pass streams only
// the next basis vector from HBM; the dot products finish with a software
// grid barrier after which every CTA sums the per-CTA partials in the same
// fixed order (identical, deterministic h_i in every CTA, no second barrier).
// Same arithmetic per element as mgs_kernel (w -= h v, conj(v) . w).
constexpr int MGSP_NT = 512;            // 1024 threads x 7 elements measured slower (0.85 vs 0.77 ms at k = 19)

struct GridBar {
    unsigned int* count;   // arrivals of the current phase
    unsigned int* gen;     // phase counter
};

__device__ __forceinline__ void grid_barrier(const GridBar& g, unsigned int& phase) {
    __syncthreads();
    if (threadIdx.x == 0) {
        ++phase;
        __threadfence();
        const unsigned int arrived = atomicAdd(g.count, 1u) + 1u;
        if (arrived == gridDim.x) {
            *g.count = 0u;
            __threadfence();
            atomicExch(g.gen, phase);
        } else {
            while (true) {
                unsigned int cur;
                asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(g.gen) : "memory");
                if ((int)(cur - phase) >= 0) break;
                __nanosleep(32);
            }
        }
        __threadfence();
    }
    __syncthreads();
}

template <typename S>
struct MgsPArgs {
    S* w; long long ldw;
    const S* V; long long ldv;     // basis v_i of system b at V + b*ldv + i*n
    S* H;                          // [k+1][B]
    double* wnorm2;                // [B]
    double* part;                  // [2][gridDim][MGSP_NV]
    GridBar bar;
    int n, k, B, slice;
};

constexpr int MGSP_R = 16;          // most slice elements per thread (slice <= MGSP_NT * MGSP_R); 12 and 14 have instantiations too
constexpr int MGSP_NV = 6;          // partial sums per CTA and phase

// Sum NV values over the CTA in a fixed order (warp shuffles, one row per
// warp; then NV groups of 32 lanes add the rows, all values at once); every
// thread gets the totals.
template <int NT, int NV>
__device__ __forceinline__ void block_sum_n(double (&v)[NV], double (*red)[NV], double* out) {
    static_assert(NT / 32 <= 32 && NV * 32 <= NT, "one 32-lane group per value");
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_down_sync(0xffffffffu, v[j], o);
    __syncthreads();                       // red / out of the previous use are free
    if (lane == 0)
#pragma unroll
        for (int j = 0; j < NV; ++j) red[wp][j] = v[j];
    __syncthreads();
    if (wp < NV) {                         // warp j adds value j over the NT / 32 rows
        double x = lane < NT / 32 ? red[lane][wp] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) out[wp] = x;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = out[j];
}

// Fused-multiply-add forms for the Krylov kernels (the library is compiled
// without contraction for the stencil sums; nothing here is compared
// bitwise -- the reference's dots go through BLAS): acc + conj(a) b and
// x - h v.
__device__ __forceinline__ double2 dot_acc(double2 acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y); acc.y = fma(-a.y, b.x, acc.y);
    return acc;
}
__device__ __forceinline__ double dot_acc(double acc, double a, double b) { return fma(a, b, acc); }
__device__ __forceinline__ double2 sub_mul(double2 x, double2 h, double2 v) {
    x.x = fma(-h.x, v.x, x.x); x.x = fma(h.y, v.y, x.x);
    x.y = fma(-h.x, v.y, x.y); x.y = fma(-h.y, v.x, x.y);
    return x;
}
__device__ __forceinline__ double sub_mul(double x, double h, double v) { return fma(-h, v, x); }

// One prefetch.global.L2 per 128-byte line of a CTA's slice.
template <typename S>
__device__ __forceinline__ void l2_prefetch_slice(const S* p, int cnt) {
    constexpr int EPL = 128 / sizeof(S);
    for (int q = threadIdx.x * EPL; q < cnt; q += MGSP_NT * EPL)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p + q));
}

// The basis vectors are taken two per phase.  For the pair (v_i, v_{i+1})
// one pass over the slice yields a = <v_i, w>, b = <v_{i+1}, w> and the
// Gram entry c = <v_{i+1}, v_i>; after the grid barrier
//     h_i = a,   h_{i+1} = b - h_i c  = <v_{i+1}, w - h_i v_i>
// which is the modified Gram-Schmidt coefficient itself (fgmres.py:76-78),
// not the classical one: c is the exact correction (it is ~1e-16 for an
// orthonormal basis, so the two forms differ far below rounding).  Both
// projections are then subtracted in MGS order at the start of the next
// phase, w <- (w - h_i v_i) - h_{i+1} v_{i+1}, with v_i kept in shared
// memory and v_{i+1} in registers: the number of grid-wide reductions per
// system drops from k + 2 to ceil((k + 1) / 2) + 1.
template <typename S, int R_>
__global__ void __launch_bounds__(MGSP_NT, 1) mgs_persist_kernel(MgsPArgs<S> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S* ws = reinterpret_cast<S*>(smem_raw);           // [slice] this CTA's w
    S* vs = ws + a.slice;                              // [slice] this CTA's v_i (first of the pair)
    __shared__ double red[MGSP_NT / 32][MGSP_NV];
    __shared__ double tot[MGSP_NV];
    constexpr bool CPLX = sizeof(S) == 16;
    const int j0 = blockIdx.x * a.slice;
    const int cnt = max(0, min(a.n, j0 + a.slice) - j0);
    unsigned int phase = 0;
    if (threadIdx.x == 0) phase = *a.bar.gen;          // barrier phases continue from here
    int par = 0;                                       // partial-sum buffer parity
    // sum the per-CTA partials of this phase: every CTA adds them in the same
    // order; the other parity buffer is written next, so one barrier suffices
    auto reduce_all = [&](double (&v)[MGSP_NV]) {
        block_sum_n<MGSP_NT, MGSP_NV>(v, red, tot);
        double* part = a.part + (size_t)par * MGSP_NV * gridDim.x;
        if (threadIdx.x < MGSP_NV) part[(size_t)blockIdx.x * MGSP_NV + threadIdx.x] = v[threadIdx.x];
        grid_barrier(a.bar, phase);     // cooperative_groups grid.sync() measured the same
#pragma unroll
        for (int j = 0; j < MGSP_NV; ++j) v[j] = 0.0;
        for (int c = threadIdx.x; c < (int)gridDim.x; c += MGSP_NT)
#pragma unroll
            for (int j = 0; j < MGSP_NV; ++j) v[j] += __ldcg(&part[(size_t)c * MGSP_NV + j]);
        block_sum_n<MGSP_NT, MGSP_NV>(v, red, tot);
        par ^= 1;
    };
    for (int b = 0; b < a.B; ++b) {
        S* w = a.w + b * a.ldw + j0;
        const S* Vb = a.V + b * a.ldv + j0;
        S hA = szero<S>(), hB = szero<S>();
        S vrB[R_];
        bool prevB = false;
        {
            S wr[R_];
#pragma unroll
            for (int r = 0; r < R_; ++r) {
                const int q = threadIdx.x + r * MGSP_NT;
                if (q < cnt) wr[r] = w[q];
            }
#pragma unroll
            for (int r = 0; r < R_; ++r) {
                const int q = threadIdx.x + r * MGSP_NT;
                if (q < cnt) ws[q] = wr[r];
            }
        }
        for (int i = 0; i <= a.k; i += 2) {
            const bool two = i + 1 <= a.k;
            if (i > 0) {
#pragma unroll
                for (int r = 0; r < R_; ++r) {
                    const int q = threadIdx.x + r * MGSP_NT;
                    if (q < cnt) {
                        S x = sub_mul(ws[q], hA, vs[q]);             // w -= h_{i-2} v_{i-2}
                        if (prevB) x = sub_mul(x, hB, vrB[r]);       // w -= h_{i-1} v_{i-1}
                        ws[q] = x;
                    }
                }
            }
            // v_i -> shared memory (every thread copies and later reads only
            // its own elements), v_{i+1} -> registers
            const S* vA = Vb + (size_t)i * a.n;
            const S* vB = vA + a.n;
#pragma unroll
            for (int r = 0; r < R_; ++r) {
                const int q = threadIdx.x + r * MGSP_NT;
                if (q < cnt) cp_async_el<sizeof(S)>(&vs[q], &vA[q], true);
            }
            cp_async_commit();
            if (two) {
#pragma unroll
                for (int r = 0; r < R_; ++r) {
                    const int q = threadIdx.x + r * MGSP_NT;
                    if (q < cnt) vrB[r] = vB[q];
                }
            }
            cp_async_wait_all();
            S dA = szero<S>(), dB = szero<S>(), cc = szero<S>();
#pragma unroll
            for (int r = 0; r < R_; ++r) {
                const int q = threadIdx.x + r * MGSP_NT;
                if (q < cnt) {
                    const S x = ws[q], va = vs[q];
                    dA = dot_acc(dA, va, x);                         // <v_i, w>
                    if (two) {
                        dB = dot_acc(dB, vrB[r], x);                 // <v_{i+1}, w>
                        cc = dot_acc(cc, vrB[r], va);                // <v_{i+1}, v_i>
                    }
                }
            }
            // next pair (or the next system's w and first pair) towards L2
            // while this phase's reduction and grid barrier run
            if (i + 2 <= a.k) {
                l2_prefetch_slice(vA + 2 * (size_t)a.n, cnt);
                if (i + 3 <= a.k) l2_prefetch_slice(vA + 3 * (size_t)a.n, cnt);
            } else if (b + 1 < a.B) {
                l2_prefetch_slice(a.w + (b + 1) * a.ldw + j0, cnt);
                l2_prefetch_slice(a.V + (b + 1) * a.ldv + j0, cnt);
                if (a.k >= 1) l2_prefetch_slice(a.V + (b + 1) * a.ldv + j0 + a.n, cnt);
            }
            double v[MGSP_NV];
            if constexpr (CPLX) {
                v[0] = dA.x; v[1] = dA.y; v[2] = dB.x; v[3] = dB.y; v[4] = cc.x; v[5] = cc.y;
            } else {
                v[0] = dA; v[1] = 0.0; v[2] = dB; v[3] = 0.0; v[4] = cc; v[5] = 0.0;
            }
            reduce_all(v);
            if constexpr (CPLX) {
                hA = make_double2(v[0], v[1]);
                hB = sub(make_double2(v[2], v[3]), mul(hA, make_double2(v[4], v[5])));
            } else {
                hA = v[0];
                hB = v[2] - hA * v[4];
            }
            prevB = two;
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                a.H[(size_t)i * a.B + b] = hA;
                if (two) a.H[(size_t)(i + 1) * a.B + b] = hB;
            }
        }
        // last projections, ||w||^2, w back to global
        double nn = 0.0;
#pragma unroll
        for (int r = 0; r < R_; ++r) {
            const int q = threadIdx.x + r * MGSP_NT;
            if (q < cnt) {
                S x = sub_mul(ws[q], hA, vs[q]);
                if (prevB) x = sub_mul(x, hB, vrB[r]);
                nn = sqacc(nn, x);
                w[q] = x;
            }
        }
        double v[MGSP_NV] = {nn, 0.0, 0.0, 0.0, 0.0, 0.0};
        reduce_all(v);
        if (blockIdx.x == 0 && threadIdx.x == 0) a.wnorm2[b] = v[0];
    }
}

// Arnoldi step tail (fgmres.py:79-80,106-107) for the systems of one MGS
// group: hk1 = sqrt(||w||^2); v_{k+1} = w / hk1 (computed for every system:
// the host's later decision to stop -- convergence, happy breakdown, the
// restart length -- simply ignores it, as the reference never reads it);
// and the packed Hessenberg column (h_0k .. h_kk, hk1) per system for one
// device->host copy.  One CTA row per system, grid-stride over n.
template <typename S>
__global__ void __launch_bounds__(MGS_NT) arnoldi_tail_kernel(const S* w, long long ldw, S* vnext,
                                                              long long ldv, const S* H, int k,
                                                              const double* n2, S* hcol, int n) {
    const int b = blockIdx.y;
    const double hk1 = sqrt(n2[b]);
    const S* wb = w + b * ldw;
    S* vb = vnext + b * ldv;
    for (int j = blockIdx.x * MGS_NT + threadIdx.x; j < n; j += gridDim.x * MGS_NT) {
        if constexpr (sizeof(S) == 16) vb[j] = make_double2(wb[j].x / hk1, wb[j].y / hk1);
        else vb[j] = wb[j] / hk1;
    }
    if (blockIdx.x == 0) {
        const int nb = gridDim.y;
        for (int i = threadIdx.x; i <= k + 1; i += MGS_NT) {
            S v;
            if (i <= k) v = H[(size_t)i * nb + b];
            else if constexpr (sizeof(S) == 16) v = make_double2(hk1, 0.0);
            else v = hk1;
            hcol[(size_t)b * (k + 2) + i] = v;
        }
    }
}

// u += Z[:, :k] y (fgmres.py:119): u[i] += sum_j Z[j][i] y[j], j ascending,
// the products unfused like numpy's complex arithmetic.
template <typename S>
__global__ void __launch_bounds__(MGS_NT) krylov_update_kernel(S* u, const S* Z, long long ldz,
                                                               const S* y, int k, int n) {
    __shared__ S ys[64];
    for (int j = threadIdx.x; j < k && j < 64; j += MGS_NT) ys[j] = y[j];
    __syncthreads();
    for (int i = blockIdx.x * MGS_NT + threadIdx.x; i < n; i += gridDim.x * MGS_NT) {
        S acc = szero<S>();
        for (int j = 0; j < k; ++j) acc = add(acc, mul(Z[(size_t)j * ldz + i], j < 64 ? ys[j] : y[j]));
        u[i] = add(u[i], acc);
    }
}

}  // namespace rg

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
constexpr int MGSP_NT = 512;

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
    double* part;                  // [gridDim][3]
    GridBar bar;
    int n, k, B, slice;
};

constexpr int MGSP_R = 16;          // slice elements per thread (slice <= MGSP_NT * MGSP_R)

template <typename S>
__global__ void __launch_bounds__(MGSP_NT, 1) mgs_persist_kernel(MgsPArgs<S> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S* ws = reinterpret_cast<S*>(smem_raw);           // [slice] this CTA's w
    S* vs = ws + a.slice;                              // [slice] this CTA's current v_i
    __shared__ double red[MGSP_NT / 32];
    __shared__ double tot[3];
    const int j0 = blockIdx.x * a.slice;
    const int cnt = max(0, min(a.n, j0 + a.slice) - j0);
    unsigned int phase = 0;
    if (threadIdx.x == 0) phase = *a.bar.gen;          // barrier phases continue from here
    int par = 0;                                       // partial-sum buffer parity
    for (int b = 0; b < a.B; ++b) {
        S* w = a.w + b * a.ldw + j0;
        const S* Vb = a.V + b * a.ldv + j0;
        S h = szero<S>();
        for (int i = 0; i <= a.k + 1; ++i) {
            const bool last = i == a.k + 1;
            const S* vn = last ? nullptr : Vb + (size_t)i * a.n;
            // all of this thread's global loads first (one latency per pass)
            S vr[MGSP_R], wr[MGSP_R];
#pragma unroll
            for (int r = 0; r < MGSP_R; ++r) {
                const int q = threadIdx.x + r * MGSP_NT;
                if (q < cnt) {
                    if (!last) vr[r] = vn[q];
                    if (i == 0) wr[r] = w[q];
                }
            }
            S dot = szero<S>();
            double nn = 0.0;
#pragma unroll
            for (int r = 0; r < MGSP_R; ++r) {
                const int q = threadIdx.x + r * MGSP_NT;
                if (q < cnt) {
                    S x = (i == 0) ? wr[r] : ws[q];
                    if (i > 0) x = sub(x, mul(h, vs[q]));      // w -= h_{i-1} v_{i-1}
                    ws[q] = x;
                    if (!last) {
                        vs[q] = vr[r];
                        dot = acc_add(dot, conj_mul(vr[r], x));  // <v_i, w>
                    } else {
                        nn = sqacc(nn, x);
                        w[q] = x;                                // w back to global
                    }
                }
            }
            double re, im = 0.0;
            if constexpr (sizeof(S) == 16) { re = dot.x; im = dot.y; } else { re = dot; }
            const double r0 = block_sum<MGSP_NT>(re, red);
            const double r1 = block_sum<MGSP_NT>(im, red);
            const double r2 = block_sum<MGSP_NT>(nn, red);
            double* part = a.part + (size_t)par * 3 * gridDim.x;
            if (threadIdx.x == 0) {
                double* p = part + (size_t)blockIdx.x * 3;
                p[0] = r0; p[1] = r1; p[2] = r2;
            }
            grid_barrier(a.bar, phase);
            // every CTA sums the partials in the same order; the other parity
            // buffer is written next, so no second barrier is needed
            double s0 = 0.0, s1 = 0.0, s2 = 0.0;
            for (int c = threadIdx.x; c < (int)gridDim.x; c += MGSP_NT) {
                s0 += __ldcg(&part[c * 3]); s1 += __ldcg(&part[c * 3 + 1]);
                s2 += __ldcg(&part[c * 3 + 2]);
            }
            s0 = block_sum<MGSP_NT>(s0, red);
            s1 = block_sum<MGSP_NT>(s1, red);
            s2 = block_sum<MGSP_NT>(s2, red);
            if (threadIdx.x == 0) { tot[0] = s0; tot[1] = s1; tot[2] = s2; }
            __syncthreads();
            if (!last) {
                if constexpr (sizeof(S) == 16) h = make_double2(tot[0], tot[1]);
                else h = tot[0];
                if (blockIdx.x == 0 && threadIdx.x == 0) a.H[(size_t)i * a.B + b] = h;
            } else if (blockIdx.x == 0 && threadIdx.x == 0) {
                a.wnorm2[b] = tot[2];
            }
            par ^= 1;
        }
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

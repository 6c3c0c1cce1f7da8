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
};

template <typename S>
__global__ void __launch_bounds__(MGS_NT) mgs_kernel(MgsArgs<S> a) {
    __shared__ double red[MGS_NT / 32];
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

}  // namespace rg

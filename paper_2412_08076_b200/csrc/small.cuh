// small.cuh — the whole solve_stationary (richardson.py:77-141) in ONE launch
// for grids that fit in shared memory (cfg1: 63^2).
//
// One CTA (1024 threads) per system keeps u (and the NAG look-ahead y) in a
// zero-bordered (s+2)^2 shared-memory field and f, r, v of its own points in
// registers, and iterates until convergence, divergence or max_outer without
// returning to the host: per inner step one pointwise update, one stencil
// pass, one deterministic block reduction of ||r||^2 and the decision of
// reduce.cuh:finalize taken by thread 0.  The launch-per-step overhead of the
// tiled kernels (~5 us x 2 launches per sweep at 63^2) disappears.
// Arithmetic is the reference's (no FMA): iterates are bitwise the oracle's.
#pragma once
#include "reduce.cuh"

namespace rg {

constexpr int SMALL_NT = 1024;
constexpr int SMALL_PPT = 4;                  // points per thread -> P <= 4096 (side <= 64)

template <typename S>
struct SmallArgs {
    const CT<S>* coef;   // [B][9]
    const CT<S>* scale;  // [B] Jacobi scale or null
    S* u;                // [B][P] initial guess in, answer out
    const S* f;          // [B][P]
    const double* omega;
    const double* alpha;
    const double* atil;
    int side, P, m;
    int shared;          // one coefficient set for every system
    SolveCfg cfg;
    SysState* st;
    double* trace;
    int trace_stride;
};

// Sum over the CTA, returned to EVERY thread with identical bits: each warp
// reduces the 32 per-warp partials in the same fixed tree order, so all
// threads can take the convergence decision themselves (one barrier).
__device__ inline double small_sum_all(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = red[lane];                       // 32 warps
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    return __shfl_sync(0xffffffffu, t, 0);
}

template <typename S, int VAR, bool JAC>
__global__ void __launch_bounds__(SMALL_NT, 1) small_solve_kernel(SmallArgs<S> a) {
    typedef CT<S> C;
    constexpr bool NAG = VAR >= V_NAG;
    constexpr bool HASV = VAR != V_PLAIN;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[32];
    const int b = blockIdx.x;
    const int s = a.side, W = s + 2, P = a.P, m = a.m;
    C* U = reinterpret_cast<C*>(smem_raw);      // [(s+2)^2], zero border
    C* Y = U + W * W;                           // NAG look-ahead field
    const size_t base = (size_t)b * P;
    const int tid = threadIdx.x;

    C c[9];
#pragma unroll
    for (int d = 0; d < 9; ++d) c[d] = a.coef[(size_t)(a.shared ? 0 : b) * 9 + d];
    const C sc = JAC ? a.scale[b] : szero<C>();

    for (int q = tid; q < W * W * (NAG ? 2 : 1); q += SMALL_NT) U[q] = szero<C>();
    __syncthreads();
    C fr[SMALL_PPT], rr[SMALL_PPT], vr[SMALL_PPT];
    int pix[SMALL_PPT];
#pragma unroll
    for (int j = 0; j < SMALL_PPT; ++j) {
        const int p = tid + j * SMALL_NT;
        const int x = p / s, y = p - (p / s) * s;
        pix[j] = (x + 1) * W + (y + 1);
        fr[j] = p < P ? to_c(a.f[base + p]) : szero<C>();
        vr[j] = szero<C>();                                  // v = 0 at entry (:95)
        rr[j] = szero<C>();
        if (p < P) U[pix[j]] = to_c(a.u[base + p]);
    }
    __syncthreads();

    auto stencil = [&](const C* X, int q) {                  // CSR order, no FMA
        C t = mul(c[0], X[q - W - 1]);
        t = add(t, mul(c[1], X[q - W]));
        t = add(t, mul(c[2], X[q - W + 1]));
        t = add(t, mul(c[3], X[q - 1]));
        t = add(t, mul(c[4], X[q]));
        t = add(t, mul(c[5], X[q + 1]));
        t = add(t, mul(c[6], X[q + W - 1]));
        t = add(t, mul(c[7], X[q + W]));
        t = add(t, mul(c[8], X[q + W + 1]));
        return t;
    };
    // residual of U at the thread's points: keeps r (plain/mom reuse it), returns ||r||^2 part
    auto residual_u = [&]() {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < SMALL_PPT; ++j) {
            if (tid + j * SMALL_NT < P) {
                rr[j] = sub(fr[j], stencil(U, pix[j]));
                acc = sqacc(acc, rr[j]);
            }
        }
        return acc;
    };
    double* trace = a.trace + (size_t)b * a.trace_stride;
    const SolveCfg cf = a.cfg;

    // ||f|| and the initial residual (:96-110); every thread holds the same
    // decision state (identical reductions), thread 0 writes trace / state.
    int status = ST_ACTIVE, outer = 0, inner = 0;
    double fnorm, trace0, rel, bad_rel = 0.0;
    {
        double ff = 0.0;
#pragma unroll
        for (int j = 0; j < SMALL_PPT; ++j) ff = sqacc(ff, fr[j]);
        const double r2 = small_sum_all(residual_u(), red);
        __syncthreads();
        const double f2 = small_sum_all(ff, red);
        fnorm = sqrt(f2);
        if (fnorm == 0.0) {                                 // :97-100
            status = ST_CONVERGED; rel = 0.0; trace0 = 0.0;
        } else {
            rel = sqrt(r2) / fnorm;
            trace0 = rel;
            if (rel <= cf.tol) status = ST_CONVERGED;
            else if (cf.max_outer <= 0) status = ST_MAXED;
        }
        if (tid == 0) trace[0] = trace0;
    }
    const double div_thr = cf.div_factor * fmax(trace0, 1.0);
    int k = 0;
    while (status == ST_ACTIVE) {
        const int i = k % m;
        const double w = a.omega[b * m + i];
        const double al = HASV ? a.alpha[b * m + i] : 0.0;
        if (NAG) {
            const double at = a.atil[b * m + i];
#pragma unroll
            for (int j = 0; j < SMALL_PPT; ++j)
                if (tid + j * SMALL_NT < P) Y[pix[j]] = add(U[pix[j]], rmul(at, vr[j]));   // (:119)
            __syncthreads();
#pragma unroll
            for (int j = 0; j < SMALL_PPT; ++j)
                if (tid + j * SMALL_NT < P) rr[j] = sub(fr[j], stencil(Y, pix[j]));
        }
        // v = a v + w B^{-1} r ; u = u + v  (:120-121), own points only
#pragma unroll
        for (int j = 0; j < SMALL_PPT; ++j) {
            if (tid + j * SMALL_NT < P) {
                const C p = JAC ? mul(sc, rr[j]) : rr[j];
                C vn = (VAR == V_PLAIN) ? rmul(w, p) : add(rmul(al, vr[j]), rmul(w, p));
                U[pix[j]] = stored<S>(add(U[pix[j]], vn));
                vr[j] = stored<S>(vn);
            }
        }
        __syncthreads();
        ++k;
        const bool test = !NAG || cf.check_inner || (k % m) == 0;   // (:123)
        if (test) {
            const double r2 = small_sum_all(residual_u(), red);
            rel = sqrt(r2) / fnorm;
            inner = k;
            const bool boundary = (k % m) == 0;
            if (!isfinite(rel) || rel > div_thr) {                 // :126-129
                status = ST_DIVERGED; bad_rel = rel;
            } else {
                if (boundary) {                                    // :133-134
                    outer = k / m;
                    if (tid == 0) trace[outer] = rel;
                }
                if ((cf.check_inner || boundary) && rel <= cf.tol) {   // :130-136
                    status = ST_CONVERGED;
                    if (!boundary) { outer = k / m + 1; if (tid == 0) trace[outer] = rel; }
                } else if (boundary && outer >= cf.max_outer) {
                    status = ST_MAXED;
                }
            }
        }
    }
    if (tid == 0) {
        SysState& st = a.st[b];
        st.fnorm = fnorm; st.trace0 = trace0; st.rel = rel; st.bad_rel = bad_rel;
        st.status = status; st.outer = outer; st.inner = inner; st.ans_buf = 0;
        st.last_j = k;
    }
    if (status != ST_DIVERGED) {
#pragma unroll
        for (int j = 0; j < SMALL_PPT; ++j) {
            const int p = tid + j * SMALL_NT;
            if (p < P) a.u[base + p] = to_s<S>(U[pix[j]]);
        }
    }
}

template <typename S>
inline size_t small_smem_bytes(int side, int variant) {
    const size_t W = side + 2;
    return W * W * sizeof(CT<S>) * (variant >= V_NAG ? 2 : 1);
}

template <typename S>
cudaError_t launch_small(const SmallArgs<S>& a, int variant, bool jac, int B, cudaStream_t st) {
    const size_t smem = small_smem_bytes<S>(a.side, variant);
#define RG_SMALL(V, J)                                                                       \
    do {                                                                                    \
        auto k = small_solve_kernel<S, V, J>;                                               \
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             (int)smem);                                    \
        if (e != cudaSuccess) return e;                                                     \
        k<<<B, SMALL_NT, smem, st>>>(a);                                                    \
    } while (0)
    if (variant == V_PLAIN) { if (jac) RG_SMALL(V_PLAIN, true); else RG_SMALL(V_PLAIN, false); }
    else if (variant == V_MOM) { if (jac) RG_SMALL(V_MOM, true); else RG_SMALL(V_MOM, false); }
    else { if (jac) RG_SMALL(V_NAG, true); else RG_SMALL(V_NAG, false); }
#undef RG_SMALL
    return cudaGetLastError();
}

}  // namespace rg

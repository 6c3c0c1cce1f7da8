// dst.cuh — orthonormal 2D DST-I on the (M-1)^2 interior (transforms.py:24-35)
// and the fused FNS correction u += dst2(lam * dst2(f - A u)) (fns.py:43-44,80).
//
// One line of N = M-1 samples x_1..x_N (M a power of two) is transformed via
// its odd extension y of length 2M (y_j = x_j, y_{2M-j} = -x_j, y_0 = y_M = 0):
//   Y_k = -2i sum_j x_j sin(pi j k / M)   =>   DST_k = -Im(Y_k) / 2.
// The real length-2M FFT is computed as one complex length-M FFT of
// z_j = y_{2j} + i y_{2j+1} (Stockham radix-4, ping-pong in shared memory,
// natural order), followed by the even/odd split
//   Y_k = E_k + e^{-i pi k/M} O_k,  E_k = (Z_k + conj Z_{M-k})/2,
//                                   O_k = (Z_k - conj Z_{M-k})/(2i).
// Orthonormal scaling sqrt(2/M) per axis (scipy dstn type=1 norm="ortho").
// Twiddles come from a host-built table tw[k] = (cos(pi k/M), sin(pi k/M)).
//
// Row lines are contiguous; column lines are strided by N and are loaded
// LPC columns at a time so every row contributes one 32 B+ segment.
// Not bitwise equal to pocketfft: agreement is ~1e-15 relative (the FNS
// parity bar is 1e-12, SURVEY.md §8(d) cfg 4).
#pragma once
#include "common.cuh"

namespace rg {

constexpr int DST_NT = 256;

struct DstArgs {
    const double* in;    // [B][N][N]
    double* out;         // [B][N][N]
    const double2* tw;   // [M] (cos, sin)(pi k / M)
    const double* lam;   // [B][N][N] symbol (column pass with lam), or null
    int N, M, logM;
    int lpc;             // lines per CTA
    int mode;            // DST_PLAIN, DST_TWICE_LAM (cols: dst, *lam, dst), DST_ADD (out += dst)
    double scale;        // sqrt(2/M)
};
enum { DST_PLAIN = 0, DST_TWICE_LAM = 1, DST_ADD = 2 };

__device__ __forceinline__ double2 cmulf(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// exp(-i pi k / M) for 0 <= k < 2M from the table tw[k] = (cos, sin)(pi k / M), k < M
__device__ __forceinline__ double2 tw_fwd(const double2* tw, int M, int k) {
    const bool hi = k >= M;
    const double2 c = __ldg(&tw[hi ? k - M : k]);
    return hi ? make_double2(-c.x, c.y) : make_double2(c.x, -c.y);
}

// Complex forward FFT of length M (power of two) on nl lines stored back to
// back, Stockham auto-sort (natural order in and out): one radix-2 pass when
// log2(M) is odd, then radix-4 passes.  Pass with sub-transform length Ns:
// thread j reads the 4 values at stride M/4 (contiguous across lanes),
// twiddles them by exp(-2 pi i (j mod Ns) r / 4Ns), does the 4-point DFT and
// writes them at idx = (j / Ns) 4 Ns + (j mod Ns) + r Ns.  Ping-pongs between
// A and B; returns the buffer holding the result.
__device__ inline double2* fft_lines(double2* A, double2* B, int nl, int M, int logM,
                                     const double2* tw) {
    double2* in = A;
    double2* out = B;
    int Ns = 1;
    if (logM & 1) {
        const int h = M >> 1;
        for (int t = threadIdx.x; t < nl * h; t += blockDim.x) {
            const int line = t >> (logM - 1), j = t & (h - 1);
            const double2 a = in[line * M + j], b = in[line * M + j + h];
            out[line * M + 2 * j] = make_double2(a.x + b.x, a.y + b.y);
            out[line * M + 2 * j + 1] = make_double2(a.x - b.x, a.y - b.y);
        }
        __syncthreads();
        double2* tmp = in; in = out; out = tmp;
        Ns = 2;
    }
    const int q = M >> 2;
    for (; Ns < M; Ns <<= 2) {
        const int kstep = M / (2 * Ns);          // twiddle index step per (jm * r)
        for (int t = threadIdx.x; t < nl * q; t += blockDim.x) {
            const int line = t >> (logM - 2), j = t & (q - 1);
            const double2* x = in + line * M + j;
            double2 v0 = x[0], v1 = x[q], v2 = x[2 * q], v3 = x[3 * q];
            const int jm = j & (Ns - 1);
            if (jm) {
                v1 = cmulf(v1, tw_fwd(tw, M, jm * kstep));
                v2 = cmulf(v2, tw_fwd(tw, M, 2 * jm * kstep));
                v3 = cmulf(v3, tw_fwd(tw, M, 3 * jm * kstep));
            }
            const double2 a = make_double2(v0.x + v2.x, v0.y + v2.y);
            const double2 b = make_double2(v0.x - v2.x, v0.y - v2.y);
            const double2 c = make_double2(v1.x + v3.x, v1.y + v3.y);
            const double2 d = make_double2(v1.x - v3.x, v1.y - v3.y);
            double2* y = out + line * M + (j - jm) * 4 + jm;
            y[0] = make_double2(a.x + c.x, a.y + c.y);
            y[Ns] = make_double2(b.x + d.y, b.y - d.x);          // b - i d
            y[2 * Ns] = make_double2(a.x - c.x, a.y - c.y);
            y[3 * Ns] = make_double2(b.x - d.y, b.y + d.x);      // b + i d
        }
        __syncthreads();
        double2* tmp = in; in = out; out = tmp;
    }
    return in;
}

// Load nl lines (line l reads x(l, j) for j = 1..N via `get`) as packed
// z_j = y_2j + i y_2j+1 of the odd extension, natural order.  LINES_FAST:
// consecutive threads take consecutive lines (strided column lines ->
// coalesced row segments).
template <bool LINES_FAST, class Get>
__device__ inline void load_lines(double2* z, int nl, int M, Get get) {
    const int N = M - 1;
    const int logM = __ffs(M) - 1;
    for (int t = threadIdx.x; t < nl * M; t += blockDim.x) {
        const int l = LINES_FAST ? t % nl : t >> logM;
        const int j = LINES_FAST ? t / nl : t & (M - 1);
        double ye, yo;   // y_{2j}, y_{2j+1}
        const int e = 2 * j, o = 2 * j + 1;
        if (e < M) {
            ye = (e >= 1) ? get(l, e) : 0.0;
            yo = (o <= N) ? get(l, o) : 0.0;
        } else {
            const int me = 2 * M - e, mo = 2 * M - o;   // mirrored indices in [1, M]
            ye = (me <= N) ? -get(l, me) : 0.0;
            yo = (mo >= 1 && mo <= N) ? -get(l, mo) : 0.0;
        }
        z[l * M + j] = make_double2(ye, yo);
    }
    __syncthreads();
}

// DST_k (k = 1..N) of line l from its transformed z, unscaled.
__device__ inline double dst_coeff(const double2* z, int l, int M, int k, const double2* tw) {
    const double2 zk = z[l * M + k];
    const double2 zm = z[l * M + (M - k)];
    // E = (zk + conj zm)/2 ; O = (zk - conj zm)/(2i)
    const double ex_im = 0.5 * (zk.y - zm.y);
    const double dre = zk.x - zm.x, dim = zk.y + zm.y;     // zk - conj(zm)
    const double ore = 0.5 * dim, oim = -0.5 * dre;        // (dre + i dim)/(2i)
    const double2 w = tw[k];                               // e^{-i pi k/M} = (c, -s)
    const double im = ex_im + (w.x * oim - w.y * ore);     // Im(E + w O)
    return -0.5 * im;
}

// ---- register-resident "4-step" FFT for 32 <= M <= 1024 (M = 32 * R2) ----
// One warp per line.  Step 1: lane n1 holds x[n1 + 32 n2] (n2 < R2) and does
// an R2-point FFT in registers; twiddle by exp(-2 pi i n1 k2 / M); write to a
// padded transpose T[k2 * 33 + n1] (conflict-free).  Step 2: lane k2 (< R2)
// reads T[k2 * 33 + n1] (n1 < 32), does a 32-point FFT in registers and
// produces X[k2 + R2 k1].  Only __syncwarp inside a line; in-register
// twiddles exp(-i pi j / 16) come from constant memory (compile-time index).
__constant__ double2 c_tw32[16];   // (cos, sin)(pi j / 16), filled by rg_dst_create

template <int R>
__device__ __forceinline__ void fft_reg(double2 (&v)[R]) {
    constexpr int LOG = (R >= 32) ? 5 : (R >= 16) ? 4 : (R >= 8) ? 3 : (R >= 4) ? 2 : (R >= 2) ? 1 : 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {                 // compile-time bit reversal
        int j = 0;
#pragma unroll
        for (int b = 0; b < LOG; ++b) j |= ((i >> b) & 1) << (LOG - 1 - b);
        if (j > i) { const double2 t = v[i]; v[i] = v[j]; v[j] = t; }
    }
#pragma unroll
    for (int h = 1; h < R; h <<= 1) {
#pragma unroll
        for (int g = 0; g < R; g += 2 * h) {
#pragma unroll
            for (int j = 0; j < h; ++j) {
                const double2 a = v[g + j];
                double2 b = v[g + j + h];
                if (j != 0) {                     // exp(-i pi j / h) = c_tw32[j * 16 / h] conj
                    const double2 c = c_tw32[j * (16 / h)];
                    b = make_double2(fma(b.x, c.x, b.y * c.y), fma(b.y, c.x, -b.x * c.y));
                }
                v[g + j] = make_double2(a.x + b.x, a.y + b.y);
                v[g + j + h] = make_double2(a.x - b.x, a.y - b.y);
            }
        }
    }
}

// FFT of the line stored at zl (natural order, M = 32 * R2 entries, buffer of
// R2 * 33 entries); result back in zl, natural order.  Called by one warp.
template <int R2>
__device__ __forceinline__ void fft_line_warp(double2* zl, int M, const double2* tw) {
    const int lane = threadIdx.x & 31;
    double2 v[R2];
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) v[n2] = zl[lane + 32 * n2];
    fft_reg<R2>(v);
#pragma unroll
    for (int k2 = 1; k2 < R2; ++k2) {
        if (lane) v[k2] = cmulf(v[k2], tw_fwd(tw, M, 2 * lane * k2));   // exp(-2 pi i n1 k2 / M)
    }
    __syncwarp();
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2) zl[k2 * 33 + lane] = v[k2];
    __syncwarp();
    if (lane < R2) {
        double2 w[32];
#pragma unroll
        for (int n1 = 0; n1 < 32; ++n1) w[n1] = zl[lane * 33 + n1];
        fft_reg<32>(w);
        __syncwarp((R2 >= 32) ? 0xffffffffu : ((1u << R2) - 1u));   // all reads of T done
#pragma unroll
        for (int k1 = 0; k1 < 32; ++k1) zl[lane + R2 * k1] = w[k1];
    }
    __syncwarp();
}

constexpr int DST4_NW = 4;   // warps (= lines) per CTA

template <int AXIS, int R2>
__global__ void __launch_bounds__(DST4_NW * 32) dst4_lines_kernel(DstArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = a.N, M = a.M;
    constexpr int LB = R2 * 33;                     // complex entries per line buffer
    double2* z = reinterpret_cast<double2*>(smem_raw);
    double* stage = reinterpret_cast<double*>(z + DST4_NW * LB);   // [NW][N] (TWICE_LAM)
    const size_t NN = (size_t)N * N;
    const int b = blockIdx.y;
    const int l0 = blockIdx.x * DST4_NW;
    const int nl = min(DST4_NW, N - l0);
    const int wp = threadIdx.x >> 5;
    const double* in = a.in + b * NN;
    auto addr = [&](int l, int j) -> size_t {
        return AXIS == 0 ? (size_t)(l0 + l) * N + (j - 1) : (size_t)(j - 1) * N + (l0 + l);
    };
    // packed odd extension, line l at z + l * LB
    auto load = [&](auto get) {
        for (int t = threadIdx.x; t < nl * M; t += blockDim.x) {
            const int l = AXIS == 1 ? t % nl : t / M;
            const int j = AXIS == 1 ? t / nl : t - (t / M) * M;
            double ye, yo;
            const int e = 2 * j, o = 2 * j + 1;
            if (e < M) {
                ye = (e >= 1) ? get(l, e) : 0.0;
                yo = (o <= N) ? get(l, o) : 0.0;
            } else {
                const int me = 2 * M - e, mo = 2 * M - o;
                ye = (me <= N) ? -get(l, me) : 0.0;
                yo = (mo >= 1 && mo <= N) ? -get(l, mo) : 0.0;
            }
            z[l * LB + j] = make_double2(ye, yo);
        }
        __syncthreads();
        if (wp < nl) fft_line_warp<R2>(z + wp * LB, M, a.tw);
        __syncthreads();
    };
    auto coeff = [&](int l, int k) {                 // unscaled DST_k of line l
        const double2 zk = z[l * LB + k];
        const double2 zm = z[l * LB + (M - k)];
        const double ex_im = 0.5 * (zk.y - zm.y);
        const double dre = zk.x - zm.x, dim = zk.y + zm.y;
        const double ore = 0.5 * dim, oim = -0.5 * dre;
        const double2 w = __ldg(&a.tw[k]);
        return -0.5 * (ex_im + (w.x * oim - w.y * ore));
    };
    load([&](int l, int j) { return in[addr(l, j)]; });
    double* out = a.out + b * NN;
    if (a.mode == DST_TWICE_LAM) {
        const double* lam = a.lam + b * NN;
        for (int t = threadIdx.x; t < nl * N; t += blockDim.x) {
            const int l = AXIS == 1 ? t % nl : t / N;
            const int k = AXIS == 1 ? t / nl + 1 : t - (t / N) * N + 1;
            stage[l * N + (k - 1)] = a.scale * coeff(l, k) * lam[addr(l, k)];
        }
        __syncthreads();
        load([&](int l, int j) { return stage[l * N + (j - 1)]; });
    }
    for (int t = threadIdx.x; t < nl * N; t += blockDim.x) {
        const int l = AXIS == 1 ? t % nl : t / N;
        const int k = AXIS == 1 ? t / nl + 1 : t - (t / N) * N + 1;
        const double v = a.scale * coeff(l, k);
        const size_t q = addr(l, k);
        if (a.mode == DST_ADD) out[q] = out[q] + v;
        else out[q] = v;
    }
}

// Row (AXIS=0) or column (AXIS=1) pass over all B*N lines.
template <int AXIS>
__global__ void __launch_bounds__(DST_NT) dst_lines_kernel(DstArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = a.N, M = a.M;
    double2* zA = reinterpret_cast<double2*>(smem_raw);
    double2* zB = zA + a.lpc * M;
    const size_t NN = (size_t)N * N;
    const int b = blockIdx.y;                           // system
    const int l0 = blockIdx.x * a.lpc;                  // first line of this CTA
    const int nl = min(a.lpc, N - l0);
    const double* in = a.in + b * NN;
    auto addr = [&](int l, int j) -> size_t {           // element j (1-based) of line l0+l
        return AXIS == 0 ? (size_t)(l0 + l) * N + (j - 1) : (size_t)(j - 1) * N + (l0 + l);
    };
    load_lines<AXIS == 1>(zA, nl, M, [&](int l, int j) { return in[addr(l, j)]; });
    double2* z = fft_lines(zA, zB, nl, M, a.logM, a.tw);
    double* out = a.out + b * NN;
    if (a.mode == DST_TWICE_LAM) {
        const double* lam = a.lam + b * NN;
        double* stage = reinterpret_cast<double*>(z == zA ? zB : zA);   // the free buffer
        for (int t = threadIdx.x; t < nl * N; t += blockDim.x) {
            // column layout: consecutive threads walk lines first (coalesced segments)
            const int l = AXIS == 1 ? t % nl : t / N;
            const int k = AXIS == 1 ? t / nl + 1 : t - (t / N) * N + 1;
            stage[l * N + (k - 1)] = a.scale * dst_coeff(z, l, M, k, a.tw) * lam[addr(l, k)];
        }
        __syncthreads();
        double2* dst = z;                                   // reload into the FFT buffer
        load_lines<false>(dst, nl, M, [&](int l, int j) { return stage[l * N + (j - 1)]; });
        z = fft_lines(dst, dst == zA ? zB : zA, nl, M, a.logM, a.tw);
    }
    for (int t = threadIdx.x; t < nl * N; t += blockDim.x) {
        const int l = AXIS == 1 ? t % nl : t / N;
        const int k = AXIS == 1 ? t / nl + 1 : t - (t / N) * N + 1;
        const double v = a.scale * dst_coeff(z, l, M, k, a.tw);
        const size_t q = addr(l, k);
        if (a.mode == DST_ADD) out[q] = out[q] + v;      // u = u + correction (fns.py:80)
        else out[q] = v;
    }
}

}  // namespace rg

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

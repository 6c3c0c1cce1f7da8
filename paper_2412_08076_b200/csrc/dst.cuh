// dst.cuh — orthonormal 2D DST-I on the (M-1)^2 interior (transforms.py:24-35)
// and the fused FNS correction u += dst2(lam * dst2(f - A u)) (fns.py:43-44,80).
//
// One line of N = M-1 samples x_1..x_N (M a power of two) is transformed via
// its odd extension y of length 2M (y_j = x_j, y_{2M-j} = -x_j, y_0 = y_M = 0):
//   Y_k = -2i sum_j x_j sin(pi j k / M)   =>   DST_k = -Im(Y_k) / 2.
// The real length-2M FFT is computed as one complex length-M FFT of
// z_j = y_{2j} + i y_{2j+1} (radix-2, in place in shared memory, loaded in
// bit-reversed order), followed by the even/odd split
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

__device__ __forceinline__ double2 cmul_conj_tw(double2 b, double2 c) {
    // b * w with w = (c.x, -c.y) = exp(-i theta), c = (cos, sin)(theta)
    return make_double2(fma(b.x, c.x, b.y * c.y), fma(b.y, c.x, -b.x * c.y));
}

// One complex radix-2 DIT FFT of length M on z (bit-reversed input order),
// executed cooperatively by the CTA on `nl` lines stored back to back.
// Stages are fused in pairs (radix-2^2): a thread loads the 4 elements
// {i, i+h, i+2h, i+3h}, applies the two butterfly stages (half sizes h and
// 2h) in registers and stores once -- half the shared-memory passes and
// barriers of plain radix-2.  An odd log2(M) leaves one radix-2 stage.
// Twiddle of stage half-size h at offset j: exp(-i pi j / h) = tw[j * M / h].
__device__ inline void fft_lines(double2* z, int nl, int M, int logM, const double2* tw) {
    int s = 1;
    if (logM & 1) {                       // one radix-2 stage (h = 1, twiddle 1)
        const int nb = nl * (M >> 1);
        for (int t = threadIdx.x; t < nb; t += blockDim.x) {
            const int i0 = 2 * t;         // lines are contiguous, M even
            const double2 a = z[i0], b = z[i0 + 1];
            z[i0] = make_double2(a.x + b.x, a.y + b.y);
            z[i0 + 1] = make_double2(a.x - b.x, a.y - b.y);
        }
        __syncthreads();
        s = 2;
    }
    for (; s < logM; s += 2) {
        const int h = 1 << (s - 1);       // first stage half-size; second is 2h
        const int nq = nl * (M >> 2);     // 4-element groups over all lines
        for (int t = threadIdx.x; t < nq; t += blockDim.x) {
            const int line = t / (M >> 2);
            const int g = t - line * (M >> 2);
            const int blk = g / h, j = g - blk * h;
            const int i0 = line * M + blk * 4 * h + j;
            double2 x0 = z[i0], x1 = z[i0 + h], x2 = z[i0 + 2 * h], x3 = z[i0 + 3 * h];
            // stage s: pairs (x0,x1), (x2,x3) with exp(-i pi j / h)
            const double2 w1 = __ldg(&tw[j * (M / h)]);
            double2 p = cmul_conj_tw(x1, w1);
            double2 q = cmul_conj_tw(x3, w1);
            double2 a0 = make_double2(x0.x + p.x, x0.y + p.y), a1 = make_double2(x0.x - p.x, x0.y - p.y);
            double2 a2 = make_double2(x2.x + q.x, x2.y + q.y), a3 = make_double2(x2.x - q.x, x2.y - q.y);
            // stage s+1: pairs (a0,a2) with exp(-i pi j / 2h), (a1,a3) with exp(-i pi (j+h) / 2h)
            const double2 w2 = __ldg(&tw[j * (M / (2 * h))]);
            const double2 w3 = __ldg(&tw[(j + h) * (M / (2 * h))]);
            p = cmul_conj_tw(a2, w2);
            q = cmul_conj_tw(a3, w3);
            z[i0] = make_double2(a0.x + p.x, a0.y + p.y);
            z[i0 + 2 * h] = make_double2(a0.x - p.x, a0.y - p.y);
            z[i0 + h] = make_double2(a1.x + q.x, a1.y + q.y);
            z[i0 + 3 * h] = make_double2(a1.x - q.x, a1.y - q.y);
        }
        __syncthreads();
    }
}

// Load nl lines (line l reads x(l, j) for j = 1..N via `get`) as packed z in
// bit-reversed order.  LINES_FAST: consecutive threads take consecutive
// lines (strided column lines -> coalesced row segments).
template <bool LINES_FAST, class Get>
__device__ inline void load_lines(double2* z, int nl, int M, int logM, Get get) {
    const int N = M - 1;
    for (int t = threadIdx.x; t < nl * M; t += blockDim.x) {
        const int l = LINES_FAST ? t % nl : t / M;
        const int j = LINES_FAST ? t / nl : t - l * M;
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
        const int r = __brev(j) >> (32 - logM);
        z[l * M + r] = make_double2(ye, yo);
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
    double2* z = reinterpret_cast<double2*>(smem_raw);
    double* stage = reinterpret_cast<double*>(z + a.lpc * a.M);   // [lpc][N] (TWICE_LAM)
    const int N = a.N, M = a.M;
    const size_t NN = (size_t)N * N;
    const int b = blockIdx.y;                           // system
    const int l0 = blockIdx.x * a.lpc;                  // first line of this CTA
    const int nl = min(a.lpc, N - l0);
    const double* in = a.in + b * NN;
    auto addr = [&](int l, int j) -> size_t {           // element j (1-based) of line l0+l
        return AXIS == 0 ? (size_t)(l0 + l) * N + (j - 1) : (size_t)(j - 1) * N + (l0 + l);
    };
    load_lines<AXIS == 1>(z, nl, M, a.logM, [&](int l, int j) { return in[addr(l, j)]; });
    fft_lines(z, nl, M, a.logM, a.tw);
    double* out = a.out + b * NN;
    if (a.mode == DST_TWICE_LAM) {
        const double* lam = a.lam + b * NN;
        for (int t = threadIdx.x; t < nl * N; t += blockDim.x) {
            // column layout: consecutive threads walk lines first (coalesced segments)
            const int l = AXIS == 1 ? t % nl : t / N;
            const int k = AXIS == 1 ? t / nl + 1 : t - (t / N) * N + 1;
            stage[l * N + (k - 1)] = a.scale * dst_coeff(z, l, M, k, a.tw) * lam[addr(l, k)];
        }
        __syncthreads();
        load_lines<false>(z, nl, M, a.logM, [&](int l, int j) { return stage[l * N + (j - 1)]; });
        fft_lines(z, nl, M, a.logM, a.tw);
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

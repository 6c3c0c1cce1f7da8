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

// One complex radix-2 DIT FFT of length M on z (bit-reversed input order),
// executed cooperatively by the CTA on `nl` lines stored back to back.
__device__ inline void fft_lines(double2* z, int nl, int M, int logM, const double2* tw) {
    const int nb = nl * (M >> 1);   // butterflies per pass over all lines
    for (int s = 1; s <= logM; ++s) {
        const int half = 1 << (s - 1);
        const int tstride = M >> s;     // twiddle index step: e^{-2 pi i j / 2half} = tw[j * M/half / 2 * 2]
        for (int t = threadIdx.x; t < nb; t += blockDim.x) {
            const int line = t / (M >> 1);
            const int bt = t - line * (M >> 1);
            const int grp = bt >> (s - 1);
            const int j = bt & (half - 1);
            const int i0 = line * M + grp * 2 * half + j;
            const int i1 = i0 + half;
            // w = exp(-2 pi i j / (2 half)) = exp(-i pi (j * M / half) / M)
            const double2 c = tw[j * tstride * 2];
            const double2 a = z[i0], bq = z[i1];
            // bq * w, w = (c.x, -c.y)
            const double2 p = make_double2(fma(bq.x, c.x, bq.y * c.y), fma(bq.y, c.x, -bq.x * c.y));
            z[i0] = make_double2(a.x + p.x, a.y + p.y);
            z[i1] = make_double2(a.x - p.x, a.y - p.y);
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

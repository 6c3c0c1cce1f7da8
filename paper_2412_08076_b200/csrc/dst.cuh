// dst.cuh — orthonormal 2D DST-I on the (M-1)^2 interior (transforms.py:24-35)
// and the fused FNS correction u += dst2(lam * dst2(f - A u)) (fns.py:43-44,80).
//
// One line of N = M-1 samples x_1..x_N (M a power of two) is transformed via
// its odd extension y of length 2M (y_j = x_j, y_{2M-j} = -x_j, y_0 = y_M = 0):
//   Y_k = -2i sum_j x_j sin(pi j k / M)   =>   DST_k = -Im(Y_k) / 2.
// The real length-2M FFT is computed as one complex length-M FFT of
// z_j = y_{2j} + i y_{2j+1}, followed by the even/odd split
//   Y_k = E_k + e^{-i pi k/M} O_k,  E_k = (Z_k + conj Z_{M-k})/2,
//                                   O_k = (Z_k - conj Z_{M-k})/(2i).
// The complex FFT is an in-place Stockham FFT in shared memory: every
// thread holds 16 values in registers, radix-16 passes (then one radix-2/4/8
// pass), one load / sync / store per pass; line buffers are XOR-swizzled and
// padded so every pass and both line orientations are bank-conflict free.
// Orthonormal scaling sqrt(2/M) per axis (scipy dstn type=1 norm="ortho").
// Twiddles come from a host-built table tw[k] = (cos(pi k/M), sin(pi k/M)),
// copied to shared memory for M <= DST_SMEM_TW_MAX.
//
// Row lines are contiguous; column lines are strided by N and are loaded
// LPC columns at a time so every row contributes one 32 B+ segment.
// Not bitwise equal to pocketfft: agreement is ~1e-15 relative (the FNS
// parity bar is 1e-12, SURVEY.md §8(d) cfg 4).  Sizes with M not a power of
// two take the dense sine-matrix path at the end of this file.
#pragma once
#include "common.cuh"

namespace rg {

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
    const double2 c = tw[hi ? k - M : k];   // shared or global table (generic load)
    return hi ? make_double2(-c.x, c.y) : make_double2(c.x, -c.y);
}

// ---- in-register DFTs (forward, W_R = exp(-2 pi i / R), natural order) ----
__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 c_mi(double2 a) { return make_double2(a.y, -a.x); }   // -i a

__device__ __forceinline__ void dft2(double2* v) {
    const double2 a = v[0], b = v[1];
    v[0] = c_add(a, b);
    v[1] = c_sub(a, b);
}
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
    const double2 a = c_add(x0, x2), b = c_sub(x0, x2);
    const double2 c = c_add(x1, x3), d = c_mi(c_sub(x1, x3));   // -i (x1 - x3)
    x0 = c_add(a, c);
    x1 = c_add(b, d);
    x2 = c_sub(a, c);
    x3 = c_sub(b, d);
}
__device__ __forceinline__ void dft4(double2* v) { dft4(v[0], v[1], v[2], v[3]); }
// The radix-8/16 kernels below work in place and leave X[k] in a permuted
// register slot, dft_slot<R>(k), so no register copies are needed.
// 8 = 2 x 4 (n = 4 n1 + n2, k = k1 + 2 k2): DFT2 over n1 in slots (n2, 4+n2),
// twiddle W8^{n2 k1}, DFT4 over n2 in slots (4 k1 + n2): X[k1 + 2 k2] in slot 4 k1 + k2.
__device__ __forceinline__ void dft8(double2* v) {
    constexpr double h = 0.70710678118654752440;   // sqrt(2)/2
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
        const double2 a = v[n2], b = v[4 + n2];
        v[n2] = c_add(a, b);          // k1 = 0
        v[4 + n2] = c_sub(a, b);      // k1 = 1
    }
    v[5] = make_double2(h * (v[5].x + v[5].y), h * (v[5].y - v[5].x));    // W8^1
    v[6] = c_mi(v[6]);                                                      // W8^2
    v[7] = make_double2(h * (v[7].y - v[7].x), -h * (v[7].x + v[7].y));   // W8^3
    dft4(v[0], v[1], v[2], v[3]);
    dft4(v[4], v[5], v[6], v[7]);
}
// 16 = 4 x 4 (n = 4 n1 + n2, k = k1 + 4 k2): DFT4 over n1 in slots
// (n2, 4+n2, 8+n2, 12+n2) leaves a[n2][k1] in slot 4 k1 + n2; twiddle
// W16^{n2 k1}; DFT4 over n2 in slots 4 k1 + (0..3): X[k1 + 4 k2] in slot 4 k1 + k2.
__device__ __forceinline__ void dft16(double2* v) {
    constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;   // cos, sin(pi/8)
    constexpr double h = 0.70710678118654752440;
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
    // W16^m = cos(pi m/8) - i sin(pi m/8), m = n2 k1
    auto rot = [](double2 x, double c, double s) {      // x * (c - i s)
        return make_double2(x.x * c + x.y * s, x.y * c - x.x * s);
    };
    v[4 * 1 + 1] = rot(v[4 * 1 + 1], c1, s1);   // k1=1 n2=1, m=1
    v[4 * 1 + 2] = rot(v[4 * 1 + 2], h, h);     // m=2
    v[4 * 1 + 3] = rot(v[4 * 1 + 3], s1, c1);   // m=3
    v[4 * 2 + 1] = rot(v[4 * 2 + 1], h, h);     // m=2
    v[4 * 2 + 2] = c_mi(v[4 * 2 + 2]);          // m=4
    v[4 * 2 + 3] = rot(v[4 * 2 + 3], -h, h);    // m=6
    v[4 * 3 + 1] = rot(v[4 * 3 + 1], s1, c1);   // m=3
    v[4 * 3 + 2] = rot(v[4 * 3 + 2], -h, h);    // m=6
    v[4 * 3 + 3] = rot(v[4 * 3 + 3], -c1, -s1); // m=9
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
}
template <int R> __device__ __forceinline__ void dftR(double2* v);
template <> __device__ __forceinline__ void dftR<2>(double2* v) { dft2(v); }
template <> __device__ __forceinline__ void dftR<4>(double2* v) { dft4(v); }
template <> __device__ __forceinline__ void dftR<8>(double2* v) { dft8(v); }
template <> __device__ __forceinline__ void dftR<16>(double2* v) { dft16(v); }
// register slot holding X[k] after dftR<R>
template <int R> __host__ __device__ constexpr int dft_slot(int k) {
    return R == 16 ? 4 * (k & 3) + (k >> 2) : (R == 8 ? 4 * (k & 1) + (k >> 1) : k);
}

// Shared-memory swizzle of complex element i of a line: XOR of bits 0-2 with
// bits 4-6 makes the first radix-16 pass's stride-16 stores (and every
// unit-stride access) bank-conflict free; it permutes within aligned blocks
// of 8, so swz(i) < M for every i < M (M a multiple of 8, or swz(i) = i).
__device__ __forceinline__ int swz(int i) { return i ^ ((i >> 4) & 7); }
// Line l of the buffer starts at l * (M + 2): the pad of two complex values
// keeps accesses that walk lines fastest (column passes) conflict-free too.
__host__ __device__ __forceinline__ int dst_ls(int M) { return M + 2; }
__device__ __forceinline__ int zi(int l, int i, int M) { return l * dst_ls(M) + swz(i); }

// Values per thread of the in-place FFT: 16 (M >= 16), else M.
__host__ __device__ inline int dst_vpt(int M) { return M >= 16 ? 16 : M; }

// One radix-R Stockham pass (sub-transform length Ns), IN PLACE: every
// thread loads its 16 / R butterflies' inputs into registers, the CTA
// synchronises, then every thread twiddles, transforms and stores.  Input
// j + r M/R, output (j - jm) R + jm + r Ns, jm = j mod Ns, twiddle
// exp(-2 pi i r jm / (R Ns)) = tw_fwd(k = 2 r jm M / (R Ns)).
template <int R, int VPT>
__device__ __forceinline__ void fft_pass(double2* x, int lo, int M, int Ns, int tl, int tpl, bool act,
                                         const double2* tw) {
    constexpr int BPT = VPT / R;
    double2 v[BPT][R];
    const int stride = M / R;
    if (act) {
#pragma unroll
        for (int q = 0; q < BPT; ++q) {
            const int j = tl + q * tpl;
#pragma unroll
            for (int r = 0; r < R; ++r) v[q][r] = x[lo + swz(j + r * stride)];
        }
    }
    __syncthreads();
    if (act) {
        const int kstep = 2 * M / (R * Ns);
#pragma unroll
        for (int q = 0; q < BPT; ++q) {
            const int j = tl + q * tpl;
            const int jm = j & (Ns - 1);
            if (jm) {
                // powers-of-two twiddles from the table, the rest as products
                // (<= 3 roundings; keeps ~4 twiddles live instead of R - 1)
                double2 w[R];
#pragma unroll
                for (int r = 1; r < R; r <<= 1) w[r] = tw_fwd(tw, M, r * jm * kstep);
#pragma unroll
                for (int r = 3; r < R; ++r)
                    if (r & (r - 1)) w[r] = cmulf(w[r & (r - 1)], w[r & -r]);
#pragma unroll
                for (int r = 1; r < R; ++r) v[q][r] = cmulf(v[q][r], w[r]);
            }
            dftR<R>(v[q]);
            const int y = (j - jm) * R + jm;
#pragma unroll
            for (int r = 0; r < R; ++r) x[lo + swz(y + r * Ns)] = v[q][dft_slot<R>(r)];
        }
    }
    __syncthreads();
}

// Complex forward FFT of length M (power of two) on nl lines stored back to
// back, in place, natural order in and out: radix-16 passes, then one
// radix-2/4/8 pass for the remaining factor.  The CTA has nl * M / VPT
// threads (VPT = dst_vpt(M)); all of them must call this.
// LOGM > 0: M = 2^LOGM known at compile time (passes unrolled, constant Ns).
template <int VPT, int LOGM>
__device__ inline void fft_lines_vpt(double2* z, int nl, int M, int logM, const double2* tw) {
    const int tpl = M / VPT;                  // threads per line
    const int line = threadIdx.x / tpl, tl = threadIdx.x - line * tpl;
    double2* x = z;
    const int lo = line * dst_ls(M);          // line offset (indices within a line: swz)
    const bool act = line < nl;
    int Ns = 1;
    if (VPT >= 16 && LOGM > 0) {
#pragma unroll
        for (int p = 0; p < (LOGM >> 2); ++p, Ns <<= 4) fft_pass<16, 16>(x, lo, M, Ns, tl, tpl, act, tw);
    } else if (VPT >= 16) {
#pragma unroll 1
        for (int p = 0; p < (logM >> 2); ++p, Ns <<= 4) fft_pass<16, 16>(x, lo, M, Ns, tl, tpl, act, tw);
    }
    switch (VPT >= 16 ? (logM & 3) : logM) {
        case 3: fft_pass<8, VPT < 8 ? 8 : VPT>(x, lo, M, Ns, tl, tpl, act, tw); break;
        case 2: fft_pass<4, VPT < 4 ? 4 : VPT>(x, lo, M, Ns, tl, tpl, act, tw); break;
        case 1: fft_pass<2, VPT < 2 ? 2 : VPT>(x, lo, M, Ns, tl, tpl, act, tw); break;
        default: break;
    }
}
template <int LOGM>
__device__ inline void fft_lines(double2* z, int nl, int M, int logM, const double2* tw) {
    switch (dst_vpt(M)) {
        case 16: fft_lines_vpt<16, LOGM>(z, nl, M, logM, tw); break;
        case 8: fft_lines_vpt<8, 0>(z, nl, M, logM, tw); break;
        default: fft_lines_vpt<4, 0>(z, nl, M, logM, tw); break;
    }
}

// Load nl lines (line l reads x(l, j) for j = 1..N via `get`) as packed
// z_j = y_2j + i y_2j+1 of the odd extension, natural order.  LINES_FAST:
// consecutive threads take consecutive lines (strided column lines ->
// coalesced row segments).  Every thread handles at most DST_VMAX entries
// (blockDim * DST_VMAX >= nl * M); all global loads are issued before the
// first shared-memory store, so their latencies overlap.
constexpr int DST_VMAX = 16;
template <bool LINES_FAST, class Get>
__device__ inline void load_lines(double2* z, int nl, int lpc, int M, int nt, Get get) {
    const int N = M - 1;
    const int logM = __ffs(M) - 1;
    const int llp = __ffs(lpc) - 1;   // lpc is a power of two: shifts, no divisions
    double2 y[DST_VMAX];
#pragma unroll
    for (int q = 0; q < DST_VMAX; ++q) {
        const int t = threadIdx.x + q * nt;
        y[q] = make_double2(0.0, 0.0);
        const int l = LINES_FAST ? t & (lpc - 1) : t >> logM;
        const int j = LINES_FAST ? t >> llp : t & (M - 1);
        if (l < nl && j < M) {
            const int e = 2 * j, o = 2 * j + 1;   // y_{2j}, y_{2j+1}
            if (e < M) {
                if (e >= 1) y[q].x = get(l, e);
                if (o <= N) y[q].y = get(l, o);
            } else {
                const int me = 2 * M - e, mo = 2 * M - o;   // mirrored indices in [1, M]
                if (me <= N) y[q].x = -get(l, me);
                if (mo >= 1 && mo <= N) y[q].y = -get(l, mo);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < DST_VMAX; ++q) {
        const int t = threadIdx.x + q * nt;
        const int l = LINES_FAST ? t & (lpc - 1) : t >> logM;
        const int j = LINES_FAST ? t >> llp : t & (M - 1);
        if (l < nl && j < M) {
            z[zi(l, j, M)] = y[q];
        }
    }
    __syncthreads();
}

// DST_k (k = 1..N) of line l from its transformed z, unscaled.
__device__ inline double dst_coeff(const double2* z, int l, int M, int k, const double2* tw) {
    const double2 zk = z[zi(l, k, M)];
    const double2 zm = z[zi(l, M - k, M)];
    // E = (zk + conj zm)/2 ; O = (zk - conj zm)/(2i)
    const double ex_im = 0.5 * (zk.y - zm.y);
    const double dre = zk.x - zm.x, dim = zk.y + zm.y;     // zk - conj(zm)
    const double ore = 0.5 * dim, oim = -0.5 * dre;        // (dre + i dim)/(2i)
    const double2 w = tw[k];                               // e^{-i pi k/M} = (c, -s)
    const double im = ex_im + (w.x * oim - w.y * ore);     // Im(E + w O)
    return -0.5 * im;
}

// Twiddle table in shared memory up to this M (16 B per entry).
constexpr int DST_SMEM_TW_MAX = 2048;

// Row (AXIS=0) or column (AXIS=1) pass over all B*N lines; lpc lines per
// CTA, lpc * M / dst_vpt(M) <= MAXNT threads, shared memory lpc * M complex
// values (+ the twiddle table for M <= DST_SMEM_TW_MAX); 128 registers per
// thread for the 16 in-flight complex values (2 CTAs/SM at MAXNT = 256).
// LOGM > 0: compile-time M = 2^LOGM and lpc = LPC (all index arithmetic
// folds to constants); LOGM = 0: runtime M, lpc.
template <int AXIS, int MAXNT, int LOGM, int LPC>
__global__ void __launch_bounds__(MAXNT, 512 / MAXNT) dst_lines_kernel(DstArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr bool CM = LOGM > 0;
    const int M = CM ? (1 << LOGM) : a.M;
    const int N = M - 1;
    const int lpc = CM ? LPC : a.lpc;                    // a power of two
    const int logM = CM ? LOGM : a.logM;
    const int llp = CM ? (LPC == 1 ? 0 : LPC == 2 ? 1 : LPC == 4 ? 2 : 3) : __ffs(lpc) - 1;
    const int nt = CM ? (LPC << LOGM) / 16 : (int)blockDim.x;
    double2* z = reinterpret_cast<double2*>(smem_raw);
    double2* tws = z + lpc * dst_ls(M);
    const bool tw_sm = CM || M <= DST_SMEM_TW_MAX;      // (CM sizes are <= DST_SMEM_TW_MAX)
    if (tw_sm)
        for (int k = threadIdx.x; k < M; k += nt) tws[k] = __ldg(&a.tw[k]);
    const double2* tw = tw_sm ? tws : a.tw;             // CM: statically shared memory
    double* lam_s = reinterpret_cast<double*>(tws + (tw_sm ? M : 0));   // [lpc][M + 8] (TWICE_LAM)
    const size_t NN = (size_t)N * N;
    const int b = blockIdx.y;                           // system
    const int l0 = blockIdx.x * lpc;                    // first line of this CTA
    const int nl = min(lpc, N - l0);
    const double* in = a.in + b * NN;
    auto addr = [&](int l, int j) -> size_t {           // element j (1-based) of line l0+l
        return AXIS == 0 ? (size_t)(l0 + l) * N + (j - 1) : (size_t)(j - 1) * N + (l0 + l);
    };
    // symbol-pass: stream this CTA's lam entries into shared memory during the
    // first transform (same thread -> entry mapping as their later use)
    if (a.mode == DST_TWICE_LAM) {
        const double* lam = a.lam + b * NN;
#pragma unroll
        for (int q = 0; q < DST_VMAX; ++q) {
            const int t = threadIdx.x + q * nt;
            const int l = AXIS == 1 ? t & (lpc - 1) : t >> logM;
            const int k = AXIS == 1 ? t >> llp : t & (M - 1);
            if (l < nl && k >= 1 && k < M) cp_async_el<8>(&lam_s[l * (M + 8) + k], lam + addr(l, k), true);
        }
        cp_async_commit();
    }
    load_lines<AXIS == 1>(z, nl, lpc, M, nt, [&](int l, int j) { return in[addr(l, j)]; });
    fft_lines<LOGM>(z, nl, M, logM, tw);
    double* out = a.out + b * NN;
    if (a.mode == DST_TWICE_LAM) {
        // coefficients * lam into registers, then (after every thread has read
        // z) scattered back into z as the next odd extension, second FFT
        constexpr int MAXC = DST_VMAX;    // >= lpc * M / blockDim = VPT
        double c[MAXC];
        cp_async_wait_all();                // own lam entries (read by the same thread)
#pragma unroll
        for (int q = 0; q < MAXC; ++q) {
            const int t = threadIdx.x + q * nt;
            c[q] = 0.0;
            // column layout: consecutive threads walk lines first (coalesced segments)
            const int l = AXIS == 1 ? t & (lpc - 1) : t >> logM;
            const int k = AXIS == 1 ? t >> llp : t & (M - 1);
            if (l < nl && k >= 1 && k < M) {
                c[q] = a.scale * dst_coeff(z, l, M, k, tw) * lam_s[l * (M + 8) + k];
            }
        }
        __syncthreads();
        double* zd = reinterpret_cast<double*>(z);      // (re, im) halves: y_{2j}, y_{2j+1}
#pragma unroll
        for (int q = 0; q < MAXC; ++q) {
            const int t = threadIdx.x + q * nt;
            const int l = AXIS == 1 ? t & (lpc - 1) : t >> logM;
            const int k = AXIS == 1 ? t >> llp : t & (M - 1);
            if (l < nl && k >= 1 && k < M) {
                // y_i lives in half (i & 1) of complex element l M + i / 2 (swizzled)
                zd[2 * zi(l, k >> 1, M) + (k & 1)] = c[q];                  // y_k = x_k
                zd[2 * zi(l, (2 * M - k) >> 1, M) + (k & 1)] = -c[q];      // y_{2M-k} = -x_k
            }
        }
        for (int l = threadIdx.x; l < nl; l += nt) {
            zd[2 * zi(l, 0, M)] = 0.0;                    // y_0
            zd[2 * zi(l, M >> 1, M)] = 0.0;               // y_M
        }
        __syncthreads();
        fft_lines<LOGM>(z, nl, M, logM, tw);
    }
    // output: DST_VMAX >= lpc * M / blockDim slots per thread (slot k = 0 idle); the
    // DST_ADD loads of u are issued together before the stores
    double v[DST_VMAX];
#pragma unroll
    for (int q = 0; q < DST_VMAX; ++q) {
        const int t = threadIdx.x + q * nt;
        v[q] = 0.0;
        const int l = AXIS == 1 ? t & (lpc - 1) : t >> logM;
        const int k = AXIS == 1 ? t >> llp : t & (M - 1);
        if (l < nl && k >= 1 && k < M) {
            v[q] = a.scale * dst_coeff(z, l, M, k, tw);
            if (a.mode == DST_ADD) v[q] = out[addr(l, k)] + v[q];   // u = u + correction (fns.py:80)
        }
    }
#pragma unroll
    for (int q = 0; q < DST_VMAX; ++q) {
        const int t = threadIdx.x + q * nt;
        const int l = AXIS == 1 ? t & (lpc - 1) : t >> logM;
        const int k = AXIS == 1 ? t >> llp : t & (M - 1);
        if (l < nl && k >= 1 && k < M) {
            out[addr(l, k)] = v[q];
        }
    }
}

// ---- dense path for any n (side + 1 not a power of two) -------------------
// The orthonormal DST-I matrix S[j][k] = sqrt(2/n) sin(pi (j+1)(k+1) / n) is
// symmetric and involutory, so dst2(X) = S X S on the N x N grid (row
// transform X S, column transform S X).  One tiled FP64 GEMM kernel, C = P Q
// per system (P or Q is the shared S: batch stride 0), with the FNS
// epilogues: store, store * lam, or accumulate into u.  2 N^3 flops per
// product: a fallback for sizes the FFT path does not take (e.g. N = 1000:
// ~0.15 ms per product per system), ~1e-15 relative like the FFT.
enum { GEMM_STORE = 0, GEMM_LAM = 1, GEMM_ADD = 2 };
constexpr int GM_T = 64, GM_K = 16, GM_NT = 256;   // 64 x 64 tile, 4 x 4 per thread

struct GemmArgs {
    const double* P; size_t sP;   // [B][N][N] or shared (sP = 0)
    const double* Q; size_t sQ;
    double* C; size_t sC;
    const double* lam;            // GEMM_LAM: [B][N][N]
    int N, mode;
};

static __global__ void __launch_bounds__(GM_NT) dst_gemm_kernel(const GemmArgs a) {
    __shared__ double Ps[GM_K][GM_T + 1];   // P tile, transposed (k, row)
    __shared__ double Qs[GM_K][GM_T + 1];   // Q tile (k, col)
    const int N = a.N, b = blockIdx.z;
    const double* P = a.P + b * a.sP;
    const double* Q = a.Q + b * a.sQ;
    const int r0 = blockIdx.y * GM_T, c0 = blockIdx.x * GM_T;
    const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;   // 16 x 16 threads, 4 x 4 outputs each
    double acc[4][4] = {};
    for (int k0 = 0; k0 < N; k0 += GM_K) {
        for (int e = threadIdx.x; e < GM_T * GM_K; e += GM_NT) {
            const int i = e / GM_K, k = e % GM_K;                 // P rows, coalesced along k
            const int gr = r0 + i, gk = k0 + k;
            Ps[k][i] = (gr < N && gk < N) ? P[(size_t)gr * N + gk] : 0.0;
            const int kk = e / GM_T, j = e % GM_T;                // Q rows, coalesced along cols
            const int gq = k0 + kk, gc = c0 + j;
            Qs[kk][j] = (gq < N && gc < N) ? Q[(size_t)gq * N + gc] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < GM_K; ++k) {
            double pr[4], qc[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) pr[i] = Ps[k][tr + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) qc[j] = Qs[k][tc + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(pr[i], qc[j], acc[i][j]);
        }
        __syncthreads();
    }
    double* C = a.C + b * a.sC;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gr = r0 + tr + 16 * i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gc = c0 + tc + 16 * j;
            if (gr < N && gc < N) {
                const size_t q = (size_t)gr * N + gc;
                if (a.mode == GEMM_LAM) C[q] = acc[i][j] * a.lam[b * a.sC + q];
                else if (a.mode == GEMM_ADD) C[q] = C[q] + acc[i][j];   // u = u + correction
                else C[q] = acc[i][j];
            }
        }
    }
}

}  // namespace rg

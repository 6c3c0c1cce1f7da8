// dstw.cu — lean DST-I line kernel for M = 256 * R3, R3 in {2, 4, 8}
// (sides 511, 1023, 2047; cfg4 is 1023), transforms.py:24-35 / fns.py:43-44.
//
// Same mathematics as dst.cuh (odd extension packed into one complex
// M-point FFT, even/odd split), organised so that a thread issues little
// besides FP64 and 128-bit shared-memory instructions:
//
//  * one line = M / 16 threads, 16 complex values per thread in registers;
//    the FFT is 16 x 16 x R3 (Stockham), two exchanges through a padded line
//    buffer (element i at i + i / 16: every offset of every pass is
//    thread-base + compile-time constant, all accesses bank-conflict free);
//  * the line is read from global memory straight into the first pass's
//    register layout (the mirrored half of the odd extension is the same
//    line read backwards) — no staging store, no zero-fill pass;
//  * in the last pass a thread takes the butterflies j and 256 - j together:
//    they hold Z_k and Z_{M-k} for the same k, so the even/odd split runs in
//    registers and yields DST_k and DST_{M-k} from one twiddle, and the
//    results go from registers to global memory (coalesced over k);
//  * ROW mapping: the M / 16 threads of a line are consecutive (contiguous
//    lines coalesce); the groups of a CTA only meet at named barriers of their
//    own, so their phases drift apart and overlap.  COL mapping: the 256 / (M / 16)
//    lines of a CTA are interleaved over the lanes, so each global access of a
//    warp covers whole 32-byte sectors of a row-major array read by columns;
//  * persistent CTAs (2 per SM) keep the twiddle table in shared memory.
//
// DSTW_TWICE_LAM (the symbol pass, fns.py:43-44 on the second axis) runs
// DST -> * lam -> DST on the lines without leaving the SM; DSTW_ADD is the
// fused u = u + correction (fns.py:80).
#include "dstw.cuh"
#include "dst.cuh"

namespace rg {

template <int LOGM> struct DW {
    static constexpr int M = 1 << LOGM;
    static constexpr int TPL = M / 16;       // threads per line
    static constexpr int R3 = M / 256;       // radix of the last pass
    static constexpr int NP = 8 / R3;        // (j, 256 - j) butterfly pairs per thread
    static constexpr int LSZ = M + M / 16;   // padded line (complex elements)
};

__device__ __forceinline__ int padi(int i) { return i + (i >> 4); }

// x * (c - i s)
__device__ __forceinline__ double2 rotf(double2 x, double c, double s) {
    return make_double2(fma(x.x, c, x.y * s), fma(x.y, c, -(x.x * s)));
}
// dft16 of dst.cuh with fused rotations (X[k1 + 4 k2] in slot 4 k1 + k2)
__device__ __forceinline__ void dft16f(double2* v) {
    constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
    constexpr double h = 0.70710678118654752440;
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
    v[5] = rotf(v[5], c1, s1);
    v[6] = make_double2(h * (v[6].x + v[6].y), h * (v[6].y - v[6].x));
    v[7] = rotf(v[7], s1, c1);
    v[9] = make_double2(h * (v[9].x + v[9].y), h * (v[9].y - v[9].x));
    v[10] = c_mi(v[10]);
    v[11] = make_double2(h * (v[11].y - v[11].x), -h * (v[11].x + v[11].y));
    v[13] = rotf(v[13], s1, c1);
    v[14] = make_double2(h * (v[14].y - v[14].x), -h * (v[14].x + v[14].y));
    v[15] = rotf(v[15], -c1, -s1);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
}

template <int LOGM, bool COL, int MODE>
__global__ void __launch_bounds__(256, 2) dstw_kernel(const DstwArgs a) {
    using W = DW<LOGM>;
    constexpr int M = W::M, TPL = W::TPL, R3 = W::R3, NP = W::NP;
    constexpr int G = 256 / TPL;                        // lines per CTA
    constexpr int LS = W::LSZ + (COL ? 8 / G : 0);      // COL: lines land on distinct banks
    constexpr int S2 = TPL + R3;                        // padded distance of TPL elements
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* tws = reinterpret_cast<double2*>(smem_raw);
    const int tid = threadIdx.x;
    for (int k = tid; k < M; k += 256) tws[k] = __ldg(&a.tw[k]);
    __syncthreads();
    const int g = COL ? tid % G : tid / TPL;            // line slot of this thread
    const int t = COL ? tid / G : tid % TPL;            // its index on the line
    double2* buf = tws + M + g * LS;
    double* bufd = reinterpret_cast<double*>(buf);
    auto gsync = [&]() {
        if (COL) __syncthreads();
        else if (TPL == 32) __syncwarp();
        else asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(TPL) : "memory");
    };
    auto twc = [&](int k) { const double2 c = tws[k]; return make_double2(c.x, -c.y); };   // exp(-i pi k / M)

    const int jm = t & 15;
    const int o1s = 17 * t;                 // pass 1 store: element 16 t + r
    const int o2l = t + (t >> 4);           // pass 2 / smem pass-1 load: element t + TPL r
    const int o2s = 272 * (t >> 4) + jm;    // pass 2 store: element 256 (t / 16) + jm + 16 r
    // pass 2 twiddles exp(-2 pi i r jm / 256), r = 1, 2, 4, 8 (the rest are products)
    double2 w2p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) w2p[i] = twc((jm << i) * (M / 128));

    // complex M-point FFT of the line held in v (pass-1 order); returns with
    // Z of the thread's last-pass butterflies in v: pair p, side s (0: j = jA,
    // 1: j = 256 - jA, or 128 for the thread with jA = 0), output r at
    // v[(2 p + s) R3 + dft_slot<R3>(r)] = Z_{j + 256 r}
    auto fft = [&](double2* v) {
        dft16f(v);
        gsync();                            // earlier readers of the line buffer are done
#pragma unroll
        for (int r = 0; r < 16; ++r) buf[o1s + r] = v[dft_slot<16>(r)];
        gsync();
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = buf[o2l + r * S2];
        gsync();
        {
            double2 w[16];
            w[1] = w2p[0]; w[2] = w2p[1]; w[4] = w2p[2]; w[8] = w2p[3];
#pragma unroll
            for (int r = 3; r < 16; ++r)
                if (r & (r - 1)) w[r] = cmulf(w[r & (r - 1)], w[r & -r]);
#pragma unroll
            for (int r = 1; r < 16; ++r) v[r] = cmulf(v[r], w[r]);
        }
        dft16f(v);
#pragma unroll
        for (int r = 0; r < 16; ++r) buf[o2s + 17 * r] = v[dft_slot<16>(r)];
        gsync();
#pragma unroll
        for (int p = 0; p < NP; ++p) {
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const int jA = t + TPL * p;
                const int j = s == 0 ? jA : (jA == 0 ? 128 : 256 - jA);
                double2* x = v + (2 * p + s) * R3;
                const int o3 = j + (j >> 4);
#pragma unroll
                for (int r = 0; r < R3; ++r) x[r] = buf[o3 + 272 * r];
                // twiddles exp(-2 pi i r j / M) = exp(-i pi (2 r j) / M)
                double2 w[R3];
#pragma unroll
                for (int r = 1; r < R3; r <<= 1) w[r] = twc(2 * r * j);
#pragma unroll
                for (int r = 3; r < R3; ++r)
                    if (r & (r - 1)) w[r] = cmulf(w[r & (r - 1)], w[r & -r]);
#pragma unroll
                for (int r = 1; r < R3; ++r) x[r] = cmulf(x[r], w[r]);
                dftR<R3>(x);
            }
        }
    };

    // DST_k and DST_{M-k} (both scaled) of pair q = p R3 + r; k returned
    auto split = [&](const double2* v, int p, int r, int& k, double& dk, double& dmk) {
        const int jA = t + TPL * p;
        const double2* A = v + (2 * p) * R3;
        const double2* Bz = v + (2 * p + 1) * R3;
        double2 zk, zm;
        zk = A[dft_slot<R3>(r)];
        zm = Bz[dft_slot<R3>(R3 - 1 - r)];
        k = jA + 256 * r;
        if (p == 0 && t == 0) {   // butterflies 0 and 128 pair with themselves
            if (r < R3 / 2) {
                zk = A[dft_slot<R3>(r + 1)];
                zm = A[dft_slot<R3>(R3 - 1 - r)];
                k = 256 * (r + 1);
            } else {
                zk = Bz[dft_slot<R3>(r - R3 / 2)];
                zm = Bz[dft_slot<R3>(R3 - 1 - (r - R3 / 2))];
                k = 128 + 256 * (r - R3 / 2);
            }
        }
        // Y_k = E + w O, E = (zk + conj zm) / 2, O = (zk - conj zm) / (2 i), w = exp(-i pi k / M):
        // Im Y_k = (a - g) / 2, Im Y_{M-k} = -(a + g) / 2 with a = Im zk - Im zm,
        // g = c (Re zk - Re zm) + s (Im zk + Im zm); DST = -Im Y / 2
        const double2 cs = tws[k];
        const double av = zk.y - zm.y;
        const double gv = fma(cs.x, zk.x - zm.x, cs.y * (zk.y + zm.y));
        dk = a.s4 * (av - gv);
        dmk = -a.s4 * (av + gv);
    };

    constexpr int NPAN = M / G;
    const long long total = COL ? (long long)a.B * NPAN : (long long)a.B * a.N;
    const long long step = COL ? (long long)gridDim.x : (long long)gridDim.x * G;
    for (long long L = COL ? (long long)blockIdx.x : (long long)blockIdx.x * G + g; L < total; L += step) {
        long long b;
        int line;
        bool valid = true;
        if (COL) {
            b = L / NPAN;
            line = (int)(L - b * NPAN) * G + g;
            valid = line >= 1 && line <= a.N;
        } else {
            b = L / a.N;
            line = (int)(L - b * a.N) + 1;
        }
        double2 v[16];
        if (valid) {
            const double* pin = a.in.base + (b * a.in.bs + a.in.off + line * a.in.ls);
            const long long es = a.in.es;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int k0 = 2 * (t + TPL * r);           // y_{2j}, y_{2j+1}, j = t + TPL r < M / 2
                v[r].x = (r > 0 || t > 0) ? pin[k0 * es] : 0.0;
                v[r].y = pin[(k0 + 1) * es];
            }
#pragma unroll
            for (int r = 8; r < 16; ++r) {
                const int jp = TPL * (16 - r) - t;          // j = M - jp: (-x_{2 jp}, -x_{2 jp - 1})
                v[r].x = (r > 8 || t > 0) ? -pin[2 * jp * es] : 0.0;
                v[r].y = -pin[(2 * jp - 1) * es];
            }
        } else {
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = make_double2(0.0, 0.0);
        }
        fft(v);
        double* pout = a.out.base + (b * a.out.bs + a.out.off + line * a.out.ls);
        const long long oes = a.out.es;
        if (MODE == DSTW_TWICE_LAM) {
            double lm[16];
            if (valid) {
                const double* pl = a.lam.base + (b * a.lam.bs + a.lam.off + line * a.lam.ls);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int p = q / R3, r = q % R3;
                    const int jA = t + TPL * p;
                    int k = jA + 256 * r;
                    if (p == 0 && t == 0) k = r < R3 / 2 ? 256 * (r + 1) : 128 + 256 * (r - R3 / 2);
                    lm[2 * q] = pl[k * a.lam.es];
                    lm[2 * q + 1] = pl[(M - k) * a.lam.es];
                }
            } else {
#pragma unroll
                for (int q = 0; q < 16; ++q) lm[q] = 0.0;
            }
            gsync();   // every thread has read its last-pass inputs
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                int k;
                double dk, dmk;
                split(v, q / R3, q % R3, k, dk, dmk);
                // x_k of the next transform at its place in the packed odd extension
                bufd[2 * padi(k >> 1) + (k & 1)] = dk * lm[2 * q];
                const int mk = M - k;
                bufd[2 * padi(mk >> 1) + (mk & 1)] = dmk * lm[2 * q + 1];
            }
            gsync();
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                v[r] = buf[o2l + r * S2];
                if (r == 0 && t == 0) v[r].x = 0.0;         // x_0
            }
#pragma unroll
            for (int r = 8; r < 16; ++r) {
                const int jp = TPL * (16 - r) - t;
                v[r].x = (r > 8 || t > 0) ? -bufd[2 * padi(jp)] : 0.0;      // x_M = 0
                v[r].y = -bufd[2 * padi(jp - 1) + 1];
            }
            fft(v);
        }
        double uo[16];
        if (MODE == DSTW_ADD && valid) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int p = q / R3, r = q % R3;
                const int jA = t + TPL * p;
                int k = jA + 256 * r;
                if (p == 0 && t == 0) k = r < R3 / 2 ? 256 * (r + 1) : 128 + 256 * (r - R3 / 2);
                uo[2 * q] = pout[k * oes];
                uo[2 * q + 1] = pout[(M - k) * oes];
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            int k;
            double dk, dmk;
            split(v, q / R3, q % R3, k, dk, dmk);
            if (MODE == DSTW_ADD) {   // u = u + correction (fns.py:80)
                dk = uo[2 * q] + dk;
                dmk = uo[2 * q + 1] + dmk;
            }
            if (valid) {
                pout[k * oes] = dk;
                pout[(M - k) * oes] = dmk;
            }
        }
    }
}

bool dstw_supported(int M) { return M == 512 || M == 1024 || M == 2048; }

template <int LOGM, bool COL, int MODE>
static cudaError_t launch_one(const DstwArgs& a, int num_sms, cudaStream_t st) {
    using W = DW<LOGM>;
    constexpr int G = 256 / W::TPL;
    constexpr int LS = W::LSZ + (COL ? 8 / G : 0);
    const size_t smem = ((size_t)W::M + (size_t)G * LS) * sizeof(double2);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(dstw_kernel<LOGM, COL, MODE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const long long units = COL ? (long long)a.B * (W::M / G) : ((long long)a.B * a.N + G - 1) / G;
    long long grid = 2LL * num_sms;
    if (grid > units) grid = units;
    dstw_kernel<LOGM, COL, MODE><<<(unsigned)grid, 256, smem, st>>>(a);
    return cudaGetLastError();
}

template <int LOGM>
static cudaError_t launch_logm(const DstwArgs& a, bool col, int mode, int num_sms, cudaStream_t st) {
    // the combinations the 2D transforms use: rows plain / add, columns plain / symbol
    if (col) {
        if (mode == DSTW_TWICE_LAM) return launch_one<LOGM, true, DSTW_TWICE_LAM>(a, num_sms, st);
        if (mode == DSTW_PLAIN) return launch_one<LOGM, true, DSTW_PLAIN>(a, num_sms, st);
        return cudaErrorInvalidValue;
    }
    if (mode == DSTW_ADD) return launch_one<LOGM, false, DSTW_ADD>(a, num_sms, st);
    if (mode == DSTW_PLAIN) return launch_one<LOGM, false, DSTW_PLAIN>(a, num_sms, st);
    return cudaErrorInvalidValue;
}

cudaError_t launch_dstw(const DstwArgs& a, int logM, bool col, int mode, int num_sms, cudaStream_t st) {
    switch (logM) {
        case 9: return launch_logm<9>(a, col, mode, num_sms, st);
        case 10: return launch_logm<10>(a, col, mode, num_sms, st);
        case 11: return launch_logm<11>(a, col, mode, num_sms, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace rg

// cblock.cuh — temporally blocked free-running sweeps for the complex
// 5-point damped-Helmholtz operator (DIAG5, complex128), the V-cycle fine
// level smoother of cfg5 (multigrid.py:126-138: plain/mom/nag, fresh v, no
// preconditioner).
//
// Same overlapped-tile scheme as block.cuh: one CTA owns an LR x LC window
// with a T-cell halo and runs T inner steps on chip.  The stencil input (u,
// or the look-ahead y = u + at v) is ping-ponged in shared memory as
// complex128, f of the window sits in shared memory, the per-node complex
// diagonal is read through L1 (it is shared by every right-hand side of the
// batch, so it stays L2/L1 resident), u and v of the thread's points live in
// registers.  Products are the unfused complex formula in CSR column order
// (-1,0),(0,-1),(0,0),(0,1),(1,0): bitwise equal to the CSR matvec.
#pragma once
#include "step.cuh"

namespace rg {

#ifndef CB_LR_ROWS   // window rows of the 5-point smoother (16 measured 724 vs 568 us at 1023^2)
#define CB_LR_ROWS 32
#endif
#ifndef CB_WARPS   // warps per CTA (16 with 1 CTA/SM measured 634 vs 565 us at 1023^2)
#define CB_WARPS 8
#endif
// 32-column windows, 3 CTAs/SM (4 points per thread, 80 registers): 538 us
// per 16-step call at 1023^2 against 564 us for 32 x 64 at 2 CTAs/SM
#ifndef CB_COLS
#define CB_COLS 32
#endif
constexpr int CB_LR = CB_LR_ROWS, CB_LC = CB_COLS, CB_NW = CB_WARPS;
#ifndef CB9_COLS
#define CB9_COLS 64   // Galerkin-level windows: 64 columns (16 x 32 at 3 CTAs/SM: 346 vs 303 us at 511^2)
#endif
constexpr int CB9_LC = CB9_COLS;
#ifndef CB_DIAG_REGS
#define CB_DIAG_REGS 1
#endif
#ifndef CB_MINB
#define CB_MINB 3
#endif

struct CBlockArgs {
    double2 off[4];        // off-diagonals in CSR order (-1,0),(0,-1),(0,1),(1,0)
    const double2* diag;   // [P] (shared operator) or [B][P]
    int diag_shared;
    int side, P;
    const double2* u_in;
    const double2* v_in;
    double2* u_out;
    double2* v_out;
    const double2* f;
    const double* omega;
    const double* alpha;
    const double* atil;
    int m;
    int k0;
    int nty;
    int zero_in;           // bit 0: v_in is all zero, bit 1: u_in is all zero (not read)
};

__host__ __device__ inline int cblock_ntiles(int side, int T, int* nty) {
    const int TX = CB_LR - 2 * T, TY = CB_LC - 2 * T;
    const int ny = (side + TY - 1) / TY;
    if (nty) *nty = ny;
    return ((side + TX - 1) / TX) * ny;
}

// REALOFF: the four off-diagonals have zero imaginary parts (the
// Helmholtz 5-point stencil: -1/h^2).  SciPy's unfused product of (a + 0i)
// with x is (a xr - 0 xi, a xi + 0 xr), which equals (a xr, a xi) except
// possibly for the sign of an exact zero (or a NaN where x is already
// infinite), so the kernel forms the 2-multiply product: values compare
// equal (==) to the reference's, with 16 of ~52 FP64 operations per
// complex point-step fewer.
template <int VAR, int T, bool REALOFF>
__global__ void __launch_bounds__(CB_NW * 32, CB_MINB) cblock_kernel(const __grid_constant__ CBlockArgs a) {
    typedef double2 C;
    constexpr int LR = CB_LR, LC = CB_LC;
    constexpr int RPW = LR / CB_NW, CPT = LC / 32;
    constexpr int TX = LR - 2 * T, TY = LC - 2 * T;
    constexpr bool NAG = VAR >= V_NAG;
    constexpr bool HASV = VAR != V_PLAIN;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    typedef C Row[LC];
    Row* buf0 = reinterpret_cast<Row*>(smem_raw);
    Row* buf1 = buf0 + LR;
    Row* sf = buf1 + LR;

    const int b = blockIdx.y;
    const int cta = blockIdx.x;
    const int tx = cta / a.nty, ty = cta - (cta / a.nty) * a.nty;
    const int gx0 = tx * TX - T, gy0 = ty * TY - T;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int side = a.side;
    const size_t base = (size_t)b * a.P;
    const double2* dg = a.diag + (a.diag_shared ? 0 : base);
    const int r0 = wp * RPW;
    const C c0 = a.off[0], c1 = a.off[1], c2 = a.off[2], c3 = a.off[3];

    C ur[RPW][CPT], vr[RPW][CPT];
#if CB_DIAG_REGS
    C dr[RPW][CPT];           // per-node diagonal, loaded once (constant over the T steps)
#endif
    int gidx[RPW][CPT];       // global index of the point, -1 outside the grid
    const double at0 = NAG ? a.atil[b * a.m + (a.k0 % a.m)] : 0.0;
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
        const int gx = gx0 + r0 + rr;
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
            const int col = lane + 32 * cc;
            const int gy = gy0 + col;
            const bool in = (gx >= 0) && (gx < side) && (gy >= 0) && (gy < side);
            const int g = in ? gx * side + gy : -1;
            gidx[rr][cc] = g;
            const C u = (in && !(a.zero_in & 2)) ? a.u_in[base + g] : szero<C>();
            const C v = (HASV && in && !(a.zero_in & 1)) ? a.v_in[base + g] : szero<C>();
            ur[rr][cc] = u;
            vr[rr][cc] = v;
            sf[r0 + rr][col] = in ? a.f[base + g] : szero<C>();
#if CB_DIAG_REGS
            dr[rr][cc] = in ? __ldg(&dg[g]) : szero<C>();
#endif
            buf0[r0 + rr][col] = (NAG && in) ? add(u, rmul(at0, v)) : u;   // (:119)
        }
    }
    // the T steps' weights, loaded once (see block.cuh)
    __shared__ double sw[3][8];
    if (threadIdx.x < T) {
        const int k = a.k0 + threadIdx.x;
        const int si = b * a.m + (k % a.m);
        sw[0][threadIdx.x] = a.omega[si];
        sw[1][threadIdx.x] = HASV ? a.alpha[si] : 0.0;
        sw[2][threadIdx.x] = NAG ? a.atil[b * a.m + ((k + 1) % a.m)] : 0.0;
    }
    __syncthreads();

#pragma unroll
    for (int t = 0; t < T; ++t) {
        const double w = sw[0][t];
        const double al = sw[1][t];
        const double atn = sw[2][t];
        Row* cur = (t & 1) ? buf1 : buf0;
        Row* nxt = (t & 1) ? buf0 : buf1;
        const bool last = (t == T - 1);
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
            const int col = lane + 32 * cc;
            const int cm = col > 0 ? col - 1 : 0;
            const int cp = col < LC - 1 ? col + 1 : LC - 1;
            const int rm = r0 > 0 ? r0 - 1 : 0;
            C up = cur[rm][col];
            C mid = cur[r0][col];
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr) {
                const int r = r0 + rr;
                const int rp = r + 1 < LR ? r + 1 : LR - 1;
                const C wv = cur[r][cm], ev = cur[r][cp], dn = cur[rp][col];
                const int g = gidx[rr][cc];
#if CB_DIAG_REGS
                const C d = dr[rr][cc];
#else
                const C d = g >= 0 ? __ldg(&dg[g]) : szero<C>();
#endif
                C s = REALOFF ? rmul(c0.x, up) : mul(c0, up);     // CSR order, unfused
                s = add(s, REALOFF ? rmul(c1.x, wv) : mul(c1, wv));
                s = add(s, mul(d, mid));
                s = add(s, REALOFF ? rmul(c2.x, ev) : mul(c2, ev));
                s = add(s, REALOFF ? rmul(c3.x, dn) : mul(c3, dn));
                const C rs = sub(sf[r][col], s);          // r = f - A x
                C vn;
                if (VAR == V_PLAIN) vn = rmul(w, rs);
                else vn = add(rmul(al, vr[rr][cc]), rmul(w, rs));   // v = a v + w r
                const C un = add(NAG ? ur[rr][cc] : mid, vn);      // u = u + v
                if (HASV) vr[rr][cc] = vn;
                ur[rr][cc] = un;
                if (!last) {
                    const C x = NAG ? add(un, rmul(atn, vn)) : un;
                    nxt[r][col] = g >= 0 ? x : szero<C>();
                }
                up = mid;
                mid = dn;
            }
        }
        if (!last) __syncthreads();
    }
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
        const int r = r0 + rr;
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
            const int col = lane + 32 * cc;
            const int g = gidx[rr][cc];
            if (g >= 0 && r >= T && r < LR - T && col >= T && col < LC - T) {
                a.u_out[base + g] = ur[rr][cc];
                if (HASV) a.v_out[base + g] = vr[rr][cc];
            }
        }
    }
}

template <int VAR, int T, bool REALOFF>
cudaError_t launch_cblock_r(const CBlockArgs& a0, int batch, cudaStream_t st) {
    auto kern = cblock_kernel<VAR, T, REALOFF>;
    const size_t smem = 3 * (size_t)CB_LR * CB_LC * sizeof(double2);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    CBlockArgs a = a0;
    const int nt = cblock_ntiles(a.side, T, &a.nty);
    kern<<<dim3(nt, batch), dim3(CB_NW * 32), smem, st>>>(a);
    return cudaGetLastError();
}

template <int VAR, int T>
cudaError_t launch_cblock_t(const CBlockArgs& a, int batch, cudaStream_t st) {
    const bool real_off = a.off[0].y == 0.0 && a.off[1].y == 0.0 && a.off[2].y == 0.0 &&
                          a.off[3].y == 0.0;
    return real_off ? launch_cblock_r<VAR, T, true>(a, batch, st)
                    : launch_cblock_r<VAR, T, false>(a, batch, st);
}

template <int VAR>
cudaError_t launch_cblock(const CBlockArgs& a, int T, int batch, cudaStream_t st) {
    switch (T) {
        case 1: return launch_cblock_t<VAR, 1>(a, batch, st);
        case 2: return launch_cblock_t<VAR, 2>(a, batch, st);
        case 3: return launch_cblock_t<VAR, 3>(a, batch, st);
        case 4: return launch_cblock_t<VAR, 4>(a, batch, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace rg

namespace rg {

// ---------------------------------------------------------------------------
// 9-point complex variant for the Galerkin levels (VAR9, multigrid.py:62-68):
// same window scheme; rows flagged in `mask` use the repeated stencil c9
// (kernel parameters), the others read their 9 planes (L1/L2).  CSR column
// order (-1,-1),(-1,0),(-1,1),(0,-1),(0,0),(0,1),(1,-1),(1,0),(1,1),
// unfused complex products: bitwise the CSR matvec (apply_op<VAR9>).

// window rows: 16 x 64 windows (4-point threads) measured faster than 32 x 64
// at 511^2 (376 vs 430 us per 16-step smoothing call) and give 255^2 enough
// CTAs to take the blocked path
#ifndef CB9_LR
#define CB9_LR 16
#endif
#ifndef CB9_MINB
#define CB9_MINB 2
#endif
__host__ __device__ inline int cblock9_ntiles(int side, int T, int* nty) {
    const int TX = CB9_LR - 2 * T, TY = CB9_LC - 2 * T;
    const int ny = (side + TY - 1) / TY;
    if (nty) *nty = ny;
    return ((side + TX - 1) / TX) * ny;
}

struct CBlock9Args {
    double2 c9[9];
    const double2* planes;        // [9][P] (one coefficient set, shared by the batch)
    const unsigned char* mask;    // [P] 1: row == c9
    int side, P;
    const double2* u_in;
    const double2* v_in;
    double2* u_out;
    double2* v_out;
    const double2* f;
    const double* omega;
    const double* alpha;
    const double* atil;
    int m;
    int k0;
    int nty;
    int zero_in;                  // as CBlockArgs
};

// REALC: the repeated stencil c9 has zero imaginary parts (the Galerkin
// coarsening of the Helmholtz operator away from the sponge: R, P and the
// interior fine rows are real), so its products take 2 multiplies instead of
// 4 multiplies + 2 adds, exactly as REALOFF above (equal values, possibly
// another sign of an exact zero).
template <int VAR, int T, bool REALC>
__global__ void __launch_bounds__(CB_NW * 32, CB9_MINB) cblock9_kernel(const __grid_constant__ CBlock9Args a) {
    typedef double2 C;
    constexpr int LR = CB9_LR, LC = CB9_LC;
    constexpr int RPW = LR / CB_NW, CPT = LC / 32;
    constexpr int TX = LR - 2 * T, TY = LC - 2 * T;
    constexpr bool NAG = VAR >= V_NAG;
    constexpr bool HASV = VAR != V_PLAIN;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    typedef C Row[LC];
    Row* buf0 = reinterpret_cast<Row*>(smem_raw);
    Row* buf1 = buf0 + LR;
    Row* sf = buf1 + LR;

    const int b = blockIdx.y;
    const int cta = blockIdx.x;
    const int tx = cta / a.nty, ty = cta - (cta / a.nty) * a.nty;
    const int gx0 = tx * TX - T, gy0 = ty * TY - T;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int side = a.side;
    const size_t base = (size_t)b * a.P;
    const int r0 = wp * RPW;
    const size_t P = a.P;

    C ur[RPW][CPT], vr[RPW][CPT];
    int gidx[RPW][CPT];       // global index, -1 outside the grid; -2 - g for band rows
    const double at0 = NAG ? a.atil[b * a.m + (a.k0 % a.m)] : 0.0;
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
        const int gx = gx0 + r0 + rr;
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
            const int col = lane + 32 * cc;
            const int gy = gy0 + col;
            const bool in = (gx >= 0) && (gx < side) && (gy >= 0) && (gy < side);
            const int g = in ? gx * side + gy : -1;
            gidx[rr][cc] = (in && !a.mask[g]) ? -2 - g : g;
            const C u = (in && !(a.zero_in & 2)) ? a.u_in[base + g] : szero<C>();
            const C v = (HASV && in && !(a.zero_in & 1)) ? a.v_in[base + g] : szero<C>();
            ur[rr][cc] = u;
            vr[rr][cc] = v;
            sf[r0 + rr][col] = in ? a.f[base + g] : szero<C>();
            buf0[r0 + rr][col] = (NAG && in) ? add(u, rmul(at0, v)) : u;
        }
    }
    // the T steps' weights, loaded once (see block.cuh)
    __shared__ double sw[3][8];
    if (threadIdx.x < T) {
        const int k = a.k0 + threadIdx.x;
        const int si = b * a.m + (k % a.m);
        sw[0][threadIdx.x] = a.omega[si];
        sw[1][threadIdx.x] = HASV ? a.alpha[si] : 0.0;
        sw[2][threadIdx.x] = NAG ? a.atil[b * a.m + ((k + 1) % a.m)] : 0.0;
    }
    __syncthreads();

#pragma unroll
    for (int t = 0; t < T; ++t) {
        const double w = sw[0][t];
        const double al = sw[1][t];
        const double atn = sw[2][t];
        Row* cur = (t & 1) ? buf1 : buf0;
        Row* nxt = (t & 1) ? buf0 : buf1;
        const bool last = (t == T - 1);
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
            const int col = lane + 32 * cc;
            const int cm = col > 0 ? col - 1 : 0;
            const int cp = col < LC - 1 ? col + 1 : LC - 1;
            const int rm = r0 > 0 ? r0 - 1 : 0;
            C upw = cur[rm][cm], up = cur[rm][col], upe = cur[rm][cp];
            C mw = cur[r0][cm], mid = cur[r0][col], me = cur[r0][cp];
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr) {
                const int r = r0 + rr;
                const int rp = r + 1 < LR ? r + 1 : LR - 1;
                const C dw = cur[rp][cm], dn = cur[rp][col], de = cur[rp][cp];
                const int g = gidx[rr][cc];
                C s;
                if (g >= -1) {   // the repeated stencil (or outside the grid)
                    auto pr = [&](int q, const C& x) -> C { return REALC ? rmul(a.c9[q].x, x) : mul(a.c9[q], x); };
                    s = pr(0, upw);
                    s = add(s, pr(1, up));
                    s = add(s, pr(2, upe));
                    s = add(s, pr(3, mw));
                    s = add(s, pr(4, mid));
                    s = add(s, pr(5, me));
                    s = add(s, pr(6, dw));
                    s = add(s, pr(7, dn));
                    s = add(s, pr(8, de));
                } else {         // band row: its own coefficient planes
                    const C* c = a.planes + (size_t)(-2 - g);
                    s = mul(__ldg(&c[0]), upw);
                    s = add(s, mul(__ldg(&c[1 * P]), up));
                    s = add(s, mul(__ldg(&c[2 * P]), upe));
                    s = add(s, mul(__ldg(&c[3 * P]), mw));
                    s = add(s, mul(__ldg(&c[4 * P]), mid));
                    s = add(s, mul(__ldg(&c[5 * P]), me));
                    s = add(s, mul(__ldg(&c[6 * P]), dw));
                    s = add(s, mul(__ldg(&c[7 * P]), dn));
                    s = add(s, mul(__ldg(&c[8 * P]), de));
                }
                const C rs = sub(sf[r][col], s);
                C vn;
                if (VAR == V_PLAIN) vn = rmul(w, rs);
                else vn = add(rmul(al, vr[rr][cc]), rmul(w, rs));
                const C un = add(NAG ? ur[rr][cc] : mid, vn);
                if (HASV) vr[rr][cc] = vn;
                ur[rr][cc] = un;
                if (!last) {
                    const C x = NAG ? add(un, rmul(atn, vn)) : un;
                    nxt[r][col] = g != -1 ? x : szero<C>();
                }
                upw = mw; up = mid; upe = me;
                mw = dw; mid = dn; me = de;
            }
        }
        if (!last) __syncthreads();
    }
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
        const int r = r0 + rr;
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
            const int col = lane + 32 * cc;
            int g = gidx[rr][cc];
            if (g < -1) g = -2 - g;
            if (g >= 0 && r >= T && r < LR - T && col >= T && col < LC - T) {
                a.u_out[base + g] = ur[rr][cc];
                if (HASV) a.v_out[base + g] = vr[rr][cc];
            }
        }
    }
}

template <int VAR, int T, bool REALC>
cudaError_t launch_cblock9_t(const CBlock9Args& a0, int batch, cudaStream_t st) {
    auto kern = cblock9_kernel<VAR, T, REALC>;
    const size_t smem = 3 * (size_t)CB9_LR * CB9_LC * sizeof(double2);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    CBlock9Args a = a0;
    const int nt = cblock9_ntiles(a.side, T, &a.nty);
    kern<<<dim3(nt, batch), dim3(CB_NW * 32), smem, st>>>(a);
    return cudaGetLastError();
}

template <int VAR>
cudaError_t launch_cblock9(const CBlock9Args& a, int T, int batch, cudaStream_t st) {
    bool realc = true;
    for (int q = 0; q < 9; ++q) realc = realc && a.c9[q].y == 0.0;
    static const bool allow = [] { const char* e = getenv("RG_CB9_REALC"); return !e || atoi(e) != 0; }();
    realc = realc && allow;
#define RG_CB9(TT) return realc ? launch_cblock9_t<VAR, TT, true>(a, batch, st) : launch_cblock9_t<VAR, TT, false>(a, batch, st)
    switch (T) {
        case 1: RG_CB9(1);
        case 2: RG_CB9(2);
        case 3: RG_CB9(3);
        case 4: RG_CB9(4);
    }
#undef RG_CB9
    return cudaErrorInvalidValue;
}

}  // namespace rg

// block.cuh — temporally blocked Richardson / MOM / NAG sweeps for the
// constant 9-point anisotropic operator (real f64 / f32).
//
// One CTA owns an output tile of (LR-2T) x (LC-2T) points of one system and
// loads an LR x LC window (T-cell halo, zero outside the Dirichlet
// interior).  It then runs T inner steps of richardson.py:111-136 entirely
// on chip, shrinking the valid region by one cell per step (overlapped
// tiling), and writes back only its owned points.  HBM traffic per inner
// step is therefore ~1/T of the unblocked sweep and the kernel becomes
// FP64-issue bound (the reference's unfused mul+add order costs 17 of the
// ~22 FP64 instructions per point-update and cannot be contracted).
//
//  * The stencil input field (u for plain/mom, the look-ahead y = u + at*v
//    for nag/nagex) lives in shared memory, ping-ponged between steps (one
//    __syncthreads per step).  For plain/mom the centre of the 3x3 window
//    IS the thread's u, so u needs no register copy.
//  * f (and v, and u for nag) of the thread's own points live in registers
//    for all T steps.
//  * Stencil coefficients and the Jacobi scale arrive as kernel parameters
//    (uniform registers, no per-use moves).
//  * Thread mapping: lane -> column (conflict-free 64-bit smem rows), warp
//    -> a band of RPW rows walked with a 3x3 register window; the CPT
//    columns of a thread are summed interleaved for ILP.
//  * The region bookkeeping is branch-free: values computed outside the
//    shrinking valid region are garbage but are never read again (regions
//    are nested), out-of-domain points are forced to 0 in shared memory,
//    and only owned points are written back.
//  * Each step's residual norm (the lagged convergence test, reduce.cuh) is
//    accumulated over the owned points and reduced by the fused epilogue.
//  * Arithmetic order is exactly the reference's (no FMA): iterates are
//    bitwise equal to the CPU oracle.
#pragma once
#include <type_traits>

#include "step.cuh"

namespace rg {

constexpr int BLK_MAXB = 64;   // systems per launch (coefficients ride in the params)

template <typename S>
struct BlockArgs {
    CT<S> coef[BLK_MAXB][9];   // CSR-order stencil of systems b0 .. b0+gridDim.y-1
    CT<S> scale[BLK_MAXB];     // Jacobi scale (JAC instantiations)
    int b0;                // first system of this launch
    int side;
    int P;
    const S* u_in;
    const S* v_in;
    S* u_out;
    S* v_out;
    S* r_out;           // residual-only launch (T = 1): r = f - A u at the owned points, no update
    const S* f;
    const double* omega;
    const double* alpha;
    const double* atil;
    int m;
    int k0;             // global inner index of the first step of this launch
    int nty;            // tiles per system along y (columns)
    int norm_first_u;   // nag: ||f - A u||^2 at t = 0 (sweep-boundary test)
    int norm_every;     // plain/mom: the step residual norm at every t
    EpiArgs epi;
};

#ifndef RG_BLK_LR
#define RG_BLK_LR 64
#endif
#ifndef RG_BLK_NW
#define RG_BLK_NW 8
#endif
#ifndef RG_BLK_LC
#define RG_BLK_LC 64
#endif

// Occupancy target per (scalar, variant): registers hold f (+v, +u for nag).
#ifndef RG_MINB_PLAIN_F64
#define RG_MINB_PLAIN_F64 2
#endif
// (f32 storage computes in f64, so the register budget does not depend on S)
template <typename S, int VAR>
struct BlockMinCtas {
    static constexpr int value = (RG_BLK_LR * RG_BLK_LC * 16 > 100 * 1024) ? 1
                                 : ((VAR == V_PLAIN) ? RG_MINB_PLAIN_F64 : 2);
};

// Tile shape used by the library (load window LR x LC, NW warps).
constexpr int BLK_LR = RG_BLK_LR, BLK_LC = RG_BLK_LC, BLK_NW = RG_BLK_NW;

__host__ __device__ inline int block_ntiles(int side, int T, int* nty) {
    const int TX = BLK_LR - 2 * T, TY = BLK_LC - 2 * T;
    const int ntx = (side + TX - 1) / TX;
    const int ny = (side + TY - 1) / TY;
    if (nty) *nty = ny;
    return ntx * ny;
}

template <typename S, int VAR, int T, int LR, int LC, int NW, bool JAC>
__global__ void __launch_bounds__(NW * 32, (BlockMinCtas<S, VAR>::value))
block_kernel(const __grid_constant__ BlockArgs<S> a) {
    constexpr int NT = NW * 32;
    constexpr int RPW = LR / NW;   // rows per warp
    constexpr int CPT = LC / 32;   // columns per thread
    constexpr int TX = LR - 2 * T;
    constexpr int TY = LC - 2 * T;
    constexpr bool NAG = (VAR >= V_NAG);
    constexpr bool HASV = (VAR != V_PLAIN);
    constexpr int NACC = NAG ? 1 : T;
    static_assert(LR % NW == 0 && LC % 32 == 0 && T >= 1 && TX > 0 && TY > 0, "tile");
    static_assert(RPW * CPT <= 32, "domain mask");

    typedef CT<S> C;   // arithmetic type (f32 storage computes in f64)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    typedef C Row[LC];
    Row* buf0 = reinterpret_cast<Row*>(smem_raw);
    Row* buf1 = buf0 + LR;
    // nag keeps f in shared memory (u, v stay in registers) so that two CTAs
    // fit per SM; plain/mom keep f in registers
    constexpr bool F_SMEM = NAG;
    Row* sf = buf1 + LR;

    const int bl = blockIdx.y;          // system within this launch
    const int b = a.b0 + bl;            // global system index
    if (a.epi.st && a.epi.st[b].status != ST_ACTIVE) return;   // st == null: free-running sweep
    const int cta = blockIdx.x;
    const int ncta = gridDim.x;
    const int tx = cta / a.nty, ty = cta - (cta / a.nty) * a.nty;
    const int gx0 = tx * TX - T, gy0 = ty * TY - T;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int side = a.side;
    const size_t base = (size_t)b * a.P;
    const int r0 = wp * RPW;

    C c[9];
#pragma unroll
    for (int d = 0; d < 9; ++d) c[d] = a.coef[bl][d];
    const C sc = JAC ? a.scale[bl] : szero<C>();

    C fr[RPW][CPT], vr[RPW][CPT], ur[RPW][CPT];
    uint32_t dom = 0;  // bit (rr*CPT+cc): point inside the interior grid
    uint32_t own = 0;  // bit (rr*CPT+cc): point owned by this tile (not halo)

    const double at0 = NAG ? a.atil[b * a.m + (a.k0 % a.m)] : 0.0;
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
        const int gx = gx0 + r0 + rr;
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
            const int col = lane + 32 * cc;
            const int gy = gy0 + col;
            const bool in = (gx >= 0) && (gx < side) && (gy >= 0) && (gy < side);
            const size_t g = base + (size_t)gx * side + gy;
            const C u = in ? to_c(a.u_in[g]) : szero<C>();
            const C fv = in ? to_c(a.f[g]) : szero<C>();
            if (F_SMEM) sf[r0 + rr][col] = fv;
            else fr[rr][cc] = fv;
            vr[rr][cc] = (HASV && in) ? to_c(a.v_in[g]) : szero<C>();
            if (NAG) ur[rr][cc] = u;
            if (in) dom |= 1u << (rr * CPT + cc);
            if (!NAG) {   // plain/mom: owned-point bits for the per-step norm (+7% at T=5)
                const int r = r0 + rr;
                if (r >= T && r < LR - T && col >= T && col < LC - T) own |= 1u << (rr * CPT + cc);
            }
            C x = u;
            if (NAG && in) x = add(x, rmul(at0, vr[rr][cc]));  // y = u + at*v
            buf0[r0 + rr][col] = x;
            if (NAG && a.norm_first_u) buf1[r0 + rr][col] = u;
        }
    }
    // the T steps' weights, loaded once (a global load after every step's
    // barrier would stall all warps on L2 latency together)
    __shared__ double sw[3][8];
    if (threadIdx.x < T && !(T == 1 && a.r_out)) {   // (a residual-only launch has no schedule)
        const int k = a.k0 + threadIdx.x;
        const int si = b * a.m + (k % a.m);
        sw[0][threadIdx.x] = a.omega[si];
        sw[1][threadIdx.x] = HASV ? a.alpha[si] : 0.0;
        sw[2][threadIdx.x] = NAG ? a.atil[b * a.m + ((k + 1) % a.m)] : 0.0;
    }
    __syncthreads();

    double acc[NACC];
#pragma unroll
    for (int q = 0; q < NACC; ++q) acc[q] = 0.0;

    // Walk the warp's row band over `src`; for every owned point call
    // body(rr, cc, r, col, s, centre) with s = A x (CSR order, no FMA) and
    // centre = x at the point.  The CPT column chains are interleaved.
    auto sweep_rows = [&](Row* src, auto body) {
        int cm[CPT], cl[CPT], cp[CPT];
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
            cl[cc] = lane + 32 * cc;
            cm[cc] = cl[cc] > 0 ? cl[cc] - 1 : 0;
            cp[cc] = cl[cc] < LC - 1 ? cl[cc] + 1 : LC - 1;
        }
        const int rm = r0 > 0 ? r0 - 1 : 0;
        C w0[CPT], w1[CPT], w2[CPT], x0[CPT], x1[CPT], x2[CPT];
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
            w0[cc] = src[rm][cm[cc]]; w1[cc] = src[rm][cl[cc]]; w2[cc] = src[rm][cp[cc]];
            x0[cc] = src[r0][cm[cc]]; x1[cc] = src[r0][cl[cc]]; x2[cc] = src[r0][cp[cc]];
        }
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) {
            const int r = r0 + rr;
            const int rp = r + 1 < LR ? r + 1 : LR - 1;
            C y0[CPT], y1[CPT], y2[CPT], s[CPT];
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) {
                y0[cc] = src[rp][cm[cc]]; y1[cc] = src[rp][cl[cc]]; y2[cc] = src[rp][cp[cc]];
            }
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) s[cc] = mul(c[0], w0[cc]);
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) s[cc] = add(s[cc], mul(c[1], w1[cc]));
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) s[cc] = add(s[cc], mul(c[2], w2[cc]));
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) s[cc] = add(s[cc], mul(c[3], x0[cc]));
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) s[cc] = add(s[cc], mul(c[4], x1[cc]));
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) s[cc] = add(s[cc], mul(c[5], x2[cc]));
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) s[cc] = add(s[cc], mul(c[6], y0[cc]));
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) s[cc] = add(s[cc], mul(c[7], y1[cc]));
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) s[cc] = add(s[cc], mul(c[8], y2[cc]));
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) {
                body(rr, cc, r, cl[cc], s[cc], x1[cc]);
                w0[cc] = x0[cc]; w1[cc] = x1[cc]; w2[cc] = x2[cc];
                x0[cc] = y0[cc]; x1[cc] = y1[cc]; x2[cc] = y2[cc];
            }
        }
    };
    auto owned = [&](int r, int col) {
        return r >= T && r < LR - T && col >= T && col < LC - T;
    };
    auto indom = [&](int rr, int cc) { return ((dom >> (rr * CPT + cc)) & 1u) != 0; };
    auto isown = [&](int rr, int cc) { return ((own >> (rr * CPT + cc)) & 1u) != 0; };

    if (NAG && a.norm_first_u) {
        // residual at u itself for the sweep-boundary convergence test (:124-125)
        sweep_rows(buf1, [&](int rr, int cc, int r, int col, C s, C) {
            const C fv = F_SMEM ? sf[r][col] : fr[rr][cc];
            const C rs = (owned(r, col) && indom(rr, cc)) ? sub(fv, s) : szero<C>();
            acc[0] = sqacc(acc[0], rs);
        });
        __syncthreads();
    }

    // T inner steps; INTERIOR tiles (no point outside the grid, the common
    // case) skip the domain masking entirely.
    auto steps = [&](auto interior) {
        constexpr bool INTERIOR = decltype(interior)::value;
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const double w = sw[0][t];
            const double al = sw[1][t];
            const double atn = sw[2][t];
            Row* cur = (t & 1) ? buf1 : buf0;
            Row* nxt = (t & 1) ? buf0 : buf1;
            const bool last = (t == T - 1);
            sweep_rows(cur, [&](int rr, int cc, int r, int col, C s, C centre) {
                const bool live = INTERIOR || indom(rr, cc);
                const C fv = F_SMEM ? sf[r][col] : fr[rr][cc];
                const C rs = sub(fv, s);                                // r = f - A x
                if (!NAG && a.norm_every) {
                    // predicated accumulation over the owned points (no selects)
                    if (live && isown(rr, cc)) acc[(NACC > 1) ? t : 0] = sqacc(acc[(NACC > 1) ? t : 0], rs);
                }
                const C p = JAC ? mul(sc, rs) : rs;                      // B^{-1} r
                C vn;
                if (VAR == V_PLAIN) vn = rmul(w, p);
                else vn = add(rmul(al, vr[rr][cc]), rmul(w, p));         // v = a v + w p
                const C uo = NAG ? ur[rr][cc] : centre;                  // plain/mom: x == u
                const C un = stored<S>(add(uo, vn));                     // u = u + v (as stored)
                vn = stored<S>(vn);
                if (HASV) vr[rr][cc] = vn;
                if (NAG) ur[rr][cc] = un;
                if (!last) {
                    const C x = NAG ? add(un, rmul(atn, vn)) : un;       // next stencil input
                    nxt[r][col] = live ? x : szero<C>();
                } else if (live && (NAG ? owned(r, col) : isown(rr, cc))) {
                    const size_t g = base + (size_t)(gx0 + r) * side + (gy0 + col);
                    if (T == 1 && a.r_out) {
                        a.r_out[g] = to_s<S>(rs);                        // fns.py:80 residual
                    } else {
                        a.u_out[g] = to_s<S>(un);
                        if (HASV) a.v_out[g] = to_s<S>(vn);
                    }
                }
            });
            if (!last) __syncthreads();
        }
    };
    constexpr uint32_t FULL = (RPW * CPT == 32) ? 0xffffffffu : ((1u << (RPW * CPT)) - 1u);
    const bool tile_inside = (gx0 >= 0) && (gy0 >= 0) && (gx0 + LR <= side) && (gy0 + LC <= side);
    (void)FULL;
    if (tile_inside) steps(std::integral_constant<bool, true>());
    else steps(std::integral_constant<bool, false>());

    if (a.epi.nslots > 0) epilogue<NT, NACC>(a.epi, b, cta, ncta, acc, 0.0);
}

// Host launcher for one (scalar, variant, jacobi): picks the T instantiation.
template <typename S, int VAR, int T, bool JAC>
cudaError_t launch_block_t(const BlockArgs<S>& a, int nsys, cudaStream_t st) {
    auto kern = block_kernel<S, VAR, T, BLK_LR, BLK_LC, BLK_NW, JAC>;
    const size_t smem = (VAR >= V_NAG ? 3 : 2) * (size_t)BLK_LR * BLK_LC * sizeof(CT<S>);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int nt = block_ntiles(a.side, T, nullptr);
    kern<<<dim3(nt, nsys), dim3(BLK_NW * 32), smem, st>>>(a);
    return cudaGetLastError();
}

template <typename S, int VAR, bool JAC>
cudaError_t launch_block_j(const BlockArgs<S>& a, int T, int nsys, cudaStream_t st) {
    switch (T) {
        case 1: return launch_block_t<S, VAR, 1, JAC>(a, nsys, st);
        case 2: return launch_block_t<S, VAR, 2, JAC>(a, nsys, st);
        case 3: return launch_block_t<S, VAR, 3, JAC>(a, nsys, st);
        case 4: return launch_block_t<S, VAR, 4, JAC>(a, nsys, st);
        case 5: return launch_block_t<S, VAR, 5, JAC>(a, nsys, st);
        case 6: return launch_block_t<S, VAR, 6, JAC>(a, nsys, st);
        case 7: return launch_block_t<S, VAR, 7, JAC>(a, nsys, st);
        case 8: return launch_block_t<S, VAR, 8, JAC>(a, nsys, st);
    }
    return cudaErrorInvalidValue;
}

// a.nty must be set by the caller (block_ntiles(side, T, &nty)).
template <typename S, int VAR>
cudaError_t launch_block(const BlockArgs<S>& a, int T, bool jac, int nsys, cudaStream_t st) {
    return jac ? launch_block_j<S, VAR, true>(a, T, nsys, st)
               : launch_block_j<S, VAR, false>(a, T, nsys, st);
}

// Explicit instantiations live in block_<dtype>_<variant>.cu (parallel build).
#define RG_DECLARE_BLOCK(S, VAR) \
    extern template cudaError_t launch_block<S, VAR>(const BlockArgs<S>&, int, bool, int, cudaStream_t);
RG_DECLARE_BLOCK(double, V_PLAIN)
RG_DECLARE_BLOCK(double, V_MOM)
RG_DECLARE_BLOCK(double, V_NAG)
RG_DECLARE_BLOCK(float, V_PLAIN)
RG_DECLARE_BLOCK(float, V_MOM)
RG_DECLARE_BLOCK(float, V_NAG)

}  // namespace rg

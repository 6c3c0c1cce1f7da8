// block.cuh — temporally blocked Richardson / MOM / NAG sweeps for the
// constant 9-point anisotropic operator (real f64 / f32).
//
// One CTA owns an output tile of (LR-2T) x (LC-2T) points of one system and
// loads an LR x LC window (T-cell halo, zero outside the Dirichlet
// interior).  It then runs T inner steps of richardson.py:111-136 entirely
// on chip, shrinking the valid region by one cell per step (overlapped
// tiling), and writes back only its owned points.  HBM traffic per inner
// step is therefore ~1/T of the unblocked sweep.
//
//  * The stencil input field (u for plain/mom, the look-ahead y = u + at*v
//    for nag/nagex) lives in shared memory, ping-ponged between steps
//    (one __syncthreads per step).
//  * u, v, f of the thread's own points live in registers for all T steps.
//  * Thread mapping: lane -> column (conflict-free 64-bit smem rows), warp
//    -> a band of RPW rows walked with a 3x3 register window.
//  * Each step's residual norm (the lagged convergence test, see
//    reduce.cuh) is accumulated over the owned points and reduced by the
//    fused epilogue.
//  * Arithmetic order is exactly the reference's (no FMA): iterates are
//    bitwise equal to the CPU oracle.
#pragma once
#include "step.cuh"

namespace rg {

template <typename S>
struct BlockArgs {
    const S* stencil;   // [B][9]
    int side;
    int P;
    const S* u_in;
    const S* v_in;
    S* u_out;
    S* v_out;
    const S* f;
    const double* omega;
    const double* alpha;
    const double* atil;
    const S* scale;     // [B] Jacobi scale or null
    int m;
    int k0;             // global inner index of the first step of this launch
    int nty;            // tiles per system along y (columns)
    int norm_first_u;   // nag: ||f - A u||^2 at t = 0 (sweep-boundary test)
    int norm_every;     // plain/mom: the step residual norm at every t
    EpiArgs epi;
};

// Occupancy target: plain keeps u, f per point in registers (2 CTAs/SM at
// f64); mom/nag also keep v and need the whole register file.
template <typename S, int VAR>
struct BlockMinCtas {
    static constexpr int value = (VAR == V_PLAIN) ? (sizeof(S) == 8 ? 2 : 3) : (sizeof(S) == 8 ? 1 : 2);
};

// Tile shape used by the library (load window LR x LC, NW warps).
constexpr int BLK_LR = 64, BLK_LC = 64, BLK_NW = 8;

__host__ __device__ inline int block_ntiles(int side, int T, int* nty) {
    const int TX = BLK_LR - 2 * T, TY = BLK_LC - 2 * T;
    const int ntx = (side + TX - 1) / TX;
    const int ny = (side + TY - 1) / TY;
    if (nty) *nty = ny;
    return ntx * ny;
}

template <typename S, int VAR, int T, int LR, int LC, int NW>
__global__ void __launch_bounds__(NW * 32, (BlockMinCtas<S, VAR>::value))
block_kernel(BlockArgs<S> a) {
    constexpr int NT = NW * 32;
    constexpr int RPW = LR / NW;   // rows per warp
    constexpr int CPT = LC / 32;   // columns per thread
    constexpr int TX = LR - 2 * T;
    constexpr int TY = LC - 2 * T;
    constexpr bool NAG = (VAR >= V_NAG);
    constexpr bool HASV = (VAR != V_PLAIN);
    constexpr int NACC = NAG ? 1 : T;
    static_assert(LR % NW == 0 && LC % 32 == 0 && T >= 1 && TX > 0 && TY > 0, "tile");

    extern __shared__ __align__(16) unsigned char smem_raw[];
    typedef S Row[LC];
    Row* buf0 = reinterpret_cast<Row*>(smem_raw);
    Row* buf1 = buf0 + LR;

    const int b = blockIdx.y;
    if (a.epi.st[b].status != ST_ACTIVE) return;
    const int cta = blockIdx.x;
    const int ncta = gridDim.x;
    const int tx = cta / a.nty, ty = cta - (cta / a.nty) * a.nty;
    const int gx0 = tx * TX - T, gy0 = ty * TY - T;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int side = a.side;
    const size_t base = (size_t)b * a.P;
    const int r0 = wp * RPW;

    S c[9];
#pragma unroll
    for (int d = 0; d < 9; ++d) c[d] = a.stencil[b * 9 + d];
    const bool jac = (a.scale != nullptr);
    const S sc = jac ? a.scale[b] : szero<S>();

    S ur[RPW][CPT], fr[RPW][CPT], vr[RPW][CPT];
    uint32_t dom = 0;  // bit (rr*CPT+cc): point inside the interior grid
    static_assert(RPW * CPT <= 32, "domain mask");

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
            ur[rr][cc] = in ? a.u_in[g] : szero<S>();
            fr[rr][cc] = in ? a.f[g] : szero<S>();
            vr[rr][cc] = (HASV && in) ? a.v_in[g] : szero<S>();
            if (in) dom |= 1u << (rr * CPT + cc);
            S x = ur[rr][cc];
            if (NAG && in) x = add(x, rmul(at0, vr[rr][cc]));  // y = u + at*v
            buf0[r0 + rr][col] = x;
            if (NAG && a.norm_first_u) buf1[r0 + rr][col] = ur[rr][cc];
        }
    }
    __syncthreads();

    double acc[NACC];
#pragma unroll
    for (int q = 0; q < NACC; ++q) acc[q] = 0.0;

    // Walk the warp's row band over `src`, calling body(rr, cc, s) with the
    // stencil sum s = A x at every point in rows [lo, hi) x cols [lo, LC-lo').
    auto sweep_rows = [&](Row* src, int lo, int hi, int clo, int chi, auto body) {
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
            const int col = lane + 32 * cc;
            const int cm = col > 0 ? col - 1 : 0;
            const int cp = col < LC - 1 ? col + 1 : LC - 1;
            const bool colok = (col >= clo) && (col < chi);
            const int rm = r0 > 0 ? r0 - 1 : 0;
            S a0 = src[rm][cm], a1 = src[rm][col], a2 = src[rm][cp];
            S b0 = src[r0][cm], b1 = src[r0][col], b2 = src[r0][cp];
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr) {
                const int r = r0 + rr;
                const int rp = r + 1 < LR ? r + 1 : LR - 1;
                const S c0 = src[rp][cm], c1 = src[rp][col], c2 = src[rp][cp];
                if (r >= lo && r < hi && colok) {
                    S s = mul(c[0], a0);
                    s = add(s, mul(c[1], a1));
                    s = add(s, mul(c[2], a2));
                    s = add(s, mul(c[3], b0));
                    s = add(s, mul(c[4], b1));
                    s = add(s, mul(c[5], b2));
                    s = add(s, mul(c[6], c0));
                    s = add(s, mul(c[7], c1));
                    s = add(s, mul(c[8], c2));
                    body(rr, cc, r, col, s);
                }
                a0 = b0; a1 = b1; a2 = b2;
                b0 = c0; b1 = c1; b2 = c2;
            }
        }
    };
    auto owned = [&](int r, int col) {
        return r >= T && r < LR - T && col >= T && col < LC - T;
    };

    if (NAG && a.norm_first_u) {
        // residual at u itself for the sweep-boundary convergence test (:124-125)
        sweep_rows(buf1, T, LR - T, T, LC - T, [&](int rr, int cc, int r, int col, S s) {
            if ((dom >> (rr * CPT + cc)) & 1u) acc[0] = sqacc(acc[0], sub(fr[rr][cc], s));
        });
        __syncthreads();
    }

#pragma unroll
    for (int t = 0; t < T; ++t) {
        const int k = a.k0 + t;
        const int si = b * a.m + (k % a.m);
        const double w = a.omega[si];
        const double al = HASV ? a.alpha[si] : 0.0;
        const double atn = NAG ? a.atil[b * a.m + ((k + 1) % a.m)] : 0.0;
        Row* cur = (t & 1) ? buf1 : buf0;
        Row* nxt = (t & 1) ? buf0 : buf1;
        const bool last = (t == T - 1);
        sweep_rows(cur, t + 1, LR - t - 1, t + 1, LC - t - 1,
                   [&](int rr, int cc, int r, int col, S s) {
            S x = szero<S>();
            if ((dom >> (rr * CPT + cc)) & 1u) {
                const S rs = sub(fr[rr][cc], s);                       // r = f - A x
                if (!NAG && a.norm_every && owned(r, col)) acc[(NACC > 1) ? t : 0] = sqacc(acc[(NACC > 1) ? t : 0], rs);
                const S p = jac ? mul(sc, rs) : rs;                     // B^{-1} r
                S vn;
                if (VAR == V_PLAIN) vn = rmul(w, p);
                else vn = add(rmul(al, vr[rr][cc]), rmul(w, p));        // v = a v + w p
                const S un = add(ur[rr][cc], vn);                       // u = u + v
                ur[rr][cc] = un;
                if (HASV) vr[rr][cc] = vn;
                x = NAG ? add(un, rmul(atn, vn)) : un;
            }
            if (!last) nxt[r][col] = x;
        });
        if (!last) __syncthreads();
    }

    // write back the owned points
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
        const int r = r0 + rr;
        const int gx = gx0 + r;
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
            const int col = lane + 32 * cc;
            if (owned(r, col) && ((dom >> (rr * CPT + cc)) & 1u)) {
                const size_t g = base + (size_t)gx * side + (gy0 + col);
                a.u_out[g] = ur[rr][cc];
                if (HASV) a.v_out[g] = vr[rr][cc];
            }
        }
    }

    if (a.epi.nslots > 0) epilogue<NT, NACC>(a.epi, b, cta, ncta, acc, 0.0);
}

// Host launcher for one (scalar, variant): picks the T instantiation.
template <typename S, int VAR, int T>
cudaError_t launch_block_t(const BlockArgs<S>& a0, int batch, cudaStream_t st) {
    auto kern = block_kernel<S, VAR, T, BLK_LR, BLK_LC, BLK_NW>;
    const size_t smem = 2 * (size_t)BLK_LR * BLK_LC * sizeof(S);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    BlockArgs<S> a = a0;
    const int nt = block_ntiles(a.side, T, &a.nty);
    kern<<<dim3(nt, batch), dim3(BLK_NW * 32), smem, st>>>(a);
    return cudaGetLastError();
}

template <typename S, int VAR>
cudaError_t launch_block(const BlockArgs<S>& a, int T, int batch, cudaStream_t st) {
    switch (T) {
        case 1: return launch_block_t<S, VAR, 1>(a, batch, st);
        case 2: return launch_block_t<S, VAR, 2>(a, batch, st);
        case 3: return launch_block_t<S, VAR, 3>(a, batch, st);
        case 4: return launch_block_t<S, VAR, 4>(a, batch, st);
        case 5: return launch_block_t<S, VAR, 5>(a, batch, st);
        case 6: return launch_block_t<S, VAR, 6>(a, batch, st);
        case 7: return launch_block_t<S, VAR, 7>(a, batch, st);
        case 8: return launch_block_t<S, VAR, 8>(a, batch, st);
    }
    return cudaErrorInvalidValue;
}

// Explicit instantiations live in block_<dtype>_<variant>.cu (parallel build).
#define RG_DECLARE_BLOCK(S, VAR) \
    extern template cudaError_t launch_block<S, VAR>(const BlockArgs<S>&, int, int, cudaStream_t);
RG_DECLARE_BLOCK(double, V_PLAIN)
RG_DECLARE_BLOCK(double, V_MOM)
RG_DECLARE_BLOCK(double, V_NAG)
RG_DECLARE_BLOCK(float, V_PLAIN)
RG_DECLARE_BLOCK(float, V_MOM)
RG_DECLARE_BLOCK(float, V_NAG)

}  // namespace rg

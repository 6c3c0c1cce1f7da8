// trigen.cuh — Gauss-Seidel / SOR / SSOR for every operator the reference
// builds them for (precond.py:86-118 takes any SparseMatrix): per-node
// coefficients (VAR9 planes: the Galerkin level operators), the Helmholtz
// DIAG5 form (constant off-diagonals, per-node diagonal) and complex128
// scalars.  The constant-coefficient real case, which is the one the
// paper's solver families use, has its own fast kernel (tri.cuh); this one
// favours generality: one CTA per system, thread t owns grid row p0 + t of
// the current pass and walks it one point per step on the slope-2 wavefront
// (point (i, j) at step j + 2 i), the row above arrives by warp shuffle /
// a two-slot mailbox between warps / `edge` between passes, one
// __syncthreads per step, and right-hand side and coefficients are read
// straight from global memory (each thread walks its own row, so an L1
// line serves 16 real / 8 complex steps).
//
// A sweep solves M x = rhs in traversal order (reversed index order when
// REV) for M = D + w L, D + w U or their transposes.  Slot s = 0..3 of a
// point p is its neighbour at traversal offset (-1,-1), (-1,0), (-1,+1),
// (0,-1), i.e. natural offset o = +-(that).  Matrix entry of the slot:
//   plain       M[p][p+o]   = w * plane(o)  read at p,
//   transposed  M^T[p][p+o] = w * plane(-o) read at p + o
// (plane(di, dj) = stencil plane 3 (di + 1) + (dj + 1); sparse.py:101-106
// CSR order).  Arithmetic: x = (rhs - sum_s m_s x_s) / d_p, complex
// products and quotient in the textbook form; SuperLU rounds differently
// (~1e-15), the reference's own bar for these maps is 1e-13
// (test_precond.py:33-62).
#pragma once
#include "common.cuh"
#include "tri.cuh"

namespace rg {

__device__ __forceinline__ double cdivq(double a, double b) { return a / b; }
__device__ __forceinline__ double2 cdivq(double2 a, double2 b) {
    // Smith's algorithm (no overflow for moderate ratios, ~1 ulp per part)
    if (fabs(b.x) >= fabs(b.y)) {
        const double r = b.y / b.x, den = b.x + b.y * r;
        return make_double2((a.x + a.y * r) / den, (a.y - a.x * r) / den);
    }
    const double r = b.x / b.y, den = b.x * r + b.y;
    return make_double2((a.x * r + a.y) / den, (a.y * r - a.x) / den);
}
__device__ __forceinline__ double tg_shfl_up(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double2 tg_shfl_up(double2 v) {
    return make_double2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}

template <typename S>
struct TriGenArgs {
    const CT<S>* stencil;   // CONST9 [B][9] | DIAG5 [B][4] | VAR9 [B][9][P]
    const CT<S>* diag;      // DIAG5 [B][P]
    int shared;
    int side, P;
    double relax;
    const S* r;
    S* z;
    S* work;                // SSOR: first sweep's result [B][P]
};

// plane(q) of system coefficients cb at natural point index p (zero where
// the stencil has no such plane)
template <typename C, int KIND>
__device__ __forceinline__ C trigen_coef(const C* cb, const C* dg, int q, long long p, int P) {
    if (KIND == K_CONST9) return cb[q];
    if (KIND == K_VAR9) return cb[(size_t)q * P + p];
    // DIAG5: c0 (-1,0) c1 (0,-1) [diag] c2 (0,+1) c3 (+1,0)
    switch (q) {
        case 1: return cb[0];
        case 3: return cb[1];
        case 4: return dg[p];
        case 5: return cb[2];
        case 7: return cb[3];
        default: return szero<C>();
    }
}

// One substitution sweep: dst = oscale * x, M x = rhs (rhs = src, or
// d * src when MULD), see the header.  edge: [side] of C; xfer: [32][2].
template <typename S, int KIND, bool REV, bool TRANS, bool MULD>
__device__ void trigen_sweep(const TriGenArgs<S>& a, const CT<S>* cb, const CT<S>* dg,
                             const S* __restrict__ src, S* __restrict__ dst, double oscale,
                             CT<S>* edge, CT<S> (*xfer)[2]) {
    typedef CT<S> C;
    const int side = a.side, P = a.P;
    const int t = threadIdx.x, NT = blockDim.x, lane = t & 31, wp = t >> 5, nw = NT >> 5;
    const double w = a.relax;
    // natural offsets of the four slots and the plane each one reads
    const int sg = REV ? -1 : 1;
    const int odi[4] = {-sg, -sg, -sg, 0}, odj[4] = {-sg, 0, sg, -sg};
    for (int p0 = 0; p0 < side; p0 += NT) {
        const int ip = p0 + t;                      // traversal-order row
        const bool row_ok = ip < side;
        const int nrows = min(NT, side - p0);
        const int nsteps = side + 2 * (nrows - 1);
        if (t < nw) xfer[t][0] = xfer[t][1] = szero<C>();
        C left = szero<C>(), nm1 = szero<C>(), n0 = szero<C>(), pub = szero<C>();
        if (t == 0 && p0 > 0) n0 = edge[0];
        __syncthreads();
        for (int s = 0; s < nsteps; ++s) {
            const int jp = s - 2 * t;               // traversal-order column
            const bool act = row_ok && (unsigned)jp < (unsigned)side;
            const C sh = tg_shfl_up(pub);
            const C mb = xfer[wp][(s + 1) & 1];
            const C ev = (p0 > 0 && (unsigned)(jp + 1) < (unsigned)side) ? edge[jp + 1] : szero<C>();
            const C nb = lane != 0 ? sh : (wp > 0 ? mb : ev);
            C x = szero<C>();
            if (act) {
                const int i = REV ? side - 1 - ip : ip, j = REV ? side - 1 - jp : jp;   // natural
                const long long p = (long long)i * side + j;
                const C d = trigen_coef<C, KIND>(cb, dg, 4, p, P);
                C m[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int ni = i + odi[q], nj = j + odj[q];
                    const bool in = (unsigned)ni < (unsigned)side && (unsigned)nj < (unsigned)side;
                    const int plane = TRANS ? 3 * (1 - odi[q]) + (1 - odj[q]) : 3 * (odi[q] + 1) + (odj[q] + 1);
                    const long long at = TRANS ? (long long)ni * side + nj : p;
                    m[q] = in ? trigen_coef<C, KIND>(cb, dg, plane, at, P) : szero<C>();
                }
                C rhs = to_c(src[p]);
                if (MULD) rhs = mul(d, rhs);
                C acc = mul(m[0], nm1);
                acc = add(acc, mul(m[1], n0));
                acc = add(acc, mul(m[2], nb));
                acc = add(acc, mul(m[3], left));
                x = cdivq(sub(rhs, rmul(w, acc)), d);
                dst[p] = to_s<S>(rmul(oscale, x));
                if (t == NT - 1) edge[jp] = x;
            }
            nm1 = n0;
            n0 = nb;
            left = x;
            pub = x;
            if (lane == 31 && wp + 1 < nw) xfer[wp + 1][s & 1] = x;
            __syncthreads();
        }
    }
}

template <typename S, int KIND, int MODE>
__global__ void __launch_bounds__(1024, 1) trigen_kernel(const TriGenArgs<S> a) {
    typedef CT<S> C;
    extern __shared__ double trigen_smem[];
    C* edge = reinterpret_cast<C*>(trigen_smem);      // [side]
    __shared__ C xfer[32][2];
    const int b = blockIdx.x;
    const size_t cstride = KIND == K_CONST9 ? 9 : (KIND == K_DIAG5 ? 4 : (size_t)9 * a.P);
    const C* cb = a.stencil + (a.shared ? 0 : (size_t)b * cstride);
    const C* dg = KIND == K_DIAG5 ? a.diag + (a.shared ? 0 : (size_t)b * a.P) : nullptr;
    const size_t base = (size_t)b * a.P;
    const double w = a.relax;
    if (MODE == TRI_SOR) {
        // relax * solve(r)  (precond.py:93)
        trigen_sweep<S, KIND, false, false, false>(a, cb, dg, a.r + base, a.z + base, w, edge, xfer);
    } else if (MODE == TRI_SOR_T) {
        // relax * solve_t(r)  (precond.py:94)
        trigen_sweep<S, KIND, true, true, false>(a, cb, dg, a.r + base, a.z + base, w, edge, xfer);
    } else if (MODE == TRI_SSOR_T) {
        // c * dlt(diag * dut(r))  (precond.py:112-113)
        trigen_sweep<S, KIND, false, true, false>(a, cb, dg, a.r + base, a.work + base, 1.0, edge, xfer);
        __syncthreads();
        trigen_sweep<S, KIND, true, true, true>(a, cb, dg, a.work + base, a.z + base, w * (2.0 - w), edge, xfer);
    } else {
        // c * du(diag * dl(r))  (precond.py:109-110)
        trigen_sweep<S, KIND, false, false, false>(a, cb, dg, a.r + base, a.work + base, 1.0, edge, xfer);
        __syncthreads();
        trigen_sweep<S, KIND, true, false, true>(a, cb, dg, a.work + base, a.z + base, w * (2.0 - w), edge, xfer);
    }
}

template <typename S, int KIND>
cudaError_t launch_trigen(const TriGenArgs<S>& a, int mode, int batch, cudaStream_t st) {
    int nt = (a.side + 31) / 32 * 32;
    if (nt > 1024) nt = 1024;
    const size_t smem = (size_t)a.side * sizeof(CT<S>);
#define RG_TG(M)                                                                                   \
    {                                                                                              \
        auto k = trigen_kernel<S, KIND, M>;                                                        \
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e != cudaSuccess) return e;                                                            \
        k<<<batch, nt, smem, st>>>(a);                                                             \
        return cudaGetLastError();                                                                 \
    }
    switch (mode) {
        case TRI_SOR: RG_TG(TRI_SOR)
        case TRI_SOR_T: RG_TG(TRI_SOR_T)
        case TRI_SSOR_T: RG_TG(TRI_SSOR_T)
        default: RG_TG(TRI_SSOR)
    }
#undef RG_TG
}

// instantiated in trigen.cu (parallel build)
#define RG_TRIGEN_EXTERN(S)                                                                              \
    extern template cudaError_t launch_trigen<S, K_CONST9>(const TriGenArgs<S>&, int, int, cudaStream_t); \
    extern template cudaError_t launch_trigen<S, K_DIAG5>(const TriGenArgs<S>&, int, int, cudaStream_t);  \
    extern template cudaError_t launch_trigen<S, K_VAR9>(const TriGenArgs<S>&, int, int, cudaStream_t);
RG_TRIGEN_EXTERN(float)
RG_TRIGEN_EXTERN(double)
RG_TRIGEN_EXTERN(double2)
#undef RG_TRIGEN_EXTERN

}  // namespace rg

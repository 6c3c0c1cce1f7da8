// wave.cuh — wavefront temporal blocking of the plain (Jacobi-)Richardson
// sweep for the constant 9-point operator (real f64 / f32 storage).
//
// The overlapped-tile kernel (block.cuh) recomputes a T-cell halo on all
// four sides of a 64 x 64 window: 1.41-1.57 computed point-steps per owned
// one at T = 5.  Here a CTA owns a strip of 128 window columns (4 per lane)
// and STREAMS DOWN the rows of a segment: at stage s it loads row s of u and
// f, and step (level) t = 1..T updates row s - 2t.  Level t's input rows were
// all produced by level t-1 at earlier stages, so the levels of one stage are
// independent, and the halo is recomputed only across strip edges (2T
// columns) and segment ends (T rows): ~1.07 x 1.05 at T = 4.
//
//  * The T levels are split over the CTA's NW warps (T/NW consecutive levels
//    each, a software pipeline): every warp keeps, for each of its levels,
//    the level's input rows rho-1 and rho over the lane's 6 window columns
//    (4*lane-1 .. 4*lane+4) in registers, and gets the new row rho+1 from the
//    level below -- its own register output (neighbour columns by warp
//    shuffle) or, at a warp boundary, a shared-memory hand-off row.  u and f
//    stream in through cp.async rings PD rows ahead.  One named barrier per
//    stage (a __syncwarp for NW = 1).  Splitting the levels halves the
//    registers a thread needs, so twice the warps fit on an SM.
//  * Steady stages (every level's row valid and owned) run a branch-free body
//    so the scheduler can interleave the levels' FP64 chains; the pipeline
//    fill/drain stages check each level's row range.
//  * Out-of-domain points are forced to 0 at every level (Dirichlet); the
//    shrinking valid region of overlapped tiling handles the strip edges
//    (garbage there never reaches an owned point).
//  * The arithmetic per point is exactly block.cuh's (CSR-order unfused
//    stencil sum, r = f - s, p = scale r, v = w p, u = u + v), so iterates
//    are bitwise those of the CPU oracle; the per-step norms accumulate over
//    the owned points and go through the fused epilogue (reduce.cuh).
#pragma once
#include "block.cuh"

namespace rg {

constexpr int WV_CPT = 4;              // columns per lane
constexpr int WV_W = 32 * WV_CPT;      // window columns per CTA
#ifndef RG_WV_PD
#define RG_WV_PD 3                     // cp.async prefetch distance (rows)
#endif
constexpr int WV_PD = RG_WV_PD;
#ifndef RG_WV_L
#define RG_WV_L 64                     // owned rows per segment
#endif
#ifndef RG_WV_NW
#define RG_WV_NW 1                     // warps per CTA (2: levels split between them; measured slower)
#endif
#ifndef RG_WV_REGS
#define RG_WV_REGS 128                 // register target per thread when NW = 2
#endif
#ifndef RG_WV_REGS1
#define RG_WV_REGS1 224                // ... when NW = 1 (9 one-warp CTAs per SM)
#endif

template <typename S>
struct WaveArgs {
    CT<S> coef[BLK_MAXB][9];
    CT<S> scale[BLK_MAXB];
    int b0;
    int side;
    int P;
    const S* u_in;
    S* u_out;
    const S* f;
    const double* omega;
    int m;
    int k0;
    int nstrip;     // column strips per system
    int seg_rows;   // owned rows per segment (last one may be shorter)
    EpiArgs epi;
};

__host__ __device__ inline int wave_ntiles(int side, int T, int L, int* nstrip) {
    const int ow = WV_W - 2 * T;
    const int ns = (side + ow - 1) / ow;
    if (nstrip) *nstrip = ns;
    return ns * ((side + L - 1) / L);
}

// warps per CTA for depth T (2 when T is even and the split is enabled)
__host__ __device__ constexpr int wave_nw(int T) {
    return (RG_WV_NW >= 2 && T % 2 == 0) ? 2 : 1;
}

template <typename S, int T>
struct WaveSmem {
    static constexpr int RU = WV_PD + 3;            // u ring: loaded PD ahead, read one stage later (+1 slack)
    static constexpr int RF = WV_PD + 2 * T + 2;    // f ring: row rho read until stage rho + 2T
    static constexpr int UW = WV_W + 2;             // zero pad column each side
    static constexpr int NH = wave_nw(T) - 1;       // hand-off rows between warps (ping-pong)
    static constexpr size_t bytes =
        sizeof(CT<S>) * ((size_t)RU * UW + (size_t)RF * WV_W + (size_t)NH * 2 * UW);
};

__device__ __forceinline__ double shfl_up1(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double shfl_dn1(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }

template <int NW>
__device__ __forceinline__ void wave_barrier() {
    if (NW > 1) asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
    else __syncwarp();
}

template <typename S, int T, int NW, bool JAC>
__device__ __forceinline__ void wave_body(const WaveArgs<S>& a, int b, int bl, int strip, int seg,
                                          double (&acc)[T / NW]) {
    typedef CT<S> C;
    typedef WaveSmem<S, T> SM;
    constexpr int NC = WV_CPT + 2;
    constexpr int LPW = T / NW;                     // levels per warp
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C (*su)[SM::UW] = reinterpret_cast<C (*)[SM::UW]>(smem_raw);
    C (*sf)[WV_W] = reinterpret_cast<C (*)[WV_W]>(smem_raw + sizeof(C) * SM::RU * SM::UW);
    C (*sh)[SM::UW] = reinterpret_cast<C (*)[SM::UW]>(
        smem_raw + sizeof(C) * (SM::RU * SM::UW + SM::RF * WV_W));   // [NW-1][2] hand-off rows

    const int lane = threadIdx.x & 31;
    const int wp = NW > 1 ? (int)(threadIdx.x >> 5) : 0;   // compile-time 0 for one warp
    const int t0 = wp * LPW;                        // this warp's levels: t0+1 .. t0+LPW
    const int side = a.side;
    const size_t base = (size_t)b * a.P;
    const int OW = WV_W - 2 * T;
    const int gc0 = strip * OW - T;                 // global column of window column 0
    const int R0 = seg * a.seg_rows;
    const int L = min(a.seg_rows, side - R0);       // owned rows
    const int gr0 = R0 - T;                         // global row of local row 0
    const int NLOAD = L + 2 * T;                    // base-level rows
    const int NS = L + 3 * T;                       // stages

    C c[9];
#pragma unroll
    for (int d = 0; d < 9; ++d) c[d] = a.coef[bl][d];
    const C sc = JAC ? a.scale[bl] : szero<C>();
    double w[LPW];
#pragma unroll
    for (int j = 0; j < LPW; ++j) w[j] = a.omega[b * a.m + ((a.k0 + t0 + j) % a.m)];

    bool colin[WV_CPT], colown[WV_CPT];
#pragma unroll
    for (int q = 0; q < WV_CPT; ++q) {
        const int lc = WV_CPT * lane + q;
        const int gc = gc0 + lc;
        colin[q] = gc >= 0 && gc < side;
        colown[q] = lc >= T && lc < WV_W - T && colin[q];
    }

    // zero the u ring and the hand-off rows (their pad columns stay 0)
    for (int i = threadIdx.x; i < SM::RU * SM::UW; i += NW * 32) (&su[0][0])[i] = szero<C>();
    for (int i = threadIdx.x; i < SM::NH * 2 * SM::UW; i += NW * 32) (&sh[0][0])[i] = szero<C>();
    wave_barrier<NW>();   // before warp 0's first cp.async into the ring

    // ring slots advance with the stage counter (no integer division)
    int ld_u = 0, ld_f = 0;                         // slots of the next row to load (warp 0)
    auto load_row = [&](int rho) {
        if (rho < NLOAD) {
            const int gr = gr0 + rho;
            const bool rin = gr >= 0 && gr < side;
            C* du = &su[ld_u][1 + WV_CPT * lane];
            C* df = &sf[ld_f][WV_CPT * lane];
#pragma unroll
            for (int q = 0; q < WV_CPT; ++q) {
                const bool in = rin && colin[q];
                const size_t g = in ? base + (size_t)gr * side + (gc0 + WV_CPT * lane + q) : base;
                cp_async_el<sizeof(S) == 8 ? 8 : 4>(du + q, a.u_in + g, in);
                cp_async_el<sizeof(S) == 8 ? 8 : 4>(df + q, a.f + g, in);
            }
        }
        cp_async_commit();
        ld_u = ld_u + 1 == SM::RU ? 0 : ld_u + 1;
        ld_f = ld_f + 1 == SM::RF ? 0 : ld_f + 1;
    };
    static_assert(sizeof(C) == sizeof(S) || sizeof(S) == 4, "storage");
    // f32 storage: the rings are typed in the arithmetic type (double) and
    // cp.async writes the 4 stored bytes at the start of each slot, so the
    // readers reinterpret the slot as S (hand-off rows hold C values)
    auto ldu = [&](int slot, int col) -> C {
        if (sizeof(S) == sizeof(C)) return su[slot][col];
        return to_c(*reinterpret_cast<const S*>(&su[slot][col]));
    };
    auto ldf = [&](int slot, int col) -> C {
        if (sizeof(S) == sizeof(C)) return sf[slot][col];
        return to_c(*reinterpret_cast<const S*>(&sf[slot][col]));
    };

    if (wp == 0) {
#pragma unroll
        for (int p = 0; p < WV_PD; ++p) load_row(p);
    }

    // per level j of this warp: input rows rho-1 (A) and rho (Bw) of level
    // t0+j+1 over the lane's 6 window columns; O = the level's newest output
    C A[LPW][NC], Bw[LPW][NC], O[LPW][WV_CPT];
#pragma unroll
    for (int j = 0; j < LPW; ++j) {
#pragma unroll
        for (int q = 0; q < NC; ++q) { A[j][q] = szero<C>(); Bw[j][q] = szero<C>(); }
#pragma unroll
        for (int q = 0; q < WV_CPT; ++q) O[j][q] = szero<C>();
    }
    int s_u = SM::RU - 1, s_f = 0;    // u slot of row s-1, f slot of row s
    // One stage.  STEADY: every level's row is valid, owned and in the grid
    // (no per-level branches, so the scheduler can interleave the levels'
    // FP64 chains).  COLIN: every window column is in the grid (no column
    // masks).
    auto stage = [&](int s, auto steady_c, auto colin_c) {
        constexpr bool STEADY = decltype(steady_c)::value;
        constexpr bool COLIN = decltype(colin_c)::value;
        // steady column-interior stages with T a multiple of 4: a lane's
        // columns are all owned or all halo, so the norm is accumulated
        // unconditionally and a halo lane's sums are dropped once, at the end
        // (no per-point selects)
        constexpr bool UNMASKED_NORM = STEADY && COLIN && (T % WV_CPT) == 0;
        if (wp == 0) {
            load_row(s + WV_PD);
            cp_async_wait_group<WV_PD>();   // row s complete (this lane's copies)
        }
        wave_barrier<NW>();                 // ... every lane's; last stage's hand-off row
#pragma unroll
        for (int j = LPW - 1; j >= 0; --j) {
            const int t = t0 + j + 1;        // level (1-based step within the launch)
            const int rho = s - 2 * t;
            C Cn[NC];
            if (j == 0) {
                if (wp == 0) {
#pragma unroll
                    for (int q = 0; q < NC; ++q) Cn[q] = ldu(s_u, WV_CPT * lane + q);
                } else {
                    const C* hr = sh[(wp - 1) * 2 + ((s - 1) & 1)];
#pragma unroll
                    for (int q = 0; q < NC; ++q) Cn[q] = hr[WV_CPT * lane + q];
                }
            } else {
#pragma unroll
                for (int q = 0; q < WV_CPT; ++q) Cn[q + 1] = O[j - 1][q];
                Cn[0] = shfl_up1(O[j - 1][WV_CPT - 1]);
                Cn[NC - 1] = shfl_dn1(O[j - 1][0]);
            }
            const bool valid = STEADY || (rho >= t && rho < NLOAD - t);
            if (valid) {
                const int gr = gr0 + rho;
                const bool rin = STEADY || (gr >= 0 && gr < side);   // steady rows are in the grid
                const bool rown = STEADY || (rho >= T && rho < T + L);
                int fslot = s_f - 2 * t;
                if (fslot < 0) fslot += SM::RF;
                C sum[WV_CPT];
#pragma unroll
                for (int q = 0; q < WV_CPT; ++q) sum[q] = mul(c[0], A[j][q]);
#pragma unroll
                for (int q = 0; q < WV_CPT; ++q) sum[q] = add(sum[q], mul(c[1], A[j][q + 1]));
#pragma unroll
                for (int q = 0; q < WV_CPT; ++q) sum[q] = add(sum[q], mul(c[2], A[j][q + 2]));
#pragma unroll
                for (int q = 0; q < WV_CPT; ++q) sum[q] = add(sum[q], mul(c[3], Bw[j][q]));
#pragma unroll
                for (int q = 0; q < WV_CPT; ++q) sum[q] = add(sum[q], mul(c[4], Bw[j][q + 1]));
#pragma unroll
                for (int q = 0; q < WV_CPT; ++q) sum[q] = add(sum[q], mul(c[5], Bw[j][q + 2]));
#pragma unroll
                for (int q = 0; q < WV_CPT; ++q) sum[q] = add(sum[q], mul(c[6], Cn[q]));
#pragma unroll
                for (int q = 0; q < WV_CPT; ++q) sum[q] = add(sum[q], mul(c[7], Cn[q + 1]));
#pragma unroll
                for (int q = 0; q < WV_CPT; ++q) sum[q] = add(sum[q], mul(c[8], Cn[q + 2]));
                C un[WV_CPT];
#pragma unroll
                for (int q = 0; q < WV_CPT; ++q) {
                    const C rs = sub(ldf(fslot, WV_CPT * lane + q), sum[q]);  // r = f - A u
                    const bool live = rin && (COLIN || colin[q]);
                    if (UNMASKED_NORM) acc[j] = sqacc(acc[j], rs);   // lane mask applied at the end
                    else if (rown && colown[q] && live) acc[j] = sqacc(acc[j], rs);
                    const C pv = JAC ? mul(sc, rs) : rs;                      // B^{-1} r
                    const C vn = rmul(w[j], pv);                              // v = 0 v + w p
                    un[q] = stored<S>(add(Bw[j][q + 1], vn));                 // u = u + v
                    if (t == T) {
                        if (rown && colown[q] && live) {
                            const size_t g = base + (size_t)gr * side + (gc0 + WV_CPT * lane + q);
                            a.u_out[g] = to_s<S>(un[q]);
                        }
                    } else {
                        un[q] = live ? un[q] : szero<C>();                     // Dirichlet
                        O[j][q] = un[q];
                    }
                }
                if (j == LPW - 1 && t < T) {
                    // the warp's top level feeds the next warp's first level
                    C* hw = sh[wp * 2 + (s & 1)];
#pragma unroll
                    for (int q = 0; q < WV_CPT; ++q) hw[1 + WV_CPT * lane + q] = un[q];
                }
            }
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                A[j][q] = Bw[j][q];
                Bw[j][q] = Cn[q];
            }
        }
        s_u = s_u + 1 == SM::RU ? 0 : s_u + 1;
        s_f = s_f + 1 == SM::RF ? 0 : s_f + 1;
    };
    // steady stages: every level's row valid (s in [3T, NLOAD + 1)), owned
    // (s < T + L + 2) and inside the grid (rows outside it only occur in the
    // first and last T rows of the first and last segments).
    typedef std::integral_constant<bool, true> Y;
    typedef std::integral_constant<bool, false> N;
    const bool colin_cta = gc0 >= 0 && gc0 + WV_W <= side;
    const int s1 = 3 * T;
    const int s2 = max(s1, min(NLOAD + 1, T + L + 2));
    int s = 0;
    for (; s < s1; ++s) stage(s, N(), N());
    if (colin_cta) {
        for (; s < s2; ++s) stage(s, Y(), Y());
    } else {
        for (; s < s2; ++s) stage(s, Y(), N());
    }
    for (; s < NS; ++s) stage(s, N(), N());
    if (wp == 0) cp_async_wait_all();
    if (colin_cta && (T % WV_CPT) == 0 && !(colown[0] && colown[WV_CPT - 1])) {
#pragma unroll
        for (int j = 0; j < LPW; ++j) acc[j] = 0.0;   // a halo lane: every column unowned
    }
}

template <int T>
struct WaveOcc {
    static constexpr int NW = wave_nw(T);
    static constexpr int REGS = NW > 1 ? RG_WV_REGS : RG_WV_REGS1;
    static constexpr int MINB = 65536 / (NW * 32 * REGS);
};

template <typename S, int T, bool JAC>
__global__ void __launch_bounds__(WaveOcc<T>::NW * 32) __maxnreg__(WaveOcc<T>::REGS)
wave_kernel(const __grid_constant__ WaveArgs<S> a) {
    constexpr int NW = WaveOcc<T>::NW;
    constexpr int LPW = T / NW;
    const int bl = blockIdx.y;
    const int b = a.b0 + bl;
    if (a.epi.st && a.epi.st[b].status != ST_ACTIVE) return;
    const int cta = blockIdx.x;
    const int strip = cta % a.nstrip, seg = cta / a.nstrip;
    double acc[LPW];
#pragma unroll
    for (int j = 0; j < LPW; ++j) acc[j] = 0.0;
    wave_body<S, T, NW, JAC>(a, b, bl, strip, seg, acc);
    if (a.epi.nslots > 0) {
        // slot t-1 holds step t's norm; warp w accumulated levels w*LPW+1 ..
        // Each warp reduces its own slots by shuffles, then the per-slot
        // warp sums go to the fused epilogue as thread 0's values.
        __shared__ double part[NW][LPW];
        const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
        for (int j = 0; j < LPW; ++j) {
            double v = acc[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
            if (lane == 0) part[wp][j] = v;
        }
        __syncthreads();
        double all[T];
#pragma unroll
        for (int t = 0; t < T; ++t) all[t] = (threadIdx.x == 0) ? part[t / LPW][t % LPW] : 0.0;
        epilogue<NW * 32, T>(a.epi, b, cta, gridDim.x, all, 0.0);
    }
}

template <typename S, int T, bool JAC>
cudaError_t launch_wave_t(const WaveArgs<S>& a, int nsys, cudaStream_t st) {
    auto kern = wave_kernel<S, T, JAC>;
    const size_t smem = WaveSmem<S, T>::bytes;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        // the whole shared-memory carveout: ~20 KB per one-warp CTA, and the
        // register-limited 9 CTAs per SM only fit in the largest carveout
        // (the default choice left 8 resident, so a 0.97-wave grid became 1.1)
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 (int)cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int nt = wave_ntiles(a.side, T, a.seg_rows, nullptr);
    kern<<<dim3(nt, nsys), dim3(WaveOcc<T>::NW * 32), smem, st>>>(a);
    return cudaGetLastError();
}

constexpr int WV_TMAX = 6;

// a.nstrip / a.seg_rows must be set by the caller (wave_ntiles).
template <typename S>
cudaError_t launch_wave(const WaveArgs<S>& a, int T, bool jac, int nsys, cudaStream_t st) {
#define RG_WV_CASE(TT) \
    case TT: return jac ? launch_wave_t<S, TT, true>(a, nsys, st) : launch_wave_t<S, TT, false>(a, nsys, st);
    switch (T) {
        RG_WV_CASE(1) RG_WV_CASE(2) RG_WV_CASE(3) RG_WV_CASE(4) RG_WV_CASE(5) RG_WV_CASE(6)
    }
#undef RG_WV_CASE
    return cudaErrorInvalidValue;
}

extern template cudaError_t launch_wave<double>(const WaveArgs<double>&, int, bool, int, cudaStream_t);
extern template cudaError_t launch_wave<float>(const WaveArgs<float>&, int, bool, int, cudaStream_t);

}  // namespace rg

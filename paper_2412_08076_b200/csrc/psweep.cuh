// psweep.cuh — free-running sweeps of small grids in ONE launch
// (multigrid.py:126-138 `_smooth` on the coarse V-cycle levels, and any
// other small rg_sweep of up to 16 x 1024 unknowns per system).
//
// On small grids a one-step launch is latency-bound (6.4 us per step at
// 31^2 .. 127^2 in the cfg5 V-cycle).  Here one thread-block cluster per
// system (up to 16 CTAs) runs all the steps with the stencil input resident
// in distributed shared memory (csweep_kernel below).  An earlier variant
// ping-ponged y through L2 with u and v updated in global memory; every
// cluster barrier invalidates L1, so each of its steps paid two L2 round
// trips (~2.7 us per step at 63^2 against ~1.3 us here).
#pragma once
#include <cooperative_groups.h>
#include <stdlib.h>
#include "step.cuh"

namespace rg {

template <typename S>
struct PsArgs {
    OpView<S> A;
    S* u;
    S* v;              // null for plain
    const S* f;
    const double* omega;
    const double* alpha;
    const double* atil;
    const CT<S>* scale;
    int precond;
    int m, k0, n_steps, B;
};

// ---- row-block variant: the stencil input in distributed shared memory ----
// For grids with at most 16 x 256 unknowns the L2 round trip of the y
// ping-pong dominates a psweep step (~2.7 us).  Here CTA c of the cluster
// owns rows [c R, c R + R) and keeps them, with one halo row above and below
// and a zero border, in two shared-memory y fields; every step each thread
// updates its point (u, v, f, the Jacobi scale and the operator row live in
// registers), writes y_{k+1} into the other field and pushes the CTA's
// boundary rows straight into the neighbours' halo rows (DSMEM) before the
// cluster barrier, as the cluster solver does.  Same arithmetic as
// step1_kernel / psweep_kernel, operation for operation.
constexpr int CS_NT = 256;        // operator row in registers (<= 16 x 256 unknowns)
constexpr int CS_NT_BIG = 1024;   // operator rows in shared memory (<= 16 x 1024)

// rows per CTA for a side x side grid on nc <= 16 CTAs of nt threads (0: does not fit)
inline int csweep_shape(int side, int nt, int* nc) {
    for (int c = 1; c <= 16; ++c) {
        const int R = (side + c - 1) / c;
        if (R * side <= nt && (c - 1) * R < side) { *nc = c; return R; }
    }
    *nc = 0;
    return 0;
}

// NT = 256: the operator row in registers (<= 16 x 256 unknowns); NT = 1024
// (<= 16 x 1024, e.g. 127^2): the rows of the CTA's points in shared memory
// (VAR9: 9 values per point), to stay within 64 registers per thread.
template <typename S, int KIND, int VAR, int NT>
__global__ void __launch_bounds__(NT) csweep_kernel(const __grid_constant__ PsArgs<S> a, int R) {
    constexpr bool CSM = NT > CS_NT;
    typedef CT<S> C;
    constexpr bool NAG = VAR >= V_NAG;
    constexpr bool HASV = VAR != V_PLAIN;
    namespace cgp = cooperative_groups;
    cgp::cluster_group cl = cgp::this_cluster();
    const int nc = cl.num_blocks();
    const int crank = (int)cl.block_rank();
    const int b = blockIdx.x / nc;
    const int side = a.A.side, W = side + 2;
    const size_t base = (size_t)b * a.A.P;
    const int row0 = crank * R;
    const int nrows = min(R, side - row0);
    const int npts = nrows * side;
    const int tid = threadIdx.x;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    (void)CSM;
    C* Yb[2] = {reinterpret_cast<C*>(smem_raw), reinterpret_cast<C*>(smem_raw) + (R + 2) * W};
    C* cfs = Yb[0] + 2 * (R + 2) * W;                        // CSM: [9][NT] operator rows
    for (int q = tid; q < 2 * (R + 2) * W; q += NT) Yb[0][q] = szero<C>();   // zero border

    constexpr int MAXW = 64;
    __shared__ double wsm[3][MAXW];
    const bool wstaged = a.n_steps <= MAXW;
    for (int t = tid; t < a.n_steps && t < MAXW; t += NT) {
        const int k = a.k0 + t;
        const int si = b * a.m + (k % a.m);
        wsm[0][t] = a.omega[si];
        wsm[1][t] = HASV ? a.alpha[si] : 0.0;
        wsm[2][t] = NAG ? a.atil[b * a.m + ((k + 1) % a.m)] : 0.0;
    }

    const bool mine = tid < npts;
    const int lr = tid / side, col = tid - (tid / side) * side;
    const int i = row0 + lr;                                  // grid row
    const size_t g = base + (size_t)i * side + col;
    const int pix = (lr + 1) * W + col + 1;
    const int bc = a.A.shared ? 0 : b;
    C cf[9], dg = szero<C>();
#pragma unroll
    for (int d = 0; d < 9; ++d) cf[d] = szero<C>();
    C ur = szero<C>(), vr = szero<C>(), fr = szero<C>(), sr = szero<C>();
    if (mine) {
        const size_t gi = (size_t)i * side + col;
        if (KIND == K_CONST9) {
#pragma unroll
            for (int d = 0; d < 9; ++d) cf[d] = a.A.stencil[(size_t)bc * 9 + d];
        } else if (KIND == K_DIAG5) {
#pragma unroll
            for (int d = 0; d < 4; ++d) cf[d] = a.A.stencil[(size_t)bc * 4 + d];
            dg = a.A.diag[(size_t)bc * a.A.P + gi];
        } else if (CSM) {
            for (int d = 0; d < 9; ++d) cfs[d * NT + tid] = a.A.stencil[((size_t)bc * 9 + d) * a.A.P + gi];
        } else {
#pragma unroll
            for (int d = 0; d < 9; ++d) cf[d] = a.A.stencil[((size_t)bc * 9 + d) * a.A.P + gi];
        }
        ur = to_c(a.u[g]);
        if (HASV) vr = to_c(a.v[g]);
        fr = to_c(a.f[g]);
        if (a.precond == P_JSCALAR) sr = a.scale[b];
        else if (a.precond == P_JFIELD) sr = a.scale[g];
    }
    // push this point's y value into Yn (own field) and, for boundary rows,
    // into the neighbours' halo rows of Yn
    auto publish = [&](C* Yn, C x) {
        Yn[pix] = x;
        if (lr == 0 && crank > 0) cl.map_shared_rank(Yn, crank - 1)[(R + 1) * W + col + 1] = x;
        if (lr == nrows - 1 && crank < nc - 1) cl.map_shared_rank(Yn, crank + 1)[col + 1] = x;
    };
    __syncthreads();                                          // zero border before any push
    cl.sync();                                                // every CTA zeroed
    if (mine) {                                               // y_0 = u (+ at v, :119)
        C x = ur;
        if (NAG) x = add(x, rmul(a.atil[b * a.m + (a.k0 % a.m)], vr));
        publish(Yb[0], to_c(to_s<S>(x)));
    }
    cl.sync();
    for (int t = 0; t < a.n_steps; ++t) {
        const int k = a.k0 + t;
        const C* Y = Yb[t & 1];
        C* Yn = Yb[(t + 1) & 1];
        if (mine) {
            const int q = pix;
            C s;
            if (KIND == K_DIAG5) {                            // apply_op<DIAG5> order
                s = mul(cf[0], Y[q - W]);
                s = add(s, mul(cf[1], Y[q - 1]));
                s = add(s, mul(dg, Y[q]));
                s = add(s, mul(cf[2], Y[q + 1]));
                s = add(s, mul(cf[3], Y[q + W]));
            } else {                                          // CSR column order
                auto cd = [&](int d) -> C {
                    return (CSM && KIND == K_VAR9) ? cfs[d * NT + tid] : cf[d];
                };
                s = mul(cd(0), Y[q - W - 1]);
                s = add(s, mul(cd(1), Y[q - W]));
                s = add(s, mul(cd(2), Y[q - W + 1]));
                s = add(s, mul(cd(3), Y[q - 1]));
                s = add(s, mul(cd(4), Y[q]));
                s = add(s, mul(cd(5), Y[q + 1]));
                s = add(s, mul(cd(6), Y[q + W - 1]));
                s = add(s, mul(cd(7), Y[q + W]));
                s = add(s, mul(cd(8), Y[q + W + 1]));
            }
            const C r = sub(fr, s);
            const C p = a.precond != P_NONE ? mul(sr, r) : r;   // precond.py:125-129
            const int si = b * a.m + (k % a.m);
            const double w = wstaged ? wsm[0][t] : a.omega[si];
            C vn;
            if (VAR == V_PLAIN) vn = rmul(w, p);
            else vn = add(rmul(wstaged ? wsm[1][t] : a.alpha[si], vr), rmul(w, p));
            const S vs = to_s<S>(vn);
            const S us = to_s<S>(add(ur, vn));
            ur = to_c(us);
            vr = to_c(vs);
            C x = ur;
            if (NAG) x = add(x, rmul(wstaged ? wsm[2][t] : a.atil[b * a.m + ((k + 1) % a.m)], vr));
            publish(Yn, to_c(to_s<S>(x)));
        }
        cl.sync();   // y_{k+1} and its halos complete; the neighbours read Y one barrier ago
    }
    if (mine) {
        a.u[g] = to_s<S>(ur);
        if (HASV) a.v[g] = to_s<S>(vr);
    }
    cl.sync();   // no CTA exits while a neighbour may still push into it
}

template <typename S, int KIND, int VAR, int NT>
cudaError_t launch_csweep_t(const PsArgs<S>& a, int nc, int R, cudaStream_t st) {
    auto kern = csweep_kernel<S, KIND, VAR, NT>;
    const size_t smem = 2 * (size_t)(R + 2) * (a.A.side + 2) * sizeof(CT<S>) +
                        (NT > CS_NT && KIND == K_VAR9 ? (size_t)9 * NT * sizeof(CT<S>) : 0);
    static bool attr_set = false;
    static size_t smem_set = 0;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    if (smem > smem_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        smem_set = smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.B * nc);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = nc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a, R);
}

template <typename S, int KIND, int VAR>
cudaError_t launch_psweep_t(const PsArgs<S>& a, cudaStream_t st) {
    int nc = 0;
    int R = csweep_shape(a.A.side, CS_NT, &nc);
    if (nc > 0) return launch_csweep_t<S, KIND, VAR, CS_NT>(a, nc, R, st);
    R = csweep_shape(a.A.side, CS_NT_BIG, &nc);
    if (nc > 0) return launch_csweep_t<S, KIND, VAR, CS_NT_BIG>(a, nc, R, st);
    return cudaErrorInvalidValue;   // (the caller checks csweep_shape first)
}

template <typename S, int KIND>
cudaError_t launch_psweep_k(const PsArgs<S>& a, int variant, cudaStream_t st) {
    switch (variant) {
        case V_PLAIN: return launch_psweep_t<S, KIND, V_PLAIN>(a, st);
        case V_MOM: return launch_psweep_t<S, KIND, V_MOM>(a, st);
        default: return launch_psweep_t<S, KIND, V_NAG>(a, st);
    }
}

template <typename S>
cudaError_t launch_psweep(const PsArgs<S>& a, int kind, int variant, cudaStream_t st) {
    switch (kind) {
        case K_CONST9: return launch_psweep_k<S, K_CONST9>(a, variant, st);
        case K_DIAG5: return launch_psweep_k<S, K_DIAG5>(a, variant, st);
        default: return launch_psweep_k<S, K_VAR9>(a, variant, st);
    }
}

}  // namespace rg

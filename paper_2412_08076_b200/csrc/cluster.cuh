// cluster.cuh — the whole solve_stationary (richardson.py:77-141) in ONE
// launch, one thread-block CLUSTER per system, for small grids (<= 4096
// unknowns; cfg1 63^2 runs on 8 CTAs).  Larger grids (cfg2 255^2 measured
// 160 ms here vs 86 ms tiled) go through the temporally blocked sweep.
//
// CTA c of a cluster owns rows [c*R, c*R+R) of the system and keeps them,
// plus one halo row above and below, in a zero-bordered shared-memory field
// (u; for NAG also the look-ahead y, ping-ponged).  f, r, v of the CTA's own
// points live in registers for the entire solve.  Per inner step:
//
//   update own points -> cluster.sync -> copy the two halo rows from the
//   neighbouring CTAs' shared memory (DSMEM) -> residual of own points ->
//   CTA partial of ||r||^2 written into every CTA's `parts` slot (DSMEM)
//   -> every thread sums the partials in the same order and takes the same
//   convergence / divergence / max_outer decision.
// plain/mom pipeline the decision one step behind (one cluster barrier per
// step, ping-ponged u) and push their boundary rows into the neighbours'
// halo rows before the barrier; nag uses two barriers.
//
// Nothing touches HBM between the initial load and the final store, and
// there is no launch per step: the solve is bound by FP64 issue and the
// two cluster barriers per step.  Arithmetic is the reference's (no FMA):
// iterates are bitwise the oracle's.
#pragma once
#include <cooperative_groups.h>

#include "reduce.cuh"

namespace rg {
namespace cg = cooperative_groups;

constexpr int CL_NT = 256;
constexpr int CL_MAXC = 16;     // non-portable cluster size limit
constexpr int CL_MAXM = 16;     // sweep length of the batched-decision loop
constexpr int CL_MAXW = 64;     // schedules up to this length are staged in shared memory

template <typename S>
struct ClusterArgs {
    const CT<S>* coef;   // [B][9] (or one set when shared)
    const CT<S>* scale;  // [B] Jacobi scale or null
    S* u;                // [B][P] initial guess in, answer out
    const S* f;          // [B][P]
    const double* omega;
    const double* alpha;
    const double* atil;
    int side, P, m;
    int shared;
    int nc;              // CTAs per cluster (= per system)
    int rows;            // rows per CTA (the last CTA may own fewer)
    SolveCfg cfg;
    SysState* st;
    double* trace;
    int trace_stride;
};

template <typename S, int VAR, bool JAC, int PPT>
__global__ void __launch_bounds__(CL_NT, 1) cluster_solve_kernel(ClusterArgs<S> a) {
    typedef CT<S> C;
    constexpr bool NAG = VAR >= V_NAG;
    constexpr bool HASV = VAR != V_PLAIN;
    cg::cluster_group cl = cg::this_cluster();
    const int nc = a.nc;
    const int crank = (int)cl.block_rank();
    const int b = blockIdx.x / nc;
    const int s = a.side, W = s + 2, m = a.m;
    const int R = a.rows;
    const int row0 = crank * R;
    const int nrows = min(R, s - row0);          // >= 1 by construction
    const int npts = nrows * s;
    const int tid = threadIdx.x;
    const size_t base = (size_t)b * a.P;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* U = reinterpret_cast<C*>(smem_raw);                   // [(R+2) * W]
    C* Yb[2] = {U + (R + 2) * W, U + 2 * (R + 2) * W};       // NAG ping-pong
    __shared__ double parts[CL_MAXC];
    __shared__ double red[CL_NT / 32];

    C c[9];
    const int cb = a.shared ? 0 : b;
#pragma unroll
    for (int d = 0; d < 9; ++d) c[d] = a.coef[(size_t)cb * 9 + d];
    const C sc = JAC ? a.scale[b] : szero<C>();

    const int fields = NAG ? 3 : 2;    // u (+ y ping-pong) | u ping-pong
    for (int q = tid; q < fields * (R + 2) * W; q += CL_NT) U[q] = szero<C>();
    // the schedule in shared memory: every cluster barrier invalidates L1
    // (CCTL.IVALL), so a global weight load after it would cost an L2 round
    // trip on every inner step's critical path
    __shared__ double wsm[3][CL_MAXW];
    const bool wstaged = m <= CL_MAXW;
    for (int q = tid; q < m && q < CL_MAXW; q += CL_NT) {
        wsm[0][q] = a.omega[b * m + q];
        wsm[1][q] = HASV ? a.alpha[b * m + q] : 0.0;
        wsm[2][q] = NAG ? a.atil[b * m + q] : 0.0;
    }
    auto W_ = [&](int i) { return wstaged ? wsm[0][i] : a.omega[b * m + i]; };
    auto AL_ = [&](int i) { return HASV ? (wstaged ? wsm[1][i] : a.alpha[b * m + i]) : 0.0; };
    auto AT_ = [&](int i) { return wstaged ? wsm[2][i] : a.atil[b * m + i]; };
    __syncthreads();

    C fr[PPT], rr[PPT], vr[PPT];
    int pix[PPT];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
        const int p = tid + j * CL_NT;
        const int lr = p / s, col = p - (p / s) * s;
        pix[j] = (lr + 1) * W + (col + 1);
        const bool mine = p < npts;
        const size_t g = base + (size_t)(row0 + lr) * s + col;
        fr[j] = mine ? to_c(a.f[g]) : szero<C>();
        vr[j] = szero<C>();                                    // v = 0 at entry (:95)
        rr[j] = szero<C>();
        if (mine) U[pix[j]] = to_c(a.u[g]);
    }

    // halo rows of field X from the neighbouring CTAs (DSMEM reads)
    auto halo = [&](C* X) {
        if (crank > 0) {
            const C* up = cl.map_shared_rank(X, crank - 1);
            for (int q = tid; q < s; q += CL_NT) X[q + 1] = up[R * W + q + 1];       // its last row
        }
        if (crank < nc - 1) {
            const C* dn = cl.map_shared_rank(X, crank + 1);
            for (int q = tid; q < s; q += CL_NT) X[(nrows + 1) * W + q + 1] = dn[W + q + 1];
        }
    };
    auto stencil = [&](const C* X, int q) {                     // CSR order, no FMA
        C t = mul(c[0], X[q - W - 1]);
        t = add(t, mul(c[1], X[q - W]));
        t = add(t, mul(c[2], X[q - W + 1]));
        t = add(t, mul(c[3], X[q - 1]));
        t = add(t, mul(c[4], X[q]));
        t = add(t, mul(c[5], X[q + 1]));
        t = add(t, mul(c[6], X[q + W - 1]));
        t = add(t, mul(c[7], X[q + W]));
        t = add(t, mul(c[8], X[q + W + 1]));
        return t;
    };
    // cluster-wide sum, identical bits in every thread of every CTA
    auto cluster_sum = [&](double v) {
        const int lane = tid & 31, w = tid >> 5;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) red[w] = v;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < CL_NT / 32; ++q) t += red[q];
            for (int r = 0; r < nc; ++r) *cl.map_shared_rank(&parts[crank], r) = t;
        }
        cl.sync();
        double tot = 0.0;
        for (int r = 0; r < nc; ++r) tot += parts[r];
        return tot;
    };
    auto residual_of = [&](const C* X) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
            if (tid + j * CL_NT < npts) {
                rr[j] = sub(fr[j], stencil(X, pix[j]));
                acc = sqacc(acc, rr[j]);
            }
        }
        return acc;
    };
    auto residual_u = [&]() { return residual_of(U); };
    C* Uout = U;                          // field holding the answer at the end

    const SolveCfg cf = a.cfg;
    double* trace = a.trace + (size_t)b * a.trace_stride;
    int status = ST_ACTIVE, outer = 0, inner = 0;
    double fnorm, trace0, rel, bad_rel = 0.0;
    cl.sync();                                                  // own rows loaded everywhere
    halo(U);
    __syncthreads();
    {
        double ff = 0.0;
#pragma unroll
        for (int j = 0; j < PPT; ++j) ff = sqacc(ff, fr[j]);
        const double r2 = cluster_sum(residual_u());
        cl.sync();                                              // parts reused
        const double f2 = cluster_sum(ff);
        fnorm = sqrt(f2);
        if (fnorm == 0.0) {                                     // :97-100
            status = ST_CONVERGED; rel = 0.0; trace0 = 0.0;
        } else {
            rel = sqrt(r2) / fnorm;
            trace0 = rel;
            if (rel <= cf.tol) status = ST_CONVERGED;
            else if (cf.max_outer <= 0) status = ST_MAXED;
        }
        if (tid == 0 && crank == 0) trace[0] = trace0;
    }
    const double div_thr = cf.div_factor * fmax(trace0, 1.0);
    int k = 0;
    // decision for the residual of iterate j (richardson.py:124-136); identical
    // in every thread because every thread sums the same partials in order
    auto decide = [&](int j, double r2) {
        rel = sqrt(r2) / fnorm;
        inner = j;
        const bool boundary = (j % m) == 0;
        if (!isfinite(rel) || rel > div_thr) {                  // :126-129
            status = ST_DIVERGED; bad_rel = rel;
            return;
        }
        if (boundary) {
            outer = j / m;
            if (tid == 0 && crank == 0) trace[outer] = rel;
        }
        if ((cf.check_inner || boundary) && rel <= cf.tol) {
            status = ST_CONVERGED;
            if (!boundary) { outer = j / m + 1; if (tid == 0 && crank == 0) trace[outer] = rel; }
        } else if (boundary && outer >= cf.max_outer) {
            status = ST_MAXED;
        }
    };
    if (!NAG && status == ST_ACTIVE && !cf.check_inner && m <= CL_MAXM) {
        // plain / mom, check = "outer": the decision logic only needs the
        // sweep-boundary norm for convergence / max_outer, and the per-step
        // norms for the divergence guard, which it can examine after the
        // sweep in step order (the first offending inner index is still the
        // one reported; a diverged solve returns no iterate).  So each inner
        // step costs one cluster barrier (halo exchange) and a shared-memory
        // store of the thread's |r|^2; the m per-step norms of a sweep are
        // reduced together, published with one more barrier and decided in
        // order.  u ping-pongs (step j reads Ub[j&1], writes Ub[(j+1)&1]);
        // a boundary stop returns the current iterate.
        __shared__ double accs[CL_MAXM][CL_NT];            // this thread's |r_j|^2
        __shared__ double redm[CL_MAXM][CL_NT / 32];
        __shared__ double partsm[2][CL_MAXM][CL_MAXC];     // by sweep parity
        __shared__ double tots[CL_MAXM];
        // tot <= fast_lim  =>  sqrt(tot) / fnorm <= div_thr / 2 (with margin;
        // an overflowing bound is +inf, still conservative)
        const double fast_lim = 0.25 * (div_thr * fnorm) * (div_thr * fnorm);
        C* Ub[2] = {U, U + (R + 2) * W};
        for (int sweep = 0; status == ST_ACTIVE; ++sweep) {
            for (int i = 0; i < m; ++i) {                 // steps k .. k+m-1 (i = k % m)
                const double w = W_(i);
                const double al = AL_(i);
                const C* Uo = Ub[k & 1];
                C* Un = Ub[(k + 1) & 1];
                C* up_nb = crank > 0 ? cl.map_shared_rank(Un, crank - 1) : nullptr;
                C* dn_nb = crank < nc - 1 ? cl.map_shared_rank(Un, crank + 1) : nullptr;
#pragma unroll
                for (int j = 0; j < PPT; ++j) {                 // (:120-121)
                    const int pp = tid + j * CL_NT;
                    if (pp < npts) {
                        const C p = JAC ? mul(sc, rr[j]) : rr[j];
                        C vn = (VAR == V_PLAIN) ? rmul(w, p) : add(rmul(al, vr[j]), rmul(w, p));
                        const C un = stored<S>(add(Uo[pix[j]], vn));
                        Un[pix[j]] = un;
                        vr[j] = stored<S>(vn);
                        // neighbours' halo rows of Un, visible after the barrier;
                        // they last read them one barrier earlier (ping-pong)
                        if (pp < s && up_nb) up_nb[(R + 1) * W + pix[j] - W] = un;
                        if (pp >= npts - s && dn_nb) dn_nb[pix[j] - nrows * W] = un;
                    }
                }
                cl.sync();
                accs[i][tid] = residual_of(Un);          // r_{k+1}
                ++k;
            }
            // the sweep's m norms: warp sums, CTA partials to every CTA, decide
            const int lane = tid & 31, wq = tid >> 5;
            for (int i = 0; i < m; ++i) {
                double v = accs[i][tid];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
                if (lane == 0) redm[i][wq] = v;
            }
            __syncthreads();
            double (*pm)[CL_MAXC] = partsm[sweep & 1];
            for (int t = tid; t < m * nc; t += CL_NT) {       // (step, destination CTA)
                const int i = t / nc, r = t - (t / nc) * nc;
                double sum = 0.0;
#pragma unroll
                for (int q = 0; q < CL_NT / 32; ++q) sum += redm[i][q];
                *cl.map_shared_rank(&pm[i][crank], r) = sum;
            }
            cl.sync();
            // the m cluster totals in parallel (thread i: pairwise tree over
            // the nc partials, the same bits in every CTA) ...
            if (tid < m) {
                double v[CL_MAXC];
#pragma unroll
                for (int r = 0; r < CL_MAXC; ++r) v[r] = r < nc ? pm[tid][r] : 0.0;
#pragma unroll
                for (int h = CL_MAXC / 2; h > 0; h >>= 1)
#pragma unroll
                    for (int r = 0; r < h; ++r) v[r] = v[r] + v[r + h];
                tots[tid] = v[0];
            }
            __syncthreads();
            // ... then the decisions in step order.  A non-boundary step whose
            // total is finite and below a quarter of the squared divergence
            // threshold can neither raise nor stop: its sqrt / division are
            // skipped (decide() only runs where it can change the state).
            const int j0 = k - m + 1;                         // first inner index of the sweep
            for (int i = 0; i < m && status == ST_ACTIVE; ++i) {
                const double tot = tots[i];
                if (i < m - 1 && tot <= fast_lim && isfinite(tot)) continue;
                decide(j0 + i, tot);
            }
            if (status != ST_ACTIVE) {
                k = inner;                                    // the decided index
                Uout = Ub[k & 1];
            }
        }
        cl.sync();                        // last remote writes to partsm complete
    } else if (!NAG && status == ST_ACTIVE) {
        // plain / mom: ONE cluster barrier per inner step.  The u field is
        // ping-ponged (iteration j reads Ub[j&1], writes Ub[(j+1)&1]), so a
        // neighbour may start its next update while this CTA still copies
        // halo rows.  Iteration j computes u_{j+1}, exchanges its halos,
        // computes r_{j+1} and publishes its partial into parts2[(j+1)&1];
        // it then decides for r_j from the partials published one iteration
        // earlier.  A stop at j leaves the answer u_j in Ub[j&1].
        __shared__ double parts2[2][CL_MAXC];
        C* Ub[2] = {U, U + (R + 2) * W};
        bool have_prev = false;           // partials of r_k available (k >= 1)
        while (true) {
            const int i = k % m;
            const double w = W_(i);
            const double al = AL_(i);
            const C* Uo = Ub[k & 1];
            C* Un = Ub[(k + 1) & 1];
            C* up_nb = crank > 0 ? cl.map_shared_rank(Un, crank - 1) : nullptr;
            C* dn_nb = crank < nc - 1 ? cl.map_shared_rank(Un, crank + 1) : nullptr;
#pragma unroll
            for (int j = 0; j < PPT; ++j) {                     // (:120-121)
                const int pp = tid + j * CL_NT;
                if (pp < npts) {
                    const C p = JAC ? mul(sc, rr[j]) : rr[j];
                    C vn = (VAR == V_PLAIN) ? rmul(w, p) : add(rmul(al, vr[j]), rmul(w, p));
                    const C un = stored<S>(add(Uo[pix[j]], vn));
                    Un[pix[j]] = un;
                    vr[j] = stored<S>(vn);
                    // push boundary rows straight into the neighbours' halo
                    // rows of Un (DSMEM stores, visible after the barrier):
                    // no halo read after it.  Safe: the neighbours last read
                    // those halo rows one barrier earlier (ping-pong).
                    if (pp < s && up_nb) up_nb[(R + 1) * W + pix[j] - W] = un;
                    if (pp >= npts - s && dn_nb) dn_nb[pix[j] - nrows * W] = un;
                }
            }
            cl.sync();
            {   // partial of r_{k+1} -> parts2[(k+1)&1] in every CTA
                double v = residual_of(Un);
                const int lane = tid & 31, wq = tid >> 5;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
                if (lane == 0) red[wq] = v;
                __syncthreads();
                if (tid < nc) {           // thread r publishes to CTA r (parallel DSMEM stores)
                    double t = 0.0;
#pragma unroll
                    for (int q = 0; q < CL_NT / 32; ++q) t += red[q];
                    *cl.map_shared_rank(&parts2[(k + 1) & 1][crank], tid) = t;
                }
            }
            if (have_prev) {              // decide for r_k (published last iteration)
                double tot = 0.0;
                for (int r = 0; r < nc; ++r) tot += parts2[k & 1][r];
                decide(k, tot);
                if (status != ST_ACTIVE) {
                    Uout = Ub[k & 1];
                    break;
                }
            }
            have_prev = true;
            ++k;
        }
        cl.sync();                        // last remote writes to parts2 complete
    }
    while (NAG && status == ST_ACTIVE) {
        const int i = k % m;
        const double w = W_(i);
        const double al = AL_(i);
        if (NAG) {
            C* Y = Yb[k & 1];
            const double at = AT_(i);
#pragma unroll
            for (int j = 0; j < PPT; ++j)
                if (tid + j * CL_NT < npts) Y[pix[j]] = add(U[pix[j]], rmul(at, vr[j]));   // (:119)
            cl.sync();
            halo(Y);
            __syncthreads();
#pragma unroll
            for (int j = 0; j < PPT; ++j)
                if (tid + j * CL_NT < npts) rr[j] = sub(fr[j], stencil(Y, pix[j]));
        }
#pragma unroll
        for (int j = 0; j < PPT; ++j) {                         // (:120-121)
            if (tid + j * CL_NT < npts) {
                const C p = JAC ? mul(sc, rr[j]) : rr[j];
                C vn = (VAR == V_PLAIN) ? rmul(w, p) : add(rmul(al, vr[j]), rmul(w, p));
                U[pix[j]] = stored<S>(add(U[pix[j]], vn));
                vr[j] = stored<S>(vn);
            }
        }
        ++k;
        const bool test = !NAG || cf.check_inner || (k % m) == 0;   // (:123)
        if (test) {
            cl.sync();                                          // updates visible
            halo(U);
            __syncthreads();
            decide(k, cluster_sum(residual_u()));
        }
    }
    if (tid == 0 && crank == 0) {
        SysState& st = a.st[b];
        st.fnorm = fnorm; st.trace0 = trace0; st.rel = rel; st.bad_rel = bad_rel;
        st.status = status; st.outer = outer; st.inner = inner; st.ans_buf = 0; st.last_j = k;
    }
    if (status != ST_DIVERGED) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
            const int p = tid + j * CL_NT;
            if (p < npts) {
                const int lr = p / s, col = p - (p / s) * s;
                a.u[base + (size_t)(row0 + lr) * s + col] = to_s<S>(Uout[pix[j]]);
            }
        }
    }
    cl.sync();   // no CTA may exit while others still read its shared memory
}

// Cluster shape for a side x side grid: nc CTAs (power of two <= 16), R rows
// each, at most PPT * CL_NT points per CTA; nc = 0 if it does not fit.
inline void cluster_shape(int side, int* nc, int* rows, int* ppt) {
    const long long P = (long long)side * side;
    int c = 1;
    if (P > 4096) { *nc = 0; return; }   // larger grids: the tiled blocked sweep is faster
    // ~1+ point per thread: per-step time is the serial work per thread
    // (cfg1 63^2: 16 CTAs 2.65 ms, 8 CTAs 3.03 ms, 4 CTAs 3.42 ms)
    long long per = 256;
    if (const char* ev = getenv("RG_CL_POINTS")) per = atoll(ev);   // tuning override
    while (c < CL_MAXC && P > (long long)c * per) c *= 2;
    while (c > 1 && (side + c - 1) / c < 2) c /= 2;             // >= 2 rows per CTA
    const int R = (side + c - 1) / c;
    if ((long long)R * side > 16LL * CL_NT || (c - 1) * R >= side) { *nc = 0; return; }
    *nc = c;
    *rows = R;
    const int need = (R * side + CL_NT - 1) / CL_NT;   // points per thread
    *ppt = need <= 1 ? 1 : (need <= 4 ? 4 : 16);
}

template <typename S>
inline size_t cluster_smem_bytes(int side, int rows, int variant) {
    return (size_t)(rows + 2) * (side + 2) * sizeof(CT<S>) * (variant >= V_NAG ? 3 : 2);
}

template <typename S, int VAR, bool JAC, int PPT>
cudaError_t launch_cluster_k(const ClusterArgs<S>& a, int B, size_t smem, cudaStream_t st) {
    auto kern = cluster_solve_kernel<S, VAR, JAC, PPT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (a.nc > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(B * a.nc, 1, 1);
    cfg.blockDim = dim3(CL_NT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.nc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

template <typename S>
cudaError_t launch_cluster(const ClusterArgs<S>& a, int variant, bool jac, int ppt, int B,
                           cudaStream_t st) {
    const size_t smem = cluster_smem_bytes<S>(a.side, a.rows, variant);
#define RG_CL(V, J, PP) return launch_cluster_k<S, V, J, PP>(a, B, smem, st)
    if (ppt == 1) {
        if (variant == V_PLAIN) { if (jac) RG_CL(V_PLAIN, true, 1); RG_CL(V_PLAIN, false, 1); }
        if (variant == V_MOM) { if (jac) RG_CL(V_MOM, true, 1); RG_CL(V_MOM, false, 1); }
        if (jac) RG_CL(V_NAG, true, 1);
        RG_CL(V_NAG, false, 1);
    }
    if (ppt == 4) {
        if (variant == V_PLAIN) { if (jac) RG_CL(V_PLAIN, true, 4); RG_CL(V_PLAIN, false, 4); }
        if (variant == V_MOM) { if (jac) RG_CL(V_MOM, true, 4); RG_CL(V_MOM, false, 4); }
        if (jac) RG_CL(V_NAG, true, 4);
        RG_CL(V_NAG, false, 4);
    }
    if (variant == V_PLAIN) { if (jac) RG_CL(V_PLAIN, true, 16); RG_CL(V_PLAIN, false, 16); }
    if (variant == V_MOM) { if (jac) RG_CL(V_MOM, true, 16); RG_CL(V_MOM, false, 16); }
    if (jac) RG_CL(V_NAG, true, 16);
    RG_CL(V_NAG, false, 16);
#undef RG_CL
}

}  // namespace rg

// reduce.cuh — deterministic fused residual-norm reduction and the device
// side of solve_stationary's convergence / divergence bookkeeping.
//
// Every launch that needs ||r|| writes one partial per CTA (fixed thread
// order inside the CTA), then the last CTA of each system (atomic ticket)
// sums the partials in a fixed strided order and applies the decision logic
// of richardson.py:105-136.  The result does not depend on which CTA
// finishes last, so runs are bitwise reproducible.  It is not bitwise equal
// to OpenBLAS ddot (np.linalg.norm); the difference is ~1e-16 relative.
#pragma once
#include "common.cuh"

namespace rg {

constexpr int NSLOT = 10;  // norm slots per launch: up to 8 inner steps + ||f||

// Sum `v` over the CTA; the result is valid in thread 0.  Fixed shuffle tree,
// then warps in index order.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (tid == 0) {
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) s += red[w];
    }
    return s;
}

struct EpiArgs {
    SysState* st;        // [B]
    double* trace;       // [B][trace_stride]
    int trace_stride;
    double* partials;    // [B][NSLOT][ncta_cap]
    int ncta_cap;
    SolveCfg cfg;
    int j0;              // global inner index of slot 0
    int nslots;          // residual-norm slots this launch produces
    int with_f;          // slot NSLOT-1 carries ||f||^2 (solver begin)
    int buf;             // ping-pong index of the launch's input iterate
    // stateless mode (st == null; rg_sweep_norm): the totals of the nslots
    // slots go to norm_out[b][nslots], tickets come from counters[b]
    int* counters = nullptr;
    double* norm_out = nullptr;
};

// richardson.py:96-136 for the norms j0 .. j0+n-1 (thread 0 of the last CTA).
__device__ inline void finalize(SysState& s, double* trace, const SolveCfg& c,
                                int j0, int n, const double* tot, int with_f,
                                double ftot, int buf) {
    if (s.status != ST_ACTIVE) return;
    if (with_f) {
        s.fnorm = sqrt(ftot);
        s.last_j = -1;
        if (s.fnorm == 0.0) {  // :97-100
            s.status = ST_CONVERGED; s.rel = 0.0; s.trace0 = 0.0; trace[0] = 0.0;
            s.outer = 0; s.inner = 0; s.ans_buf = buf; s.last_j = 0;
            return;
        }
    }
    for (int q = 0; q < n; ++q) {
        const int j = j0 + q;
        if (j <= s.last_j) continue;          // already decided by a flush
        s.last_j = j;
        const double rel = sqrt(tot[q]) / s.fnorm;
        if (j == 0) {                          // :105-110
            s.trace0 = rel; trace[0] = rel; s.rel = rel; s.outer = 0; s.inner = 0;
            s.ans_buf = buf;
            if (rel <= c.tol) { s.status = ST_CONVERGED; return; }
            if (c.max_outer <= 0) { s.status = ST_MAXED; return; }
            continue;
        }
        s.rel = rel;
        s.inner = j;
        if (!isfinite(rel) || rel > c.div_factor * fmax(s.trace0, 1.0)) {  // :126-129
            s.status = ST_DIVERGED; s.bad_rel = rel;
            return;
        }
        const bool boundary = (j % c.m) == 0;
        if (boundary) { s.outer = j / c.m; trace[s.outer] = rel; }          // :133-134
        if ((c.check_inner || boundary) && rel <= c.tol) {                  // :130-136
            s.status = ST_CONVERGED; s.ans_buf = buf;
            if (!boundary) { s.outer = j / c.m + 1; trace[s.outer] = rel; }
            return;
        }
        if (boundary && s.outer >= c.max_outer) {                           // :111
            s.status = ST_MAXED; s.ans_buf = buf;
            return;
        }
    }
}

// Called by every thread of every CTA of system b that computed norms.
// acc[q] = this thread's sum of |r|^2 for slot q; facc = sum of |f|^2.
template <int NT, int MAXS>
__device__ void epilogue(const EpiArgs& e, int b, int cta, int ncta,
                         const double (&acc)[MAXS], double facc) {
    __shared__ double red[NT / 32];
    __shared__ int is_last;
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    double* part = e.partials + (size_t)b * NSLOT * e.ncta_cap;
#pragma unroll
    for (int q = 0; q < MAXS; ++q) {
        if (q < e.nslots) {
            const double s = block_sum<NT>(acc[q], red);
            if (tid == 0) part[q * e.ncta_cap + cta] = s;
        }
    }
    if (e.with_f) {
        const double s = block_sum<NT>(facc, red);
        if (tid == 0) part[(NSLOT - 1) * e.ncta_cap + cta] = s;
    }
    // only thread 0 wrote partials: it alone fences before taking a ticket
    if (tid == 0) {
        __threadfence();
        const int t = atomicAdd(e.st ? &e.st[b].counter : &e.counters[b], 1);
        is_last = (t == ncta - 1);
        if (is_last) __threadfence();
    }
    __syncthreads();
    if (!is_last) return;
    __shared__ double tot[NSLOT];
    for (int q = 0; q < NSLOT; ++q) {
        const bool want = (q < e.nslots) || (q == NSLOT - 1 && e.with_f);
        if (!want) continue;
        double local = 0.0;
        for (int c = tid; c < ncta; c += NT) local += __ldcg(&part[q * e.ncta_cap + c]);
        const double s = block_sum<NT>(local, red);
        if (tid == 0) tot[q] = s;
    }
    if (tid == 0) {
        if (e.st) {
            finalize(e.st[b], e.trace + (size_t)b * e.trace_stride, e.cfg, e.j0, e.nslots,
                     tot, e.with_f, tot[NSLOT - 1], e.buf);
            e.st[b].counter = 0;
        } else {
            for (int q = 0; q < e.nslots; ++q) e.norm_out[(size_t)b * e.nslots + q] = tot[q];
            e.counters[b] = 0;
        }
        __threadfence();
    }
}

// Plain two-pass reduction (rg_residual): one partial per CTA ...
template <int NT>
__device__ void write_partial(double* part, int cta, double acc) {
    __shared__ double red[NT / 32];
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const double s = block_sum<NT>(acc, red);
    if (tid == 0) part[cta] = s;
}

// ... then one CTA per system sums them in a fixed order.
template <int NT>
__global__ void __launch_bounds__(NT) sum_partials_kernel(const double* part, int ncta,
                                                          double* out) {
    __shared__ double red[NT / 32];
    const int b = blockIdx.x;
    double local = 0.0;
    for (int c = threadIdx.x; c < ncta; c += NT) local += part[(size_t)b * ncta + c];
    const double s = block_sum<NT>(local, red);
    if (threadIdx.x == 0) out[b] = s;
}

}  // namespace rg

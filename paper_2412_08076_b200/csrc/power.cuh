// power.cuh — one fused launch per power-iteration step (spectral.py:31-57).
//
// Step k of the reference:
//     y = A x            (or sigma*x - A x for the shifted iteration, :75-76)
//     lam = Re <x, y>    (np.vdot)
//     ny = ||y||
//     x = y / ny
// Here launch k reads the previous step's y and ny and forms x = y_prev / ny
// on the fly for every stencil input (the same division the reference does,
// so x is bit-identical to the reference's x), applies the stencil in CSR
// order, writes y, and reduces <x, y> and <y, y> per CTA; the last CTA of
// each system (atomic ticket) sums the partials in a fixed order and writes
// lam[k], ny[k].  The next launch reads ny[k] from memory, so a batch of
// steps is a chain of kernels with no host round trip and no library calls.
#pragma once
#include "step.cuh"

namespace rg {

struct PowerArgs {
    OpView<double> A;
    const double* y_prev;   // [B][P]: previous y (step 0: the normalised start vector)
    const double* ny_prev;  // [B]: previous ||y|| (null: 1.0, i.e. y_prev is x itself)
    double* y_out;          // [B][P]
    double* x_out;          // [B][P] or null: x of this step
    double sigma;
    int shifted;            // y = sigma*x - A x
    double* part;           // [B][2][ncta_cap]
    int ncta_cap;
    int* counter;           // [B], zero between launches
    double* lam_out;        // [B]
    double* ny_out;         // [B]
};

template <int KIND>
__global__ void __launch_bounds__(STEP_NT) power_step_kernel(PowerArgs a) {
    const int b = blockIdx.z;
    const int side = a.A.side;
    const int cta = blockIdx.x + gridDim.x * blockIdx.y;
    const int ncta = gridDim.x * gridDim.y;
    const int j = blockIdx.x * STEP_BX + threadIdx.x;
    const int i = blockIdx.y * STEP_BY + threadIdx.y;
    const size_t base = (size_t)b * a.A.P;
    const double* yp = a.y_prev + base;
    const bool scaled = a.ny_prev != nullptr;
    const double ny = scaled ? a.ny_prev[b] : 1.0;
    double xy = 0.0, yy = 0.0;
    if (i < side && j < side) {
        const size_t idx = (size_t)i * side + j;
        auto X = [&](int di, int dj) -> double {
            const int ii = i + di, jj = j + dj;
            if (ii < 0 || ii >= side || jj < 0 || jj >= side) return 0.0;
            const double v = yp[idx + (ptrdiff_t)di * side + dj];
            return scaled ? v / ny : v;
        };
        const double x = X(0, 0);
        double y = apply_op<double, KIND>(a.A, b, idx, X);
        if (a.shifted) y = a.sigma * x - y;
        a.y_out[base + idx] = y;
        if (a.x_out) a.x_out[base + idx] = x;
        xy = x * y;
        yy = y * y;
    }
    __shared__ double red[STEP_NT / 32];
    __shared__ int is_last;
    const int tid = threadIdx.x + blockDim.x * threadIdx.y;
    double* part = a.part + (size_t)b * 2 * a.ncta_cap;
    const double s1 = block_sum<STEP_NT>(xy, red);
    if (tid == 0) part[cta] = s1;
    const double s2 = block_sum<STEP_NT>(yy, red);
    if (tid == 0) {
        part[a.ncta_cap + cta] = s2;
        __threadfence();
        const int t = atomicAdd(&a.counter[b], 1);
        is_last = (t == ncta - 1);
        if (is_last) __threadfence();
    }
    __syncthreads();
    if (!is_last) return;
    double l1 = 0.0, l2 = 0.0;
    for (int c = tid; c < ncta; c += STEP_NT) {
        l1 += __ldcg(&part[c]);
        l2 += __ldcg(&part[a.ncta_cap + c]);
    }
    const double t1 = block_sum<STEP_NT>(l1, red);
    const double t2 = block_sum<STEP_NT>(l2, red);
    if (tid == 0) {
        a.lam_out[b] = t1;
        a.ny_out[b] = sqrt(t2);
        a.counter[b] = 0;
        __threadfence();
    }
}

}  // namespace rg

// mg.cuh — V-cycle grid transfers and the coarsest-level solve
// (multigrid.py:24-59, 151-163).
//
// Full weighting R = kron(r1, r1), r1 = (1/4)[1 2 1] (multigrid.py:24-42) and
// bilinear prolongation P = kron(p1, p1), p1 = 2 r1^T (:45-49).  Every weight
// is a power of two, so each product is exact and the result only depends
// on the summation order, which follows the CSR column order of the
// reference's kron matrices: bitwise equal to R.matvec / P.matvec.
#pragma once
#include "common.cuh"

namespace rg {

constexpr int MG_BX = 32, MG_BY = 8;

// coarse[I, J] = sum_{a,b in 0..2} (w_a w_b) fine[2I+a, 2J+b]  (a major, b minor)
template <typename S>
__global__ void __launch_bounds__(MG_BX * MG_BY)
restrict_kernel(const S* __restrict__ fine, S* __restrict__ coarse, int nf, int nc) {
    const int b = blockIdx.z;
    const int J = blockIdx.x * MG_BX + threadIdx.x;
    const int I = blockIdx.y * MG_BY + threadIdx.y;
    if (I >= nc || J >= nc) return;
    const S* x = fine + (size_t)b * nf * nf + (size_t)(2 * I) * nf + 2 * J;
    const double w[3] = {0.25, 0.5, 0.25};
    CT<S> s = rmul(w[0] * w[0], to_c(x[0]));
#pragma unroll
    for (int q = 1; q < 9; ++q) {
        const int a = q / 3, c = q % 3;
        s = add(s, rmul(w[a] * w[c], to_c(x[(size_t)a * nf + c])));
    }
    coarse[(size_t)b * nc * nc + (size_t)I * nc + J] = to_s<S>(s);
}

// fine[p, q] = fine[p, q] + sum_{I in I(p)} sum_{J in J(q)} (pw_I pw_J) e[I, J]
// with I(p) = {p/2 - 1, p/2} (weights 1/2, 1/2) for even p, {(p-1)/2} (weight 1)
// for odd p, restricted to [0, nc).
template <typename S>
__global__ void __launch_bounds__(MG_BX * MG_BY)
prolong_add_kernel(const S* __restrict__ e, S* __restrict__ fine, int nf, int nc) {
    const int b = blockIdx.z;
    const int q = blockIdx.x * MG_BX + threadIdx.x;
    const int p = blockIdx.y * MG_BY + threadIdx.y;
    if (p >= nf || q >= nf) return;
    int Ii[2], Jj[2], ni = 0, nj = 0;
    double wi[2], wj[2];
    if (p & 1) { Ii[ni] = (p - 1) >> 1; wi[ni++] = 1.0; }
    else {
        if (p / 2 - 1 >= 0) { Ii[ni] = p / 2 - 1; wi[ni++] = 0.5; }
        if (p / 2 < nc) { Ii[ni] = p / 2; wi[ni++] = 0.5; }
    }
    if (q & 1) { Jj[nj] = (q - 1) >> 1; wj[nj++] = 1.0; }
    else {
        if (q / 2 - 1 >= 0) { Jj[nj] = q / 2 - 1; wj[nj++] = 0.5; }
        if (q / 2 < nc) { Jj[nj] = q / 2; wj[nj++] = 0.5; }
    }
    const S* ec = e + (size_t)b * nc * nc;
    CT<S> s = szero<CT<S>>();
    bool first = true;
    for (int i = 0; i < ni; ++i)
        for (int j = 0; j < nj; ++j) {
            const CT<S> t = rmul(wi[i] * wj[j], to_c(ec[(size_t)Ii[i] * nc + Jj[j]]));
            s = first ? t : add(s, t);
            first = false;
        }
    S* u = fine + (size_t)b * nf * nf + (size_t)p * nf + q;
    if (!first) *u = to_s<S>(add(to_c(*u), s));   // u = u + P e  (multigrid.py:162)
}

// y[b] = M[bm] x[b], M dense [n][n] row-major (coarsest-level inverse), one
// warp per row, fixed-order shuffle reduction.
template <typename S>
__global__ void __launch_bounds__(256) dense_apply_kernel(const S* __restrict__ M, int shared,
                                                          const S* __restrict__ x, S* __restrict__ y,
                                                          int n) {
    const int b = blockIdx.y;
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const S* Mr = M + (shared ? 0 : (size_t)b * n * n) + (size_t)row * n;
    const S* xb = x + (size_t)b * n;
    CT<S> s = szero<CT<S>>();
    for (int j = lane; j < n; j += 32) s = add(s, mul(to_c(Mr[j]), to_c(xb[j])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = add(s, shfl_down(s, o));
    if (lane == 0) y[(size_t)b * n + row] = to_s<S>(s);
}

}  // namespace rg

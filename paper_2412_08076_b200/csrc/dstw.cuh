// dstw.cuh — the lean DST-I line kernel for M = 512, 1024, 2048 (csrc/dstw.cu):
// interface shared with capi.cu.  Same transform as dst.cuh (transforms.py:24-35,
// fns.py:43-44); see dstw.cu for the kernel design.
#pragma once
#include <cuda_runtime.h>

namespace rg {

// Element k (1..N) of line L (1..N) of system b lives at
//   base[b * bs + off + L * ls + k * es]           (doubles; off may be negative:
// an unpadded [N][N] array has off = -(N + 1), a padded [M][M] array off = 0).
struct DstwView {
    double* base;
    long long bs, off, ls, es;
};

enum { DSTW_PLAIN = 0, DSTW_TWICE_LAM = 1, DSTW_ADD = 2 };

struct DstwArgs {
    DstwView in, out, lam;   // lam: DSTW_TWICE_LAM only
    const double2* tw;       // [M] (cos, sin)(pi k / M)
    int B, N;
    double s4;               // -0.25 * sqrt(2 / M): orthonormal scale with the -Im/2 of the odd extension
};

// col = false: lines are walked with consecutive threads on one line (rows of a
// row-major array: es = 1); col = true: 256 / (M / 16) adjacent lines are
// interleaved across the lanes of every warp (columns: ls = 1).  Both take
// any strides; the mapping only decides what coalesces.
cudaError_t launch_dstw(const DstwArgs& a, int logM, bool col, int mode, int num_sms, cudaStream_t st);
bool dstw_supported(int M);

}  // namespace rg

// Microbenchmark: one inner step of the cfg1 cluster solver's skeleton.
//   A: cluster.sync only;  B: DSMEM store of one row (63 doubles) to each
//   neighbour + cluster.sync;  C: B + a dependent 17-op FP64 chain per thread.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void loop(int n, double* out) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double buf[2][8 * 65];
    const int cr = cl.block_rank(), nc = cl.num_blocks();
    double x = threadIdx.x * 1e-3;
    for (int i = 0; i < n; ++i) {
        double* b = buf[i & 1];
        if (MODE >= 1 && threadIdx.x < 63) {
            if (cr > 0) cl.map_shared_rank(b, cr - 1)[7 * 65 + threadIdx.x] = x;
            if (cr < nc - 1) cl.map_shared_rank(b, cr + 1)[threadIdx.x] = x;
        }
        cl.sync();
        if (MODE >= 2) {
            double s = b[threadIdx.x % 65] * 0.5;
#pragma unroll
            for (int q = 0; q < 8; ++q) s = s + b[(threadIdx.x + q) % 65] * 0.25;
            x = s;
        }
    }
    if (x == 12345.0) out[0] = x;
}

template <int MODE>
void run(int C, double* d) {
    cudaFuncSetAttribute(loop<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    const int n = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, loop<MODE>, 100, d);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, loop<MODE>, n, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("mode %d cluster %2d: %.1f ns per step (%s)\n", MODE, C, ms * 1e6 / n, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    for (int C : {2, 16}) { run<0>(C, d); run<1>(C, d); run<2>(C, d); }
    return 0;
}

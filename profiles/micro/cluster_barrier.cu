// Microbenchmark: cost of a thread-block-cluster barrier on B200 (cluster of
// C CTAs x 256 threads, N barriers in a loop), and of a split arrive/wait.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void bar_loop(int n, int* out) {
    cg::cluster_group cl = cg::this_cluster();
    int x = 0;
    for (int i = 0; i < n; ++i) {
        cl.sync();
        x += threadIdx.x;
    }
    if (x == -1) out[0] = x;
}

__global__ void sync_loop(int n, int* out) {
    int x = 0;
    for (int i = 0; i < n; ++i) {
        __syncthreads();
        x += threadIdx.x;
    }
    if (x == -1) out[0] = x;
}

int main() {
    int* d;
    cudaMalloc(&d, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int n = 20000;
    for (int C : {1, 2, 4, 8, 16}) {
        cudaFuncSetAttribute(bar_loop, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C);
        cfg.blockDim = dim3(256);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, bar_loop, 100, d);
        cudaEventRecord(a);
        cudaLaunchKernelEx(&cfg, bar_loop, n, d);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("cluster %2d CTAs: %.1f ns per cluster.sync (err %s)\n", C, ms * 1e6 / n,
               cudaGetErrorString(cudaGetLastError()));
    }
    sync_loop<<<1, 256>>>(100, d);
    cudaEventRecord(a);
    sync_loop<<<1, 256>>>(n, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("__syncthreads (256 threads): %.1f ns\n", ms * 1e6 / n);
    return 0;
}

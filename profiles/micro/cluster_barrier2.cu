// Microbenchmark: cluster barrier flavours on B200 (16-CTA cluster, 256
// threads): cg::cluster.sync() vs PTX arrive.release/wait.acquire vs
// arrive.relaxed/wait + fence.acq_rel.cluster, each after a DSMEM store.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void loop(int n, double* out) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double buf[2][64];
    const int cr = cl.block_rank(), nc = cl.num_blocks();
    double x = threadIdx.x;
    for (int i = 0; i < n; ++i) {
        double* b = buf[i & 1];
        if (threadIdx.x < 63) cl.map_shared_rank(b, (cr + 1) % nc)[threadIdx.x] = x;
        if (MODE == 0) {
            cl.sync();
        } else if (MODE == 1) {
            asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else {
            asm volatile("fence.acq_rel.cluster;\n\tbarrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
        }
        x += b[threadIdx.x & 63];
    }
    if (x == 12345.0) out[0] = x;
}

template <int MODE>
void run(double* d) {
    cudaFuncSetAttribute(loop<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
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
    printf("mode %d: %.1f ns per step (%s)\n", MODE, ms * 1e6 / n, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    run<0>(d); run<1>(d); run<2>(d);
    return 0;
}

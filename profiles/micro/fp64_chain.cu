// Dependent-chain latencies on one warp (cycles per link): DFMA, DADD, 64-bit
// shuffle-up, shuffle + select + DFMA (the wavefront step of csrc/tri.cuh),
// and the same with 4 / 8 warps per SM quadrant-sharing the FP64 pipe.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=false -o fp64_chain fp64_chain.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 4096;
__global__ void k_dfma(double* out, long long* cyc, double a, double b) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __fma_rn(a, x, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_dadd(double* out, long long* cyc, double a, double b) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = x + b;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_ffma(float* out, long long* cyc, float a, float b) {
    float x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __fmaf_rn(a, x, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_shfl(double* out, long long* cyc, double a, double b) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __shfl_up_sync(0xffffffffu, x, 1);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_step(double* out, long long* cyc, double a, double b) {
    double x = out[threadIdx.x], left = x;
    const int lane = threadIdx.x & 31;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) {
        double sh = __shfl_up_sync(0xffffffffu, x, 1);
        double nb = lane ? sh : b;
        double u = __fma_rn(a, left, b);
        x = __fma_rn(a, nb, u);
        left = x;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// float pair (double-float) step for comparison of the shuffle path only
__global__ void k_shfl32(float* out, long long* cyc) {
    float x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __shfl_up_sync(0xffffffffu, x, 1);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double* d; long long* c; float* f;
    cudaMalloc(&d, 1024 * 8); cudaMalloc(&c, 64 * 8); cudaMalloc(&f, 1024 * 4);
    cudaMemset(d, 0, 1024 * 8); cudaMemset(f, 0, 1024 * 4);
    long long h[64];
    for (int nt : {32, 128, 256, 512, 1024}) {
        auto rep = [&](const char* name) {
            cudaDeviceSynchronize();
            cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
            printf("%-10s threads %4d: %.1f cycles/link\n", name, nt, (double)h[0] / N);
        };
        k_dfma<<<1, nt>>>(d, c, 0.999, 1e-3); rep("dfma");
        k_dadd<<<1, nt>>>(d, c, 0.999, 1e-3); rep("dadd");
        k_ffma<<<1, nt>>>(f, c, 0.999f, 1e-3f); rep("ffma");
        k_shfl<<<1, nt>>>(d, c, 0.999, 1e-3); rep("shfl64");
        k_shfl32<<<1, nt>>>(f, c); rep("shfl32");
        k_step<<<1, nt>>>(d, c, 0.499, 1e-3); rep("step");
    }
    return 0;
}

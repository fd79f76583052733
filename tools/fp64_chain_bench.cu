// FP64 dependent-chain latency / throughput on the B200 (why the encode's
// sequential double reductions cost what they cost).  One chain per thread of
// `steps` dependent DFMAs; prints cycles per step for 1 warp/SM (latency) and
// for many warps/SM with all lanes active vs lane 0 only (throughput).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_chain_bench tools/fp64_chain_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(const float* __restrict__ x, double* out, int steps, int lane0_only,
                      long long* cyc) {
    const int lane = threadIdx.x & 31;
    if (lane0_only && lane != 0) return;
    double acc = 0.0;
    float v = x[threadIdx.x & 1023];
    long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < steps; ++i) {
        acc = __fma_rn((double)v, (double)v, acc);
        v += 1.0f;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void chain_smem(double* out, int steps, long long* cyc) {
    __shared__ float row[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) row[i] = 0.001f * i;
    __syncthreads();
    double acc = 0.0;
    long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < steps; ++i) acc = __fma_rn((double)row[(i + threadIdx.x) & 4095], (double)row[(i + threadIdx.x) & 4095], acc);
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    float* x; double* out; long long* cyc;
    cudaMalloc(&x, 4096 * 4); cudaMemset(x, 0, 4096 * 4);
    cudaMalloc(&out, 148 * 64 * 1024 * 8); cudaMallocManaged(&cyc, 8);
    const int steps = 1536;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int l0 = 0; l0 < 2; ++l0)
        for (int wps : {1, 4, 16, 32, 64}) {
            chain<<<148, 32 * wps>>>(x, out, steps, l0, cyc);
            cudaEventRecord(a);
            chain<<<148, 32 * wps>>>(x, out, steps, l0, cyc);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("reg chain  lane0_only=%d warps/SM=%2d: %.1f cyc/step (thread 0), kernel %.3f ms, "
                   "%.2f warp-DFMA/clk/SM\n", l0, wps, (double)*cyc / steps, ms,
                   (double)wps * steps / (ms * 1e-3 * 1.965e9));
        }
    for (int wps : {1, 16}) {
        chain_smem<<<148, 32 * wps>>>(out, steps, cyc);
        cudaDeviceSynchronize();
        printf("smem chain warps/SM=%2d: %.1f cyc/step\n", wps, (double)*cyc / steps);
    }
    return 0;
}

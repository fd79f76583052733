// Pipe-rate microbenchmark for the SM2 distance inner loop: POPC vs LOP3 vs
// IADD3 throughput (warp-instructions per SM per cycle) with 8 independent
// chains per thread.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// tools/popc_bench.cu -o build/popc_bench && build/popc_bench
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void pipe_kernel(unsigned* out, int iters, unsigned seed) {
    unsigned v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) v[i] = __popc(v[i]) + v[i];                         // POPC + IADD
            if (OP == 1) v[i] = (v[i] ^ (v[i] >> 3)) & (v[(i + 1) & 7] | 0x5u);  // LOP3-ish
            if (OP == 2) v[i] = v[i] + v[(i + 1) & 7] + 7u;                   // IADD3
        }
    }
    long long t1 = clock64();
    unsigned s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
    if (threadIdx.x == 0) out[blockIdx.x * 2] = (unsigned)(t1 - t0);
    if (s == 0x12345678u) out[1] = s;
}

int main() {
    unsigned* d;
    cudaMalloc(&d, 4096 * 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 4096;
    const char* names[3] = {"popc+iadd", "shf+lop3", "iadd3"};
    for (int op = 0; op < 3; ++op) {
        for (int warps : {1, 4, 16, 32}) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            auto launch = [&]() {
                if (op == 0) pipe_kernel<0><<<sms, warps * 32>>>(d, iters, 3);
                if (op == 1) pipe_kernel<1><<<sms, warps * 32>>>(d, iters, 3);
                if (op == 2) pipe_kernel<2><<<sms, warps * 32>>>(d, iters, 3);
            };
            launch();
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            unsigned cyc = 0;
            cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
            // ops per thread = iters * 8 (each op = 2 instructions for popc / lop variants)
            const double warp_ops = (double)iters * 8 * warps;
            printf("%-10s warps/SM %2d: %8u cyc  -> %.3f warp-ops/SM/cyc  (%.3f ms)\n", names[op],
                   warps, cyc, warp_ops / cyc, ms);
        }
    }
    return 0;
}

// Microbenchmark: achievable bandwidth of random code-row gathers on B200.
// Rows of RB bytes (192 = D768 codes) at random ids; each warp handles a
// stream of "expansions" of R rows, computing an XOR/popcount sum so loads
// cannot be elided.  Variants:
//   0  LDG.128, G lanes per row (chunks interleaved), PB passes in flight
//   1  cp.async.bulk (TMA 1-D bulk) one copy per row into smem, mbarrier wait
//   2  LDG.128, one lane per row (row streamed by one lane)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e_ = (x);                                                  \
        if (e_ != cudaSuccess) {                                               \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

__device__ __forceinline__ uint4 ldg_nc(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ uint32_t mix(uint4 a) { return __popc(a.x ^ a.y) + __popc(a.z & a.w); }

// ids: warps x exps x R
template <int W, int G, int PB>
__global__ void k_ldg(const uint4* __restrict__ codes, const uint32_t* __restrict__ ids, int exps,
                      int R, unsigned long long* out) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    constexpr int CPL = W / G, RPP = 32 / G;
    const int sub = lane % G, grp = lane / G;
    uint32_t acc = 0;
    const uint32_t* my = ids + (size_t)warp * exps * R;
    for (int e = 0; e < exps; ++e) {
        const uint32_t* row_ids = my + (size_t)e * R;
        for (int b0 = 0; b0 < R; b0 += RPP * PB) {
            uint4 buf[PB][CPL];
#pragma unroll
            for (int b = 0; b < PB; ++b) {
                const int r = b0 + b * RPP + grp;
                const uint32_t id = r < R ? __ldg(row_ids + r) : 0;
#pragma unroll
                for (int c = 0; c < CPL; ++c)
                    buf[b][c] = r < R ? ldg_nc(codes + (size_t)id * W + sub + c * G) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int b = 0; b < PB; ++b)
#pragma unroll
                for (int c = 0; c < CPL; ++c) acc += mix(buf[b][c]);
        }
        acc = __reduce_add_sync(0xffffffff, acc) & 0xffff;  // serialise expansions
    }
    if (lane == 0) atomicAdd(out, acc);
}

// one lane per row: lane streams its row's W chunks
template <int W>
__global__ void k_lane(const uint4* __restrict__ codes, const uint32_t* __restrict__ ids, int exps,
                       int R, unsigned long long* out) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t acc = 0;
    const uint32_t* my = ids + (size_t)warp * exps * R;
    for (int e = 0; e < exps; ++e) {
        for (int r0 = 0; r0 < R; r0 += 32) {
            const int r = r0 + lane;
            if (r < R) {
                const uint32_t id = __ldg(my + (size_t)e * R + r);
                uint4 buf[W];
#pragma unroll
                for (int c = 0; c < W; ++c) buf[c] = ldg_nc(codes + (size_t)id * W + c);
#pragma unroll
                for (int c = 0; c < W; ++c) acc += mix(buf[c]);
            }
        }
        acc = __reduce_add_sync(0xffffffff, acc) & 0xffff;
    }
    if (lane == 0) atomicAdd(out, acc);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
        "r"(phase)
        : "memory");
}

// TMA 1-D bulk copy per row into per-warp smem, then compute from smem
template <int W>
__global__ void k_tma(const uint4* __restrict__ codes, const uint32_t* __restrict__ ids, int exps,
                      int R, unsigned long long* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + wib * (16 + R * W * 16));
    uint4* buf = reinterpret_cast<uint4*>(sm + wib * (16 + R * W * 16) + 16);
    if (lane == 0) mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t acc = 0, phase = 0;
    const uint32_t* my = ids + (size_t)warp * exps * R;
    for (int e = 0; e < exps; ++e) {
        const uint32_t id = lane < R ? __ldg(my + (size_t)e * R + lane) : 0;
        const uint32_t id2 = lane + 32 < R ? __ldg(my + (size_t)e * R + lane + 32) : 0;
        if (lane == 0) mbar_expect_tx(bar, R * W * 16);
        __syncwarp();
        if (lane < R) bulk_g2s(buf + lane * W, codes + (size_t)id * W, W * 16, bar);
        if (lane + 32 < R) bulk_g2s(buf + (lane + 32) * W, codes + (size_t)id2 * W, W * 16, bar);
        mbar_wait(bar, phase);
        phase ^= 1;
        for (int i = lane; i < R * W; i += 32) acc += mix(buf[i]);
        acc = __reduce_add_sync(0xffffffff, acc) & 0xffff;
        __syncwarp();
    }
    if (lane == 0) atomicAdd(out, acc);
}

// TMA tile::gather4: 4 random rows per TMA instruction (sm_100a)
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int r0, int r1,
                                            int r2, int r3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
        "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
        "r"((uint32_t)__cvta_generic_to_shared(bar))
        : "memory");
}

template <int W>
__global__ void k_g4(const __grid_constant__ CUtensorMap map, const uint32_t* __restrict__ ids,
                     int exps, int R, unsigned long long* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const size_t per = 128 + 64 * W * 16;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + wib * per);
    uint4* buf = reinterpret_cast<uint4*>(sm + wib * per + 128);
    if (lane == 0) mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t acc = 0, phase = 0;
    const uint32_t* my = ids + (size_t)warp * exps * R;
    const int ng = (R + 3) / 4;
    for (int e = 0; e < exps; ++e) {
        if (lane == 0) mbar_expect_tx(bar, ng * 4 * W * 16);
        __syncwarp();
        if (lane < ng) {
            const uint32_t* p = my + (size_t)e * R + lane * 4;
            int r[4];
            for (int j = 0; j < 4; ++j) r[j] = lane * 4 + j < R ? (int)__ldg(p + j) : (int)__ldg(p);
            tma_gather4(buf + lane * 4 * W, &map, r[0], r[1], r[2], r[3], bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        for (int i = lane; i < R * W; i += 32) acc += mix(buf[i]);
        acc = __reduce_add_sync(0xffffffff, acc) & 0xffff;
        __syncwarp();
    }
    if (lane == 0) atomicAdd(out, acc);
}

int main(int argc, char** argv) {
    const size_t N = argc > 3 ? (size_t)atol(argv[3]) : 1000000;
    const int W = 12;  // 192-B rows
    const int R = 64;
    const int exps = argc > 1 ? atoi(argv[1]) : 40;
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint4* codes;
    CK(cudaMalloc(&codes, N * W * 16));
    CK(cudaMemset(codes, 0x5a, N * W * 16));
    const int max_warps = sms * 64;
    const size_t nid = (size_t)max_warps * exps * R;
    uint32_t* hid = (uint32_t*)malloc(nid * 4);
    uint64_t s = 88172645463325252ull;
    for (size_t i = 0; i < nid; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        hid[i] = (uint32_t)(s % N);
    }
    uint32_t* ids;
    CK(cudaMalloc(&ids, nid * 4));
    CK(cudaMemcpy(ids, hid, nid * 4, cudaMemcpyHostToDevice));
    unsigned long long* out;
    CK(cudaMalloc(&out, 8));
    void* flush;
    CK(cudaMalloc(&flush, 512 << 20));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto kern, int warps_per_sm, size_t smem_per_warp) {
        const int wpb = 4;
        const int blocks = sms * warps_per_sm / wpb;
        const int warps = blocks * wpb;
        if (smem_per_warp) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem_per_warp * wpb)));
        float best = 1e9;
        for (int it = 0; it < 3; ++it) {
            CK(cudaMemset(flush, it, 512 << 20));
            cudaEventRecord(a);
            kern<<<blocks, wpb * 32, smem_per_warp * wpb>>>(codes, ids, exps, R, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const double bytes = (double)warps * exps * R * W * 16;
        printf("%-28s warps/SM %2d : %8.3f ms  %7.1f GB/s  (%.2f us/expansion/warp)\n", name,
               warps_per_sm, best, bytes / best / 1e6, best * 1e3 / exps);
    };
    int mode = argc > 2 ? atoi(argv[2]) : 0;
    // tensor map over the code rows: 2D {W*2 u64 columns, N rows}
    CUtensorMap tmap;
    {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        cuuint64_t gdim[2] = {(cuuint64_t)(W * 2), (cuuint64_t)N};
        cuuint64_t gstride[1] = {(cuuint64_t)(W * 16)};
        cuuint32_t box[2] = {(cuuint32_t)(W * 2), 1};
        cuuint32_t es[2] = {1, 1};
        CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, codes, gdim, gstride, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("tensor map encode failed %d\n", (int)r); return 1; }
    }
    auto run_g4 = [&](int rr, int wps) {
        const int wpb = wps < 4 ? wps : 4;
        const int blocks = sms * wps / wpb;
        const int warps = blocks * wpb;
        const size_t smem = (128 + 64 * W * 16) * wpb;
        CK(cudaFuncSetAttribute(k_g4<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        float best = 1e9;
        for (int it = 0; it < 3; ++it) {
            CK(cudaMemset(flush, it, 512 << 20));
            cudaEventRecord(a);
            k_g4<12><<<blocks, wpb * 32, smem>>>(tmap, ids, exps, rr, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const double bytes = (double)warps * exps * rr * W * 16;
        printf("%-22s R=%2d warps/SM %2d : %7.2f us/expansion  %7.1f GB/s\n", "tma gather4", rr, wps,
               best * 1e3 / exps, bytes / best / 1e6);
    };
    if (mode == 2) {
        for (int rr : {1, 8, 32, 64})
            for (int wps : {1, 8, 16}) run_g4(rr, wps);
        return 0;
    }
    if (mode == 1) {
        // latency model: rows per expansion R' in {1, 8, 32, 64}, 1..8 warps/SM
        for (int rr : {1, 8, 32, 64}) {
            for (int wps : {1, 4, 8}) {
                auto runR = [&](const char* name, auto kern, size_t smem_per_warp) {
                    const int wpb = wps < 4 ? wps : 4;
                    const int blocks = sms * wps / wpb;
                    const int warps = blocks * wpb;
                    if (smem_per_warp) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem_per_warp * wpb)));
                    float best = 1e9;
                    for (int it = 0; it < 3; ++it) {
                        CK(cudaMemset(flush, it, 512 << 20));
                        cudaEventRecord(a);
                        kern<<<blocks, wpb * 32, smem_per_warp * wpb>>>(codes, ids, exps, rr, out);
                        cudaEventRecord(b);
                        CK(cudaEventSynchronize(b));
                        CK(cudaGetLastError());
                        float ms;
                        cudaEventElapsedTime(&ms, a, b);
                        if (ms < best) best = ms;
                    }
                    const double bytes = (double)warps * exps * rr * W * 16;
                    printf("%-22s R=%2d warps/SM %d : %7.2f us/expansion  %7.1f GB/s\n", name, rr, wps,
                           best * 1e3 / exps, bytes / best / 1e6);
                };
                runR("ldg G4 PB8", k_ldg<12, 4, 8>, 0);
                runR("tma", k_tma<12>, 16 + 64 * W * 16);
            }
        }
        return 0;
    }
    for (int wps : {8, 16, 24, 32, 48}) {
        run("ldg G4 PB2 (16 rows)", k_ldg<12, 4, 2>, wps, 0);
        run("ldg G4 PB4 (32 rows)", k_ldg<12, 4, 4>, wps, 0);
        run("ldg G4 PB8 (64 rows)", k_ldg<12, 4, 8>, wps, 0);
        run("ldg G2 PB4 (64 rows)", k_ldg<12, 2, 4>, wps, 0);
        run("lane-per-row (32 rows)", k_lane<12>, wps, 0);
        if (wps <= 16) run("tma bulk per row (64 rows)", k_tma<12>, wps, 16 + R * W * 16);
    }
    return 0;
}

// Device primitives shared by the search (search.cu) and build (build.cu)
// kernels: the SM2 chunk distance and the TMA / mbarrier PTX wrappers.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace qvg {
namespace dev {

// SM2 distance contribution of one 16-B chunk {pos word, strong word}
// (encoding.hpp:169-176): popc(x) + popc(x & (sa|sb)) + 2*popc(x & sa & sb)
__device__ __forceinline__ uint32_t sm2_chunk(const uint4 q, const uint4 v) {
    const uint32_t x0 = q.x ^ v.x, x1 = q.y ^ v.y;
    const uint32_t o0 = x0 & (q.z | v.z), o1 = x1 & (q.w | v.w);
    const uint32_t a0 = x0 & q.z & v.z, a1 = x1 & q.w & v.w;
    return __popc(x0) + __popc(x1) + __popc(o0) + __popc(o1) + 2u * (__popc(a0) + __popc(a1));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n QVG_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra QVG_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// four rows (ids r0..r3) x one box of columns from column `col` -> dst (the 4
// rows packed consecutively; dst must be 128-B aligned), one TMA instruction
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint32_t col,
                                            uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}
// one contiguous range (1-D bulk copy; 16-B multiple, 16-B aligned)
__device__ __forceinline__ void bulk_row(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// warm L2 with a contiguous range (TMA bulk prefetch; size multiple of 16)
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// warm L2 with a small range through the LSU (one prefetch per 128-B line):
// unlike the bulk prefetch it does not queue behind the TMA gathers
__device__ __forceinline__ void prefetch_lines_l2(const void* src, uint32_t bytes) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(src) & ~uintptr_t(127);
    const uintptr_t a1 = reinterpret_cast<uintptr_t>(src) + bytes;
    for (uintptr_t a = a0; a < a1; a += 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}
// order this thread's generic-proxy smem accesses before later async-proxy
// (TMA) writes to the same smem
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace dev
}  // namespace qvg

// Device helpers shared by the search kernels (search.cu: one warp per query;
// search_coop.cu: a block of warps per query).  Key layout, visited hash,
// binary searches and the SM2 row accumulator; see search.cu's header for the
// algorithm and the reference lines each piece follows.
#pragma once

#include <cuda.h>
#include <stdint.h>

#include "bq_device.cuh"

namespace qvg {
namespace {

using namespace dev;  // sm2_chunk, TMA / mbarrier wrappers (bq_device.cuh)

// cross-proxy WAR fence before a TMA overwrites a stage the warp has read
#ifdef QVG_NO_TMA_FENCE
#define TMA_WAR_FENCE() ((void)0)
#else
#define TMA_WAR_FENCE() fence_proxy_async()
#endif

constexpr uint64_t kInfKey = ~0ull;
constexpr uint64_t kExp = 1ull << 32;
constexpr unsigned kFull = 0xFFFFFFFFu;

__device__ __forceinline__ uint64_t mkkey(uint32_t dist, uint32_t id) {
    return ((uint64_t)dist << 33) | id;
}
__device__ __forceinline__ uint64_t ordk(uint64_t k) { return k & ~kExp; }
__device__ __forceinline__ uint32_t kdist(uint64_t k) { return (uint32_t)(k >> 33); }

__device__ __forceinline__ uint32_t vhash(uint32_t id, uint32_t lg) {
    return (id * 0x9E3779B1u) >> (32 - lg);
}


// column 0 (code rows are one TMA box wide)
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint32_t r0,
                                            uint32_t r1, uint32_t r2, uint32_t r3,
                                            uint64_t* bar) {
    dev::tma_gather4(dst, map, 0, r0, r1, r2, r3, bar);
}
__device__ __forceinline__ void tma_gather4_col(void* dst, const CUtensorMap* map, uint32_t col,
                                                uint32_t r0, uint32_t r1, uint32_t r2,
                                                uint32_t r3, uint64_t* bar) {
    dev::tma_gather4(dst, map, col, r0, r1, r2, r3, bar);
}

// Row distance accumulator in bit planes (carry-save adders).  Per chunk the
// SM2 terms are four weight-1 words (x0, x1, o0, o1) and two weight-2 words
// (a0, a1) (encoding.hpp:169-176: popc(x) + popc(x & (sa|sb)) +
// 2 popc(x & sa & sb)).  LOP3 runs on the ALU pipe (2 warp-ops per SM per
// cycle) and POPC on the XU pipe (0.5; tools/popc_bench.cu), and the distance
// loop is ALU-pipe bound (ncu: math-pipe throttle on the CSA lines), so the
// reduction stops where the two pipes balance: three CSAs fold the four
// weight-1 words and their two carries, and the three words left per chunk
// (one weight-4 carry, a0, a1) are counted at once.  14 ALU + 3 XU ops per
// chunk; measured on cfg 2 (same box, profiles/r2e_sm2acc_ab.txt): six POPCs
// (round 1 start) XU bound; five CSAs + a weight-8 half adder, 19 ALU + 1 XU
// (round 1 final) 4.17 M QPS; four CSAs 4.37 M; three CSAs (this) 4.39 M;
// two CSAs 4.36 M.
__device__ __forceinline__ void csa(uint32_t& a, uint32_t b, uint32_t c, uint32_t& carry) {
    const uint32_t u = a ^ b;
    carry = (a & b) | (u & c);
    a = u ^ c;
}
struct Sm2Acc {
    uint32_t ones = 0, twos = 0, d2 = 0, d4 = 0;
    __device__ __forceinline__ void add(const uint4 q, const uint4 v) {
        const uint32_t x0 = q.x ^ v.x, x1 = q.y ^ v.y;
        const uint32_t o0 = x0 & (q.z | v.z), o1 = x1 & (q.w | v.w);
        const uint32_t a0 = x0 & q.z & v.z, a1 = x1 & q.w & v.w;
        uint32_t c1, c2, f1;
        csa(ones, x0, x1, c1);  // weight 1 -> carries of weight 2
        csa(ones, o0, o1, c2);
        csa(twos, c1, c2, f1);  // weight 2 -> carry of weight 4
        d4 += __popc(f1);  // (IMAD adds, to move them to the FMA pipe: no gain)
        d2 += __popc(a0) + __popc(a1);
    }
    __device__ __forceinline__ uint32_t total() const {
        return __popc(ones) + 2u * (__popc(twos) + d2) + 4u * d4;
    }
};

// SM2 distance of one staged row, taken by one of the LPR lanes that share
// the row: part p (t = p, p+LPR, ... < W) reads chunk (rot + t - p) mod W,
// rot = lane mod W — the per-lane rotation that keeps the 8 lanes of an
// LDS.128 phase on distinct bank quads.  One lockstep loop (a per-lane wrap
// point must not become a branch: divergent segments cost +50 %), unrolled by
// 4 with the four chunk indices computed first so the eight loads can issue
// together.
__device__ __forceinline__ uint32_t row_sm2(const uint4* __restrict__ qc,
                                            const uint4* __restrict__ row, uint32_t W,
                                            uint32_t rot, uint32_t part, uint32_t LPR) {
    Sm2Acc acc;
    const uint32_t iters = (W - part + LPR - 1) / LPR;
    uint32_t cc = rot, i = 0;
    auto nxt = [&](uint32_t x) {
        x += LPR;
        return x >= W ? x - W : x;
    };
    for (; i + 4 <= iters; i += 4) {
        const uint32_t c0 = cc, c1 = nxt(c0), c2 = nxt(c1), c3 = nxt(c2);
        cc = nxt(c3);
        const uint4 q0 = qc[c0], v0 = row[c0], q1 = qc[c1], v1 = row[c1];
        const uint4 q2 = qc[c2], v2 = row[c2], q3 = qc[c3], v3 = row[c3];
        acc.add(q0, v0);
        acc.add(q1, v1);
        acc.add(q2, v2);
        acc.add(q3, v3);
    }
    for (; i < iters; ++i) {
        acc.add(qc[cc], row[cc]);
        cc = nxt(cc);
    }
    return acc.total();
}

// The same with the code width WC and the lanes per row L as compile-time
// constants (wide rows: WC = 24 with L = 2, WC = 48 with L = 4; rows start on
// the same bank quad, 16·WC being a multiple of 128 B).  Lane (row r, part p)
// starts at chunk s = L·(r mod 8/L) + p <= 7 and steps by L: the 8 lanes of an
// LDS.128 phase (8/L rows x L parts) hit 8 distinct bank quads, and the first
// (WC - 8)/L + 1 chunks of every lane need no wrap — constant offsets from two
// base pointers instead of per-chunk index arithmetic.
template <int WC, int L>
__device__ __forceinline__ uint32_t row_sm2_fixed(const uint4* __restrict__ qc,
                                                  const uint4* __restrict__ row, uint32_t lane) {
    static_assert(WC % L == 0 && 8 % L == 0 && (16 * WC) % 128 == 0, "geometry");
    constexpr int N = WC / L;             // chunks per lane
    constexpr int NF = (WC - 8) / L + 1;  // of which wrap-free for every start <= 7
    const uint32_t s = L * ((lane / L) & (8 / L - 1)) + (lane & (L - 1));
    const uint4* q = qc + s;
    const uint4* r = row + s;
    Sm2Acc acc;
#pragma unroll
    for (int i = 0; i < NF; ++i) acc.add(q[L * i], r[L * i]);
#pragma unroll
    for (int i = NF; i < N; ++i) {
        uint32_t c = s + (uint32_t)(L * i);
        c = c >= (uint32_t)WC ? c - WC : c;
        acc.add(qc[c], row[c]);
    }
    return acc.total();
}

// The same for rows that alternate between two bank-quad bases (16·WC is an odd
// multiple of 64 B, e.g. WC = 12): two adjacent rows cover all 8 quads once they
// share a start chunk, so the rotation advances by L per PAIR of rows; start
// chunks are <= 3 and the first (WC - 4)/L + 1 chunks of every lane are wrap-free.
template <int WC, int L>
__device__ __forceinline__ uint32_t row_sm2_fixed_alt(const uint4* __restrict__ qc,
                                                      const uint4* __restrict__ row, uint32_t lane) {
    static_assert(WC % L == 0 && 4 % L == 0 && (16 * WC) % 128 == 64, "geometry");
    constexpr int N = WC / L;
    constexpr int NF = (WC - 4) / L + 1;
    const uint32_t s = L * ((lane / (2 * L)) & (4 / L - 1)) + (lane & (L - 1));
    const uint4* q = qc + s;
    const uint4* r = row + s;
    Sm2Acc acc;
#pragma unroll
    for (int i = 0; i < NF; ++i) acc.add(q[L * i], r[L * i]);
#pragma unroll
    for (int i = NF; i < N; ++i) {
        uint32_t c = s + (uint32_t)(L * i);
        c = c >= (uint32_t)WC ? c - WC : c;
        acc.add(qc[c], row[c]);
    }
    return acc.total();
}

// first index i in [0, n) with ordk(a[i]) >= x.  4-ary: three independent
// pivot loads per round, half the dependent shared-memory round trips of a
// binary search (cfg 2 ef 256: 10.16 -> 10.13 ms; with the merge's broadcast
// shift 9.79 ms, profiles/r2e_sm2acc_ab.txt)
__device__ __forceinline__ uint32_t lower_bound_key(const uint64_t* a, uint32_t n, uint64_t x) {
    uint32_t lo = 0;
    while (n >= 4) {
        const uint32_t q = n >> 2;
        const uint64_t k1 = ordk(a[lo + q - 1]), k2 = ordk(a[lo + 2 * q - 1]),
                       k3 = ordk(a[lo + 3 * q - 1]);
        const uint32_t c = (uint32_t)(k1 < x) + (uint32_t)(k2 < x) + (uint32_t)(k3 < x);
        lo += c * q;
        n = c == 3 ? n - 3 * q : q - 1;
    }
    uint32_t r = 0;
#pragma unroll
    for (uint32_t i = 0; i < 3; ++i) r += (i < n && ordk(a[lo + i]) < x) ? 1u : 0u;
    return lo + r;
}

// #{j < m : a[j] <= x} for non-decreasing a
__device__ __forceinline__ uint32_t upper_bound_u32(const uint32_t* a, uint32_t m, uint32_t x) {
    uint32_t lo = 0, hi = m;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}


// bytes of one 4-row TMA group in the stage; gather4 destinations must be
// 128-B aligned, so groups are padded (row j of a half lives at
// (j/4)*group_stride + (j%4)*16W)
__host__ __device__ inline uint32_t group_stride(uint32_t W) { return (64u * W + 127u) & ~127u; }

}  // namespace
}  // namespace qvg

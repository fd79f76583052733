// K2/K3/K4 — exact BQ beam search fused with the float32 rerank, one warp per
// query, persistent grid with an atomic query counter.
//
// Reference behaviour reproduced (paths under /root/reference/proj/core):
//   beam_search_words  search.cpp:27-81   dual-heap best-first search
//   candidate_less     graph.hpp:28-30    (dist, id) order == key order
//   sm2_distance_words encoding.hpp:169-176
//   rerank             search.cpp:96-120  4-chain double dot (vec_math.hpp:13-26),
//                                         sort (score desc, id asc), take k
//
// Memory path (B200): the code rows of an expansion's surviving neighbours are
// fetched by the Tensor Memory Accelerator with cp.async.bulk.tensor
// .tile::gather4 (four random rows per TMA instruction) into a double-buffered
// shared-memory stage guarded by mbarriers; a warp's 64-row gather takes ~2 us
// this way versus ~5 us with per-lane 128-bit loads (tools/gather_bench.cu).
// Distances are then computed lane-per-row from shared memory.  The adjacency
// row of the predicted next pick is prefetched while the gather is in flight.
//
// Search state (validated against the reference):
//   P   sorted pool of <= ef keys in shared memory.  key = dist<<33 | exp<<32 | id;
//       the order ignores the `exp` (expanded) bit, so (dist, id) order is a
//       plain u64 compare of (key & ~EXP).
//   T   tie stack: keys evicted from P while unexpanded whose dist equals the
//       pool's worst dist.  The worst dist never increases once P is full, so
//       all live T entries share one dist (tdist) and new entries (always
//       smaller keys) are pushed on top; a drop of the worst dist kills all of T.
//   vis lossy direct-mapped visited table.  A forgotten node that is scored
//       again is either already in P (exact lookup, dropped) or has key > max(P)
//       and is rejected, so results are unchanged.
// Admission of a row is the exact parallel form of the sequential loop: the
// i-th surviving neighbour c_i is admitted iff
//   #{p in P : p < c_i} + #{j < i : c_j < c_i} < ef
// and P' = first ef of merge(P, admitted).  Only "contenders" (c < max(P), or
// any c while P is not full) can matter, so only they are ranked and merged;
// the merge moves only the tail of P after the first insertion point, in place.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "bq_device.cuh"
#include "qvg_internal.cuh"
#include "search_common.cuh"

namespace qvg {

namespace {

using namespace dev;  // sm2_chunk, TMA / mbarrier wrappers (bq_device.cuh)

// per-phase cycle counters of the search loop: only in the instrumented build
// (python paper_2605_02171_b200/build.py --variant phases -DQVG_PHASES)
#ifdef QVG_PHASES
#define QVG_PH(...) __VA_ARGS__
#else
#define QVG_PH(...)
#endif

__device__ __forceinline__ float4 ldg_f4_noalloc(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

// 4 strided double chains combined as (s0+s1)+(s2+s3) (vec_math.hpp:13-26).
// Products of floats are exact in double, so FMA == mul+add here.
template <bool NOALLOC>
__device__ __forceinline__ float dot4_exact(const float* __restrict__ q,
                                            const float* __restrict__ v, uint32_t dim) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const float4* q4 = reinterpret_cast<const float4*>(q);
    const float4* v4 = reinterpret_cast<const float4*>(v);
    const uint32_t n4 = dim >> 2;
    uint32_t t = 0;
    for (; t + 8 <= n4; t += 8) {  // 128 B of the row in flight per lane
        float4 b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) b[u] = NOALLOC ? ldg_f4_noalloc(v4 + t + u) : __ldg(v4 + t + u);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float4 a = __ldg(q4 + t + u);
            s0 = __fma_rn((double)a.x, (double)b[u].x, s0);
            s1 = __fma_rn((double)a.y, (double)b[u].y, s1);
            s2 = __fma_rn((double)a.z, (double)b[u].z, s2);
            s3 = __fma_rn((double)a.w, (double)b[u].w, s3);
        }
    }
    for (; t < n4; ++t) {
        const float4 a = __ldg(q4 + t), b = __ldg(v4 + t);
        s0 = __fma_rn((double)a.x, (double)b.x, s0);
        s1 = __fma_rn((double)a.y, (double)b.y, s1);
        s2 = __fma_rn((double)a.z, (double)b.z, s2);
        s3 = __fma_rn((double)a.w, (double)b.w, s3);
    }
    for (uint32_t i = n4 << 2; i < dim; ++i)
        s0 = __fma_rn((double)__ldg(q + i), (double)__ldg(v + i), s0);
    return __double2float_rn(__dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3)));
}

struct SmemLayout {
    uint32_t bars, stage0, stage1, pk, ctd, evk, crp, csrp, cid, stg, qc, tie, vis, qsl, qd, acd, axk,
        axr, total;
};


// Per-warp shared-memory carve-up (bytes).  Stage halves are 128-B aligned
// (TMA destinations); the total is a multiple of 128 so every warp's base is.
// EFM = pool + extra-depth capacity rounded to 32; xa > 0 adds the extra-depth
// candidate buffers.
__host__ __device__ inline SmemLayout smem_layout(uint32_t EFM, uint32_t RM, uint32_t W,
                                                  uint32_t tie_cap, uint32_t vis_bytes,
                                                  uint32_t stage_rows, uint32_t xa = 0,
                                                  bool lean_ranks = false, bool geo = false) {
    SmemLayout L;
    uint32_t o = 0;
    auto take = [&](uint32_t bytes, uint32_t align) {
        o = (o + align - 1) & ~(align - 1);
        const uint32_t at = o;
        o += bytes;
        return at;
    };
    // geo: the stage first (no alignment gap) and the rerank query slices in
    // the contender buffer (dead during the rerank) — 496 B less per warp
    if (!geo) L.bars = take(16, 16);
    L.stage0 = take((stage_rows / 4) * group_stride(W), 128);
    L.stage1 = take((stage_rows / 4) * group_stride(W), 128);
    if (geo) L.bars = take(16, 16);
    L.pk = take(8 * EFM, 16);    // pool keys P[0, ef), then extra-depth keys A
    // contenders (row order) and their ranks in P.  geo: in stage half 0 — an
    // expansion has at most two halves there, every lane has consumed half 0
    // before the first contender is stored (the ballot in emit), and the
    // buffers are dead before the next step's TMA refills it (the proxy fence
    // in issue() orders these generic writes before the TMA's)
    L.ctd = geo ? L.stage0 : take(8 * RM, 16);
    L.evk = L.ctd;               // keys evicted this step (ctd is dead by then)
    L.crp = geo ? L.stage0 + 8 * RM : take(4 * RM, 16);  // contender rank in P, row order
    // contender rank in P, key order (lean_ranks: in the compacted-id buffer,
    // which is dead between the last distance pass and the next compaction)
    L.csrp = lean_ranks ? 0 : take(4 * RM, 16);
    L.cid = take(4 * RM, 16);    // compacted row ids to score
    if (lean_ranks) L.csrp = L.cid;
    L.stg = L.crp;               // tie-stack additions (crp is dead by then)
    L.qc = take(16 * W, 16);     // query code chunks
    L.tie = take(4 * tie_cap, 16);
    // visited table (vis_bytes = slots x entry width); the rerank scores
    // (EFM floats) alias this region
    L.vis = take(vis_bytes > 4 * EFM ? vis_bytes : 4 * EFM, 16);
    // rerank query slices (geo: over the compacted-id buffer and the query
    // code, contiguous and both dead during the rerank)
    L.qsl = geo && 4 * RM + 16 * W >= 2 * 48 * 4 ? L.cid : take(2 * 48 * 4, 16);
    // the current rerank round's query slice as doubles (converted once per
    // warp instead of once per lane)
    // (outside geo the contender buffer is ordinary shared memory, dead during
    // the rerank)
    L.qd = !geo && 8 * RM >= 48 * 8 ? L.ctd : take(48 * 8, 16);
    // extra depth: A candidates of one step (<= RM: each scored key is a P
    // contender or an A candidate, and evictions <= P contenders), sorted copy
    // and their ranks in A
    L.acd = take(xa ? 8 * RM : 0, 16);
    L.axk = take(xa ? 8 * RM : 0, 16);
    L.axr = take(xa ? 4 * RM : 0, 16);
    L.total = (o + 127u) & ~127u;
    return L;
}

// rows per stage half: a multiple of 4 (gather4 granularity), capped by the
// row count of an expansion, floor 4
__host__ __device__ inline uint32_t stage_rows_for(uint32_t W, uint32_t RM, uint32_t half_bytes) {
    uint32_t r = 4u * (half_bytes / group_stride(W));
    const uint32_t cap = (RM + 3u) & ~3u;
    if (r > cap) r = cap;
    if (r < 4) r = 4;
    return r;
}

// register budget per template: enough blocks that shared memory, not
// registers, bounds residency at the BASELINE geometries (R=32 rows -> ~9
// blocks of 2 warps fit in smem; R=64 -> ~7)
template <int RW, int RELP = 0>
#ifndef QVG_MINBLOCKS_RW2
#define QVG_MINBLOCKS_RW2 7
#endif
struct MinBlocks {
    static constexpr int value =
        RELP ? (RW <= 2 ? 8 : 7) : (RW == 1 ? 9 : (RW == 2 ? QVG_MINBLOCKS_RW2 : 5));
};

// XA: rerank deeper than ef.  A = the best `xa` scored keys outside P, kept
// sorted at pk[ef, ef + na): every A key exceeds max(P) (it was rejected or
// evicted while above the then-worst pool key, and the worst only falls), so
// pk[0, np + na) is the sorted list of the best scored keys.  A takes the
// step's non-contenders below max(A) and the keys leaving P; the search itself
// (pick, stop test, tie stack) never reads A.
// SPLIT: several lanes per scored row (wide rows, few rows per stage half); a
// separate instantiation because the extra loop costs the narrow-row kernels
// ~1.5% even when unused (cfg2 A/B, tools/tune_search.py).
// RELP > 0: the RELAXED variant (reported separately,
// never used for parity): each step expands the RELP best unexpanded pool
// entries at once and scores the union of their neighbours, admission is
// merge-then-truncate (no prefix rule) and there is no tie stack — fewer,
// wider serial steps per query.  RW is then the capacity of RELP rows, each
// lane holding RW / RELP slots of every picked row.
// WC > 0: the code width W as a compile-time constant (the headline geometry
// W = 12 has its own instantiation: constant row/group strides, fully
// unrolled distance loop).
// GEO: also the default stage geometry as constants (32 rows per stage half,
// 48-float rerank slices), dispatched when the launch uses exactly those.
// PRO: the fused-K1 prologue is compiled in (host queries, pipelined upload);
// the GEO instantiation for device-resident queries leaves it out.
// LEAN: the launch has both tensor maps and no exact-visited bitmaps, so the
// fallbacks and debug timers compile out (GEO implies it).
// ONE: one block per SM with as many warps as fit (GEO implies it), for the
// wide-row geometries whose per-warp shared memory leaves few warps per SM.
template <int RW, bool XA, bool SPLIT, int RELP = 0, int WC = 0, bool GEO = false, bool PRO = true,
          bool LEAN = GEO, bool ONE = GEO>
__global__ void __launch_bounds__((GEO || ONE) ? kGeoMaxWarps * 32 : kWarpsPerBlock * 32,
                                  (GEO || ONE) ? 1 : MinBlocks<RW, RELP>::value)
    search_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap cmap,
                  const SearchLaunch a, const uint32_t warp_bytes, const uint32_t SR_in,
                  const int use_tmap_in, const uint32_t SL_in) {
    // LEAN launches always have the code-row and cold-row tensor maps and never
    // the exact-visited bitmaps (the host dispatches them only then), so the
    // fallbacks compile out
    const int use_tmap = LEAN ? 1 : use_tmap_in;
    const uint32_t SR = GEO ? 32u : SR_in;
    const uint32_t SL = (GEO && SL_in) ? 48u : SL_in;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr uint32_t RM = RW * 32;
    constexpr bool REL = RELP > 0;
    constexpr int SPL = REL ? RW / RELP : RW;  // adjacency slots per lane per picked row
    static_assert(!REL || (SPL >= 1 && SPL * RELP == RW && !XA), "relaxed geometry");
    const uint32_t lane = threadIdx.x & 31;
    // (broadcast from lane 0: tells the compiler the warp index, and every
    // shared-memory address derived from it, is warp-uniform; cfg 2 +0.5 %)
    const uint32_t wib = __shfl_sync(0xFFFFFFFFu, threadIdx.x >> 5, 0);
    const uint32_t lt_mask = (1u << lane) - 1u;
    const DevIndex ix = a.ix;
    const uint32_t W = WC ? (uint32_t)WC : ix.W;
    const uint32_t rowb = 16u * W;
    const uint32_t gstride = group_stride(W);  // bytes per 4-row TMA group (128-B aligned)
    const uint32_t VS = 1u << a.vis_log2;
    const uint32_t ef = a.ef;  // (a compile-time ef = 64 instantiation measured +0.3 %)
    const uint32_t xa = XA ? extra_depth(ef, a.depth) : 0u;
    const uint32_t EFM = (ef + xa + 31u) & ~31u;
    // visited-table entry width: byte / short tags where they identify ids
    // exactly, else full ids
    // (the headline kernel is dispatched only when a short tag identifies ids
    // exactly, and always keeps 2-byte entries: compile-time table code)
    const uint32_t vtw = GEO ? 2u : vis_tag_bytes(ix.n, a.vis_log2);
    const uint32_t vbits = vis_id_bits(ix.n);
    const uint32_t vmask = vbits >= 32 ? ~0u : (1u << vbits) - 1u;
    const uint32_t vtb = vbits > a.vis_log2 ? vbits - a.vis_log2 : 0u;  // tag bits
    const SmemLayout L = smem_layout(EFM, RM, W, a.tie_cap, VS * vtw, SR, xa, true, GEO);
    unsigned char* base = smem_raw + (size_t)wib * warp_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + L.bars);
    unsigned char* const stage0 = base + L.stage0;
    const uint32_t stage_delta = L.stage1 - L.stage0;  // half h at stage0 + h * delta
    uint64_t* pk = reinterpret_cast<uint64_t*>(base + L.pk);
    uint64_t* ctd = reinterpret_cast<uint64_t*>(base + L.ctd);
    uint64_t* evk = reinterpret_cast<uint64_t*>(base + L.evk);
    uint32_t* crp = reinterpret_cast<uint32_t*>(base + L.crp);
    uint32_t* csrp = reinterpret_cast<uint32_t*>(base + L.csrp);
    uint32_t* cid = reinterpret_cast<uint32_t*>(base + L.cid);
    uint32_t* stg = reinterpret_cast<uint32_t*>(base + L.stg);
    uint4* qc = reinterpret_cast<uint4*>(base + L.qc);
    // tie stack: shared memory, or (re-run of queries whose shared-memory stack
    // overflowed; never in LEAN kernels) a per-warp-slot region of global memory
    // holding up to n entries — every node enters the stack at most once, so it
    // cannot overflow (the reference's frontier is unbounded, search.cpp:38-68)
    const bool tie_glob = !LEAN && a.tie_spill != nullptr;
    const uint64_t gwarp = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wib;
    uint32_t* tie = tie_glob ? a.tie_spill + gwarp * a.tie_spill_cap
                             : reinterpret_cast<uint32_t*>(base + L.tie);
    const uint32_t tie_cap = tie_glob ? a.tie_spill_cap : a.tie_cap;
    uint32_t* vis = reinterpret_cast<uint32_t*>(base + L.vis);
    float* sc = reinterpret_cast<float*>(base + L.vis);
    float* qsl = reinterpret_cast<float*>(base + L.qsl);
    double* qd = reinterpret_cast<double*>(base + L.qd);
    (void)qd;
    // visited-table test-and-set: true if `id` was not recorded (lossy: a
    // forgotten node is only re-scored, never wrongly skipped)
    auto vis_insert = [&](uint32_t id) -> bool {
        if constexpr (GEO) {
            const uint32_t mx = (id * 0x9E3779B1u) & vmask;
            const uint32_t s = mx >> vtb, tg = mx & ((1u << vtb) - 1u);
            uint16_t* v16 = reinterpret_cast<uint16_t*>(vis);
            if (v16[s] == tg) return false;
            v16[s] = (uint16_t)tg;
            return true;
        }
        if (vtw == 4u) {
            const uint32_t s = vhash(id, a.vis_log2);
            if (vis[s] == id) return false;
            vis[s] = id;
            return true;
        }
        const uint32_t mx = (id * 0x9E3779B1u) & vmask;
        const uint32_t s = mx >> vtb, tg = mx & ((1u << vtb) - 1u);
        if (vtw == 1u) {
            uint8_t* v8 = reinterpret_cast<uint8_t*>(vis);
            if (v8[s] == tg) return false;
            v8[s] = (uint8_t)tg;
            return true;
        }
        uint16_t* v16 = reinterpret_cast<uint16_t*>(vis);
        if (v16[s] == tg) return false;
        v16[s] = (uint16_t)tg;
        return true;
    };
    uint64_t* acd = reinterpret_cast<uint64_t*>(base + L.acd);
    uint64_t* axk = reinterpret_cast<uint64_t*>(base + L.axk);
    uint32_t* axr = reinterpret_cast<uint32_t*>(base + L.axr);
    uint64_t* pa = pk + ef;  // A

    uint32_t* xbits = (!LEAN && a.exact_bits) ? a.exact_bits + gwarp * a.exact_words : nullptr;
    const uint32_t rot = lane % W;  // per-lane chunk rotation (bank spreading)
    // lanes per scored row: the largest power of two with LPR * SR <= 32
    uint32_t lpr_log = 0;
    while (SPLIT && (SR << (lpr_log + 1)) <= 32u) ++lpr_log;
    const uint32_t LPR = SPLIT ? 1u << lpr_log : 1u;
    // x / SR == __umulhi(x, sr_m) for x < 2^32 / SR (x <= a few hundred here)
    const uint32_t sr_m = 0xFFFFFFFFu / SR + 1u;
    constexpr bool ctd_prefetch = true;  // prefetch the best contender's adjacency row
    // tail balancing (SearchLaunch::susp_*): the saved state is the contiguous
    // shared-memory range from the pool to the end of the visited table
    // (compiled only into the one-block-per-SM kernels: in the R = 32 kernels the
    // extra live state cost 5 % and their ~100-us queries gain nothing from units)
#ifdef QVG_NOSUSP
    constexpr bool SUSP = false;
#else
    constexpr bool SUSP = (GEO || ONE) && !REL && !XA;
#endif
    const uint32_t susp_end = GEO ? L.qd : L.qsl;

    if (lane == 0) {
        mbar_init(&bars[0]);
        mbar_init(&bars[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t phs = 0;  // bit h = phase parity of bars[h]

    // issue the TMA fetch of compacted rows [r0, r0+cnt) into stage half h
    auto issue = [&](uint32_t r0, uint32_t cnt, uint32_t h, bool fence = true) {
        uint64_t* bar = &bars[h];
        const uint32_t ng = use_tmap ? (cnt + 3u) >> 2 : cnt;
        const uint32_t bytes = use_tmap ? ng * 4u * rowb : cnt * rowb;
        if (fence) {
            TMA_WAR_FENCE();  // order this lane's reads of the half before TMA writes
            __syncwarp();         // all lanes finished reading this half
        }
        // (one elected lane issuing every group in a warp-uniform loop, with
        // broadcast index loads, measured 12 % slower than this per-lane
        // election loop: profiles/r2f_issue_ab.txt)
        if (lane == 0) mbar_expect_tx(bar, bytes);
        __syncwarp();
        for (uint32_t g = lane; g < ng; g += 32) {
            if (use_tmap) {
                const uint32_t j = r0 + 4u * g;  // multiple of 4: one 16-B load
                const uint4 c4 = *reinterpret_cast<const uint4*>(cid + j);
                const uint32_t i0 = c4.x;
                const uint32_t i1 = 4u * g + 1u < cnt ? c4.y : i0;
                const uint32_t i2 = 4u * g + 2u < cnt ? c4.z : i0;
                const uint32_t i3 = 4u * g + 3u < cnt ? c4.w : i0;
                tma_gather4(stage0 + h * stage_delta + (size_t)g * gstride, &tmap, i0, i1, i2, i3, bar);
            } else {
                bulk_row(stage0 + h * stage_delta + (size_t)(g >> 2) * gstride + (g & 3u) * rowb, ix.codes + (size_t)cid[r0 + g] * W, rowb,
                         bar);
            }
        }
    };

    for (;;) {
        unsigned long long qq = 0;
        if (lane == 0) qq = atomicAdd(a.counter, 1ull);
        qq = __shfl_sync(kFull, qq, 0);
        bool resume = false;  // this unit continues a suspended query
        if (qq >= a.nq) {
            if (!(SUSP && a.susp_ctl)) break;
            // fresh queries are gone: serve the FIFO of suspended queries until
            // every budgeted query has completed
            uint32_t ent = 0;
            if (lane == 0) {
                const uint32_t slot = atomicAdd(a.susp_ctl + 1, 1u);
                const uint32_t nb = (uint32_t)a.nq - a.susp_from;
                if (slot < a.susp_cap) {
                    for (uint32_t spins = 0; spins < (1u << 24); ++spins) {  // (bounded: ~4 s)
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(ent) : "l"(a.susp_list + slot) : "memory");
                        if (ent) break;
                        uint32_t done;
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(done) : "l"(a.susp_ctl + 2) : "memory");
                        if (done >= nb) {  // no push can follow: a last look at the slot
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(ent) : "l"(a.susp_list + slot) : "memory");
                            break;
                        }
                        __nanosleep(200);
                        // (never seen: a watchdog so a lost hand-off fails the call
                        // instead of hanging it)
                        if (spins + 1 == (1u << 24) && a.flags) atomicOr(a.flags, 1u << 30);
                    }
                }
            }
            ent = __shfl_sync(kFull, ent, 0);
            __syncwarp();  // lane 0's acquire orders every lane's reads of the saved state
            if (ent == 0) break;
            qq = ent - 1u;
            resume = true;
        }
        // a re-run launch serves a list of queries (qmap), never a LEAN kernel
        const uint64_t q = (!LEAN && a.qmap) ? (uint64_t)a.qmap[qq] : qq;
        const bool budgeted = SUSP && a.susp_ctl && q >= a.susp_from;
        if (a.ready && !resume) {  // pipelined upload: wait until this query's row has landed
            if (lane == 0) {
                uint32_t r;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(a.ready) : "memory");
                    if (r > q) break;
                    __nanosleep(256);
                }
            }
            __syncwarp();
        }

        int32_t qst = 0;
        if (resume) {
            // (encoded, validated and initialised by the unit that started it)
        } else if (PRO && a.qraw) {
            // fused K1 (encode.cu semantics, bit-exact): the stage is idle
            // between queries and holds the raw row; lane 0 runs the two
            // index-ordered double reductions (vec_math.hpp:28-44,
            // encoding.cpp:23-30); the rest is lane-parallel
            float* row = reinterpret_cast<float*>(stage0);
            const float* src = a.qraw + q * ix.dim;
            const uint32_t dim = ix.dim;
            // when the stage also holds the row as doubles (12 B per element),
            // all lanes convert in parallel and lane 0's chains read doubles:
            // 48 warp-wide conversions per query instead of 1536 single-lane
            // ones on the FP64-class pipe the reranking warps also need
            const uint32_t xd_off = (4u * dim + 15u) & ~15u;
            const bool use_xd = xd_off + 8u * dim <= 2u * (SR / 4u) * gstride;
            double* xd = reinterpret_cast<double*>(stage0 + xd_off);
            bool fin = true;
            for (uint32_t i = lane; i < dim; i += 32) {
                // L2-only load: with a pipelined upload the row may have been
                // written by a copy engine during this launch (no stale L1 line)
                const float v = __ldcg(src + i);
                fin &= isfinite(v);
                row[i] = v;
                if (use_xd) xd[i] = (double)v;
            }
            fin = __all_sync(kFull, fin);
            __syncwarp();
            qst = fin ? QVG_Q_OK : QVG_Q_NONFINITE_COORD;
            double inv_d = 0.0;
            if (lane == 0 && qst == QVG_Q_OK) {
                double acc = 0.0;
                uint32_t i = 0;
                if (use_xd) {
                    for (; i + 8 <= dim; i += 8) {
                        double v[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) v[u] = xd[i + u];
#pragma unroll
                        for (int u = 0; u < 8; ++u) acc = __fma_rn(v[u], v[u], acc);
                    }
                    for (; i < dim; ++i) acc = __fma_rn(xd[i], xd[i], acc);
                }
                for (; i + 8 <= dim; i += 8) {
                    float v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = row[i + u];
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc = __fma_rn((double)v[u], (double)v[u], acc);
                }
                for (; i < dim; ++i) acc = __fma_rn((double)row[i], (double)row[i], acc);
                const double nrm = __dsqrt_rn(acc);
                if (!(nrm > 0.0) || isinf(nrm)) qst = QVG_Q_BAD_NORM;
                else inv_d = __ddiv_rn(1.0, nrm);
            }
            qst = __shfl_sync(kFull, qst, 0);
            const float inv = __double2float_rn(__shfl_sync(kFull, inv_d, 0));
            bool yfin = true;
            float* qout = a.qn_out + q * ix.Dp;
            for (uint32_t i = lane; i < ix.Dp; i += 32) {
                const float y = (i < dim && qst == QVG_Q_OK) ? __fmul_rn(row[i], inv) : 0.0f;
                yfin &= isfinite(y);
                if (i < dim) {
                    row[i] = y;
                    if (use_xd) xd[i] = fabs((double)y);
                }
                qout[i] = y;
            }
            yfin = __all_sync(kFull, yfin);
            if (qst == QVG_Q_OK && !yfin) qst = QVG_Q_NONFINITE_CODE;
            __syncwarp();
            float tau_l = 0.0f;
            if (lane == 0 && qst == QVG_Q_OK) {
                double s = 0.0;
                uint32_t i = 0;
                if (use_xd) {
                    for (; i + 8 <= dim; i += 8) {
                        double v[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) v[u] = xd[i + u];
#pragma unroll
                        for (int u = 0; u < 8; ++u) s = __dadd_rn(s, v[u]);
                    }
                    for (; i < dim; ++i) s = __dadd_rn(s, xd[i]);
                }
                for (; i + 8 <= dim; i += 8) {
                    float v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = row[i + u];
#pragma unroll
                    for (int u = 0; u < 8; ++u) s = __dadd_rn(s, fabs((double)v[u]));
                }
                for (; i < dim; ++i) s = __dadd_rn(s, fabs((double)row[i]));
                tau_l = __double2float_rn(__ddiv_rn(s, (double)dim));
            }
            const float tau = __shfl_sync(kFull, tau_l, 0);
            for (uint32_t w = lane; w < W; w += 32) {
                uint32_t p0 = 0, p1 = 0, s0 = 0, s1 = 0;
                const uint32_t b0 = w * 64, lim = min(64u, dim - b0);
                for (uint32_t b = 0; b < lim; ++b) {
                    const float y = row[b0 + b];
                    const uint32_t pb = y > 0.0f, sb = fabsf(y) > tau;
                    if (b < 32) {
                        p0 |= pb << b;
                        s0 |= sb << b;
                    } else {
                        p1 |= pb << (b - 32);
                        s1 |= sb << (b - 32);
                    }
                }
                qc[w] = make_uint4(p0, p1, s0, s1);
            }
            if (qst != QVG_Q_OK && lane == 0 && a.flags) atomicOr(a.flags, 1u << qst);
            __syncwarp();
        } else {
            qst = a.qstatus ? a.qstatus[q] : 0;
        }
        if (qst != 0) {
            for (uint32_t i = lane; i < a.k; i += 32) {
                if (a.out_ids) a.out_ids[q * a.k + i] = kSentinel;
                if (a.out_scores) a.out_scores[q * a.k + i] = __int_as_float(0x7fc00000);
            }
            if (a.pool_ids)
                for (uint32_t i = lane; i < ef; i += 32) {
                    a.pool_ids[q * ef + i] = kSentinel;
                    a.pool_dists[q * ef + i] = kSentinel;
                }
            if (lane == 0) {
                if (a.out_count) a.out_count[q] = 0;
                if (a.out_status) a.out_status[q] = qst;
                if (a.pool_n) a.pool_n[q] = 0;
                if (a.qctr)
                    for (int i = 0; i < 8; ++i) a.qctr[q * 8 + i] = i == 7 ? (uint32_t)qst : 0u;
                if (budgeted) atomicAdd(a.susp_ctl + 2, 1u);
            }
            continue;
        }

        // ---- per-query init --------------------------------------------------
        // per-query cycle timers (QVG_VARIANT bit 16, debug; not in LEAN kernels)
        constexpr bool kTimers = !LEAN;
        const long long t_start = kTimers ? clock64() : 0;
#ifdef QVG_TAIL  // occupancy-over-time build (tools/tail_profile.py): wall-clock span per query
        unsigned long long tg0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tg0));
#endif
        if (!a.qraw && !resume)
            for (uint32_t w = lane; w < W; w += 32) qc[w] = a.qcodes[q * W + w];
        if (resume) {
        } else if (xbits) {
            uint4* xb4 = reinterpret_cast<uint4*>(xbits);
            for (uint64_t i = lane; i < a.exact_words / 4; i += 32) xb4[i] = make_uint4(0, 0, 0, 0);
            __syncwarp();
        } else {
            const uint32_t vwords = (VS * vtw) / 4u;
            for (uint32_t i = lane; i < vwords; i += 32) vis[i] = kSentinel;  // all 0xFF
        }
        const uint32_t entry = a.entry;
        if (lane == 0 && !resume) {
            if (xbits) atomicOr(xbits + (entry >> 5), 1u << (entry & 31));
            else vis_insert(entry);
        }
        uint32_t np = 0, tn = 0, tdist = 0, hint = 0;
        uint32_t na = 0;  // |A| (XA only)
        uint32_t c_exp = 0, c_tie = 0, c_eval = 0, c_drop = 0, c_slots = 0, c_maxtie = 0;
        bool overflow = false;
#ifdef QVG_TAIL
        uint32_t c_mtot = 0;  // contenders per query (diagnostics)
#endif
        uint32_t n = 1;  // rows to score in cid[0..n)
        if (lane == 0 && !resume) cid[0] = entry;
        // suspended-query state: a 64-B header of scalars, then the shared-memory
        // range [pk, qd) (pool, compacted rows, query code, tie stack, visited table)
        // budget_left: expansions left in this unit (kNoBudget: whole query).  It
        // is 0 after the loop exactly when the query was handed over: the hand-over
        // happens at the top of an iteration, before that iteration's pick could
        // end the search, and nothing decrements it after the final pick
        constexpr uint32_t kNoBudget = 0x7FFFFFFFu;
        uint32_t budget_left = kNoBudget;
        if constexpr (SUSP) {
            if (budgeted) budget_left = a.susp_budget;
            if (resume) {
                const uint4* sstate = a.susp_state + (size_t)(q - a.susp_from) * a.susp_stride16;
                const uint32_t blob16 = (susp_end - L.pk) / 16u;
                uint4* dst = reinterpret_cast<uint4*>(base + L.pk);
                for (uint32_t i = lane; i < blob16; i += 32) dst[i] = __ldcg(sstate + 4 + i);
                const uint4 h0 = __ldcg(sstate), h1 = __ldcg(sstate + 1), h2 = __ldcg(sstate + 2);
                np = h0.x, tn = h0.y, tdist = h0.z, hint = h0.w;
                n = h1.x, c_exp = h1.y, c_tie = h1.z, c_eval = h1.w;
                c_drop = lane == 0 ? h2.x : 0u, c_slots = h2.y, c_maxtie = h2.z, overflow = h2.w != 0;
            }
        }
        __syncwarp();
        uint32_t spec_u = kSentinel;  // speculatively prefetched adjacency row
        uint64_t spec_key = kInfKey;  // its key (the predicted next pick)
        uint32_t guess_idx = kSentinel;  // its index in P (kSentinel: not in P)
        uint32_t spec_rel[REL ? RELP : 1];  // relaxed: the predicted picks, spec_n of them
        uint32_t spec_n = 0;
        (void)spec_rel;
        (void)spec_n;
        uint32_t spec_v[RW];
        // relaxed: the first (up to RELP) unexpanded pool entries at/after the
        // hint, in key order -> ids[], count returned; mark = set their EXP bit
        auto first_unexpanded = [&](uint32_t* ids, bool mark, uint32_t& last) -> uint32_t {
            uint32_t cnt = 0;
            for (uint32_t b0 = hint & ~31u; b0 < np && cnt < (uint32_t)RELP; b0 += 32) {
                const uint32_t idx = b0 + lane;
                const bool un = idx < np && idx >= hint && !(pk[idx] & kExp);
                unsigned bal = __ballot_sync(kFull, un);
                while (bal && cnt < (uint32_t)RELP) {
                    const uint32_t at = b0 + __ffs(bal) - 1;
                    const uint32_t id = (uint32_t)pk[at];
#pragma unroll
                    for (int t = 0; t < (REL ? RELP : 1); ++t)
                        if ((uint32_t)t == cnt) ids[t] = id;
                    if (mark && lane == 0) pk[at] |= kExp;
                    last = at;
                    ++cnt;
                    bal &= bal - 1;
                }
            }
            return cnt;
        };
        // relaxed: slots of picked row p -> v[p*SPL, (p+1)*SPL)
        auto load_rows = [&](uint32_t* vv, const uint32_t* ids, uint32_t cnt) {
#pragma unroll
            for (int p = 0; p < (REL ? RELP : 1); ++p) {
                const bool have = (uint32_t)p < cnt && lane * SPL < ix.RS;
                const uint32_t* row = ix.adj + (size_t)(have ? ids[p] : 0u) * ix.RS;
                if (SPL == 1) {
                    vv[p * SPL] = have ? __ldg(row + lane) : kSentinel;
                } else {
                    const uint2 t = have ? __ldg(reinterpret_cast<const uint2*>(row) + lane)
                                         : make_uint2(kSentinel, kSentinel);
                    vv[p * SPL] = t.x;
                    vv[p * SPL + SPL - 1] = t.y;
                }
            }
        };
        (void)first_unexpanded;
        (void)load_rows;

        // ---- best-first loop (iteration 0 scores the entry point) --------------
        QVG_PH(long long ph_issue = 0, ph_wait = 0, ph_dist = 0, ph_merge = 0, ph_pick = 0, ph_tma = 0;)
        for (;;) {  // (re-entered only when a hand-over finds the FIFO full)
        for (;;) {
            QVG_PH(long long tp0 = clock64();)
            if constexpr (SUSP) {
                if (__builtin_expect(budget_left == 0, 0)) break;  // end of this unit (below)
            }
            c_eval += n;
            // (a) TMA-gather the code rows (double-buffered halves of SR rows)
            const uint32_t nsub = __umulhi(n + SR - 1, sr_m);  // (n + SR - 1) / SR
            if (nsub > 0) issue(0, min(n, SR), 0);
            if (nsub > 1) issue(SR, min(n - SR, SR), 1, false);  // (same fence covers both halves)
            QVG_PH(ph_tma += clock64() - tp0;)
            // speculative prefetch: adjacency row of the current best unexpanded
            // entry (the next pick unless this row inserts a better one)
            if constexpr (REL) {
                uint32_t last = 0;
                spec_n = first_unexpanded(spec_rel, false, last);
                load_rows(spec_v, spec_rel, spec_n);
            } else {
                uint32_t guess = kSentinel;
                spec_key = kInfKey;
                guess_idx = kSentinel;
                for (uint32_t b0 = hint & ~31u; b0 < np; b0 += 32) {
                    const uint32_t idx = b0 + lane;
                    const uint64_t pv = idx < np ? pk[idx] : kExp;
                    const bool un = idx >= hint && !(pv & kExp);
                    const unsigned bal = __ballot_sync(kFull, un);
                    if (bal) {
                        const uint32_t src = __ffs(bal) - 1;
                        guess_idx = b0 + src;
                        spec_key = __shfl_sync(kFull, pv, src);  // (exp bit clear)
                        guess = (uint32_t)spec_key;
                        break;
                    }
                }
                if (guess == kSentinel && tn > 0) guess = tie[tn - 1];
                spec_u = guess;
                if (guess != kSentinel) {
                    const uint32_t* row = ix.adj + (size_t)guess * ix.RS;
                    if (lane * RW < ix.RS) {
                        if (RW == 1) {
                            spec_v[0] = __ldg(row + lane);
                        } else if (RW == 2) {
                            const uint2 t = __ldg(reinterpret_cast<const uint2*>(row) + lane);
                            spec_v[0] = t.x;
                            spec_v[RW - 1] = t.y;
                        } else {
                            const uint4 t = __ldg(reinterpret_cast<const uint4*>(row) + lane);
                            spec_v[0] = t.x;
                            spec_v[1 % RW] = t.y;
                            spec_v[2 % RW] = t.z;
                            spec_v[3 % RW] = t.w;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < RW; ++j) spec_v[j] = kSentinel;
                    }
                }
            }
            QVG_PH(long long tp1 = clock64(); ph_issue += tp1 - tp0;)
            // (b) SM2 distances lane-per-row from the stage; contenders -> ctd/crp
            const uint64_t worst = np == ef ? ordk(pk[ef - 1]) : kInfKey;
            const uint64_t worst_a = (XA && na == xa) ? pa[xa - 1] : kInfKey;
            uint32_t m = 0, ma = 0;
            // contender test + row-order compaction of one scored row per lane
            auto emit = [&](bool valid, uint32_t d, uint32_t id) {
                const uint64_t key = mkkey(d, id);
                bool c = valid && key < worst;
                uint32_t rp = 0;
                if (c) {
                    rp = lower_bound_key(pk, np, key);
                    if (rp < np && ordk(pk[rp]) == key) {
                        c = false;  // already pooled (visited-table miss)
                        ++c_drop;
                    }
                }
                const unsigned bal = __ballot_sync(kFull, c);
                if (c) {
                    const uint32_t pos = m + __popc(bal & lt_mask);
                    ctd[pos] = key;
                    crp[pos] = rp;
                }
                m += __popc(bal);
                if (ctd_prefetch && !REL && bal) {
                    // the smallest contender is always admitted (no smaller
                    // earlier contender, and it beats max(P)); if it also beats
                    // the predicted pick it becomes the next pick: fetch its
                    // adjacency row now, under the remaining distance work
                    const uint32_t dmin = __reduce_min_sync(kFull, c ? d : ~0u);
                    const uint32_t imin = __reduce_min_sync(kFull, (c && d == dmin) ? id : ~0u);
                    const uint64_t kmin = mkkey(dmin, imin);
                    if (kmin < spec_key) {
                        spec_key = kmin;
                        spec_u = imin;
                        const uint32_t* row = ix.adj + (size_t)imin * ix.RS;
                        if (lane * RW < ix.RS) {
                            if (RW == 1) {
                                spec_v[0] = __ldg(row + lane);
                            } else if (RW == 2) {
                                const uint2 t = __ldg(reinterpret_cast<const uint2*>(row) + lane);
                                spec_v[0] = t.x;
                                spec_v[RW - 1] = t.y;
                            } else {
                                const uint4 t = __ldg(reinterpret_cast<const uint4*>(row) + lane);
                                spec_v[0] = t.x;
                                spec_v[1 % RW] = t.y;
                                spec_v[2 % RW] = t.z;
                                spec_v[3 % RW] = t.w;
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < RW; ++j) spec_v[j] = kSentinel;
                        }
                    }
                }
                if constexpr (XA) {
                    // above max(P) (key == max(P) is P's own entry) and below
                    // max(A); a key already in A is a visited-table miss
                    bool ac = valid && np == ef && key > worst && key < worst_a;
                    if (ac) {
                        const uint32_t r = lower_bound_key(pa, na, key);
                        ac = !(r < na && pa[r] == key);
                    }
                    const unsigned ba = __ballot_sync(kFull, ac);
                    if (ac) acd[ma + __popc(ba & lt_mask)] = key;
                    ma += __popc(ba);
                }
            };
            // (a paired pass — wait for both halves, then score 2 rows per lane —
            // measured slower than overlapping half-0 scoring with the arrival of
            // half 1: cfg2 3.95 vs 3.03 ms; removed)
            for (uint32_t k = 0; k < nsub; ++k) {
                const uint32_t h = k & 1u;
                QVG_PH(long long tw0 = clock64();)
                mbar_wait(&bars[h], (phs >> h) & 1u);
                phs ^= 1u << h;
                QVG_PH(ph_wait += clock64() - tw0;)
                const uint32_t r0 = k * SR;
                const uint32_t cnt = min(n - r0, SR);
                const uint4* st = reinterpret_cast<const uint4*>(stage0 + h * stage_delta);
                // LPR lanes per row (wide rows leave a half with < 32 rows): part
                // p of row r reads chunks (lane + LPR*i) mod W, i.e. offsets
                // p, p+LPR, ... from the row's rotation LPR*r — every chunk once,
                // and the 8 lanes of an LDS.128 phase hit distinct bank quads
                for (uint32_t i0 = 0; LPR == 1u && i0 < cnt; i0 += 32) {
                    const uint32_t j = i0 + lane;
                    const bool valid = j < cnt;
                    uint32_t d = 0;
                    if (valid) {
                        const uint4* rowp = st + ((j >> 2) * gstride + (j & 3u) * rowb) / 16u;
                        // (row_sm2 here measured 0.8 % slower at W = 12)
                        Sm2Acc acc;
                        if constexpr (WC > 0 && ((16 * WC) & 127) == 64) {
                            // rows 64 B past a 128-B boundary: a rotation by
                            // (lane >> 1) & 3 puts an 8-lane LDS.128 phase on 8
                            // distinct bank quads and lets the first W - 3 chunks
                            // use constant offsets (no wrap)
                            const uint32_t r4 = (lane >> 1) & 3u;
                            const uint4* qr = qc + r4;
                            const uint4* rr = rowp + r4;
#pragma unroll
                            for (int c = 0; c < WC - 3; ++c) acc.add(qr[c], rr[c]);
#pragma unroll
                            for (int c = WC - 3; c < WC; ++c) {
                                uint32_t cc = (uint32_t)c + r4;
                                cc = cc >= (uint32_t)WC ? cc - WC : cc;
                                acc.add(qc[cc], rowp[cc]);
                            }
                        } else if constexpr (WC == 6) {
                            // 96-B rows: row r starts on bank quad 6r mod 8 = {0,6,4,2} x 2,
                            // so starting rows r and r + 4 of an LDS.128 phase one chunk
                            // apart puts the 8 lanes on 8 distinct quads; five chunks of
                            // every lane need no wrap
                            const uint32_t r1 = (lane >> 2) & 1u;
                            const uint4* qr = qc + r1;
                            const uint4* rr = rowp + r1;
#pragma unroll
                            for (int c = 0; c < 5; ++c) acc.add(qr[c], rr[c]);
                            const uint32_t cl = r1 ? 0u : 5u;
                            acc.add(qc[cl], rowp[cl]);
                        } else {
                            uint32_t cc = rot;
#pragma unroll 4
                            for (uint32_t c = 0; c < W; ++c) {
                                acc.add(qc[cc], rowp[cc]);
                                cc = cc + 1u == W ? 0u : cc + 1u;
                            }
                        }
                        d = acc.total();
                    }
                    emit(valid, d, valid ? cid[r0 + j] : kSentinel);
                }
                for (uint32_t i0 = 0; LPR > 1u && i0 < cnt; i0 += 32u >> lpr_log) {
                    const uint32_t j = i0 + (lane >> lpr_log);
                    const uint32_t part = lane & (LPR - 1u);
                    const bool valid = j < cnt;
                    uint32_t d = 0;
                    if (valid) {
                        const uint4* rowp = st + ((j >> 2) * gstride + (j & 3u) * rowb) / 16u;
                        // (cfg 3 3.95 -> 3.80 ms, cfg 4 7.13 -> 6.86 ms: profiles/r3_smfix_*)
                        if constexpr (WC == 24 || WC == 48) {
                            if (LPR == (uint32_t)(WC / 12)) d = row_sm2_fixed<WC, WC / 12>(qc, rowp, lane);
                            else d = row_sm2(qc, rowp, W, rot, part, LPR);
                        } else {
                            d = row_sm2(qc, rowp, W, rot, part, LPR);
                        }
                    }
                    for (uint32_t o = 1; o < LPR; o <<= 1) d += __shfl_xor_sync(kFull, d, o);
                    const bool lead = valid && part == 0;
                    emit(lead, d, lead ? cid[r0 + j] : kSentinel);
                }
                if (k + 2 < nsub) issue((k + 2) * SR, min(n - (k + 2) * SR, SR), h);
            }
            __syncwarp();
            QVG_PH(long long tp2 = clock64(); ph_dist += tp2 - tp1;)
            // (L2 prefetch of the predicted next pick's neighbour rows here was
            // measured: TMA bulk prefetch +25% time, LSU line prefetch +0.7%)

            if constexpr (REL) {
                // relaxed: a node reached through two picked rows (past a lossy
                // visited-table collision) can be a contender twice; keep the
                // first copy (later copies become +inf and sort past the rest)
                if (m > 1) {
                    bool dup[RW];
#pragma unroll
                    for (int i = 0; i < RW; ++i) dup[i] = false;
                    uint64_t yv[RW];
#pragma unroll
                    for (int i = 0; i < RW; ++i) yv[i] = lane + 32u * i < m ? ctd[lane + 32u * i] : kInfKey;
                    for (uint32_t j = 0; j < m; ++j) {
                        const uint64_t yj = ctd[j];
#pragma unroll
                        for (int i = 0; i < RW; ++i) dup[i] |= (yj == yv[i]) & (j < lane + 32u * i);
                    }
                    __syncwarp();
#pragma unroll
                    for (int i = 0; i < RW; ++i)
                        if (dup[i] && lane + 32u * i < m) ctd[lane + 32u * i] = kInfKey;
                    __syncwarp();
                }
            }
            uint32_t ins_lo = kSentinel;  // P index of this step's smallest contender
#ifdef QVG_TAIL
            c_mtot += m;
#endif
            if (m > 0) {
                // (c) contender ranks (key order) and prefix counts (row order)
                uint64_t y[RW];
                uint32_t rk[RW], pre[RW], rp[RW];
#pragma unroll
                for (int i = 0; i < RW; ++i) {
                    const uint32_t idx = lane + 32u * i;
                    y[i] = idx < m ? ctd[idx] : kInfKey;
                    rp[i] = idx < m ? crp[idx] : 0u;
                    rk[i] = 0;
                    pre[i] = 0;
                }
                for (uint32_t j = 0; j < m; ++j) {
                    const uint64_t yj = ctd[j];
#pragma unroll
                    for (int i = 0; i < RW; ++i) {
                        const uint32_t lt = yj < y[i];
                        rk[i] += lt;
                        pre[i] += lt & (j < lane + 32u * i);
                    }
                }
                uint32_t mu = m;  // distinct contenders (relaxed: duplicates are +inf)
                if constexpr (REL) {
                    uint32_t fin = 0;
#pragma unroll
                    for (int i = 0; i < RW; ++i)
                        fin += __popc(__ballot_sync(kFull, lane + 32u * i < m && y[i] != kInfKey));
                    mu = fin;
                }
#pragma unroll
                for (int i = 0; i < RW; ++i)
                    if (lane + 32u * i < m && (!REL || y[i] != kInfKey)) csrp[rk[i]] = rp[i];
                __syncwarp();

                // (d) in-place merge: P entries at index >= lo shift right by
                // #{contenders with rank-in-P <= index}; walk chunks backwards so
                // no entry is overwritten before it is read
                const uint32_t lo = mu ? csrp[0] : np;
                ins_lo = lo;
                const uint32_t total = np + mu;
                // few contenders (the usual case): their ranks padded to 8 with
                // +inf, two broadcast 16-B loads per chunk and eight compares
                // instead of a dependent binary search per pool entry
                const bool few = mu <= 8u;
                if (few && lane >= mu && lane < 8u) csrp[lane] = 0xFFFFFFFFu;
                __syncwarp();
                // two 32-entry chunks per round (both read before either is
                // written: entries only move right), half the warp barriers: ef 256
                // 8.53 -> 8.34 ms, ef 128 +0.7 %, ef 64 unchanged.  Not in the
                // fused-prologue instantiations (there its mere presence cost 0.5 %
                // at ef 64, profiles/r3_merge2_ab.txt) nor in the R = 32 kernels
                // (cfg 1 -3.5 %, profiles/r3_w6_ab.txt)
                if ((GEO || ONE) && !PRO && lo < np && few) {
                    const uint4 r0 = reinterpret_cast<const uint4*>(csrp)[0];
                    const uint4 r1 = reinterpret_cast<const uint4*>(csrp)[1];
                    auto dest = [&](uint32_t idx) {
                        return idx + (r0.x <= idx) + (r0.y <= idx) + (r0.z <= idx) + (r0.w <= idx) +
                               (r1.x <= idx) + (r1.y <= idx) + (r1.z <= idx) + (r1.w <= idx);
                    };
                    for (int cb = (int)((np - 1) & ~31u); cb >= (int)(lo & ~31u); cb -= 64) {
                        const uint32_t ia = (uint32_t)cb + lane;
                        const uint32_t ib = ia - 32u;  // (wraps below chunk 0: then >= np)
                        const bool ma = ia < np && ia >= lo, mb = ib < np && ib >= lo;
                        uint64_t pa = 0, pb = 0;
                        if (ma) pa = pk[ia];
                        if (mb) pb = pk[ib];
                        const uint32_t na2 = dest(ia), nb2 = dest(ib);
                        __syncwarp();
                        if (ma) {
                            if (na2 < ef) pk[na2] = pa;
                            else if (!REL) evk[na2 - ef] = pa;
                        }
                        if (mb) {
                            if (nb2 < ef) pk[nb2] = pb;
                            else if (!REL) evk[nb2 - ef] = pb;
                        }
                        __syncwarp();
                    }
                } else if (lo < np) {
                    for (int cb = (int)((np - 1) & ~31u); cb >= (int)(lo & ~31u); cb -= 32) {
                        const uint32_t idx = (uint32_t)cb + lane;
                        const bool mv = idx < np && idx >= lo;
                        uint64_t p = 0;
                        uint32_t npos = 0;
                        if (few) {
                            const uint4 r0 = reinterpret_cast<const uint4*>(csrp)[0];
                            const uint4 r1 = reinterpret_cast<const uint4*>(csrp)[1];
                            if (mv) p = pk[idx];
                            npos = idx + (r0.x <= idx) + (r0.y <= idx) + (r0.z <= idx) + (r0.w <= idx) +
                                   (r1.x <= idx) + (r1.y <= idx) + (r1.z <= idx) + (r1.w <= idx);
                        } else if (mv) {
                            p = pk[idx];
                            npos = idx + upper_bound_u32(csrp, mu, idx);
                        }
                        __syncwarp();
                        if (mv) {
                            if (npos < ef) pk[npos] = p;
                            else if (!REL) evk[npos - ef] = p;  // exp bit set = not a tie candidate
                        }
                        __syncwarp();
                    }
                }
#pragma unroll
                for (int i = 0; i < RW; ++i) {
                    if (lane + 32u * i < m && (!REL || y[i] != kInfKey)) {
                        const uint32_t npos = rk[i] + rp[i];
                        if (npos < ef) pk[npos] = y[i];
                        else if (!REL) evk[npos - ef] = (rp[i] + pre[i]) < ef ? y[i] : (y[i] | kExp);
                    }
                }
                __syncwarp();
                if (lo < hint) hint = lo;

                // (e) tie stack maintenance (none in the relaxed variant)
                if (!REL && total > ef) {
                    const uint32_t wd = kdist(pk[ef - 1]);
                    if (tn == 0 || wd < tdist) {
                        tn = 0;
                        tdist = wd;
                    }
                    const uint32_t nev = total - ef;
                    uint32_t adds = 0;
                    for (uint32_t e0 = 0; e0 < nev; e0 += 32) {
                        const uint32_t e = e0 + lane;
                        uint32_t idv = kSentinel;
                        if (e < nev) {
                            const uint64_t kk = evk[e];
                            if (!(kk & kExp) && kdist(kk) == wd) idv = (uint32_t)kk;
                        }
                        const unsigned b = __ballot_sync(kFull, idv != kSentinel);
                        if (idv != kSentinel) stg[adds + __popc(b & lt_mask)] = idv;
                        adds += __popc(b);
                    }
                    if (adds) {
                        __syncwarp();
                        const uint32_t room = tie_cap - tn;
                        if (adds > room) overflow = true;
                        const uint32_t put = adds < room ? adds : room;
                        // smallest key on top of the stack
                        for (uint32_t r = lane; r < put; r += 32) tie[tn + put - 1 - r] = stg[r];
                        tn += put;
                        if (tn > c_maxtie) c_maxtie = tn;
                    }
                    if constexpr (XA) {  // keys leaving P (rejected or evicted) -> A candidates
                        for (uint32_t e = lane; e < nev; e += 32) acd[ma + e] = ordk(evk[e]);
                        ma += nev;
                    }
                }
                np = total < ef ? total : ef;
                __syncwarp();
            }
            if constexpr (XA) {
                if (ma > 0) {
                    // merge the step's candidates into A (ascending, capped at xa):
                    // candidate i (key order) lands at rankA(i) + i; A[idx] moves
                    // right by #{candidates with rankA <= idx}
                    __syncwarp();
                    for (uint32_t i = lane; i < ma; i += 32) {
                        const uint64_t x = acd[i];
                        uint32_t rx = 0;
                        for (uint32_t j = 0; j < ma; ++j) rx += acd[j] < x;
                        axk[rx] = x;
                        axr[rx] = lower_bound_key(pa, na, x);
                    }
                    __syncwarp();
                    const uint32_t lo = axr[0];
                    if (lo < na) {
                        for (int cb = (int)((na - 1) & ~31u); cb >= (int)(lo & ~31u); cb -= 32) {
                            const uint32_t idx = (uint32_t)cb + lane;
                            const bool mv = idx < na && idx >= lo;
                            uint64_t p = 0;
                            uint32_t npos = 0;
                            if (mv) {
                                p = pa[idx];
                                npos = idx + upper_bound_u32(axr, ma, idx);
                            }
                            __syncwarp();
                            if (mv && npos < xa) pa[npos] = p;
                            __syncwarp();
                        }
                    }
                    for (uint32_t i = lane; i < ma; i += 32) {
                        const uint32_t npos = axr[i] + i;
                        if (npos < xa) pa[npos] = axk[i];
                    }
                    na = na + ma < xa ? na + ma : xa;
                    __syncwarp();
                }
            }

            QVG_PH(long long tp3 = clock64(); ph_merge += tp3 - tp2;)
            // (f) pick: first unexpanded pool entry at or after the hint, else
            // the top of the tie stack (every live tie entry has dist ==
            // worst(P).dist, so the reference's stop test, search.cpp:48, does
            // not fire for it)
            uint32_t u = kSentinel;
            uint32_t v[RW];
            if constexpr (REL) {
                // relaxed: take the first RELP unexpanded entries; stop when none
                uint32_t picks[RELP], last = 0;
                const uint32_t cnt = first_unexpanded(picks, true, last);
                if (cnt == 0) break;
                hint = last + 1;
                c_exp += cnt;
                bool same = cnt == spec_n;
#pragma unroll
                for (int t = 0; t < RELP; ++t) same &= (uint32_t)t >= cnt || picks[t] == spec_rel[t];
                if (same) {
#pragma unroll
                    for (int j = 0; j < RW; ++j) v[j] = spec_v[j];
                } else {
                    load_rows(v, picks, cnt);
                }
                __syncwarp();  // EXP marks visible before the next scan
            }
            // No scan: entries of P before this step's first insertion point
            // are unchanged, so the first unexpanded entry at/after the hint is
            // the predicted pick (first unexpanded after the last pick, found by
            // the speculative scan) unless the smallest new contender — always
            // admitted, at index ins_lo — comes first.
            if (!REL) {
                const uint32_t pick = ins_lo < guess_idx ? ins_lo : guess_idx;
                if (pick != kSentinel) {
                    // spec_key already is this entry's key: the speculative scan
                    // set it to the predicted pick and the contender prefetch
                    // lowered it to the smallest admitted contender if smaller
                    u = (uint32_t)spec_key;
                    __syncwarp();
                    if (lane == 0) pk[pick] = spec_key | kExp;
                    hint = pick + 1;
                }
            }
            if (!REL && u == kSentinel) {
                hint = np;
                if (tn == 0) break;
                u = tie[tn - 1];
                --tn;
                ++c_tie;
                if (!LEAN && a.exp_out) spec_key = mkkey(tdist, u);  // (expanded-node list)
            }
            // builder searches: the expanded nodes in expansion order — Vamana's
            // visited set V, the RobustPrune candidates of the build's second
            // pass (never in LEAN kernels)
            if (!LEAN && !REL && a.exp_out && lane == 0 && c_exp < a.exp_cap)
                a.exp_out[q * a.exp_cap + c_exp] = ordk(spec_key);
            if (!REL) ++c_exp;
            if (SUSP) --budget_left;

            // (g) adjacency row (stored order): the speculative prefetch when it
            // guessed right, else a fresh vectorised load
            if (REL) {
                // loaded above
            } else if (u == spec_u) {
#pragma unroll
                for (int j = 0; j < RW; ++j) v[j] = spec_v[j];
            } else {
                const uint32_t* row = ix.adj + (size_t)u * ix.RS;
                if (lane * RW < ix.RS) {
                    if (RW == 1) {
                        v[0] = __ldg(row + lane);
                    } else if (RW == 2) {
                        const uint2 t = __ldg(reinterpret_cast<const uint2*>(row) + lane);
                        v[0] = t.x;
                        v[RW - 1] = t.y;
                    } else {
                        const uint4 t = __ldg(reinterpret_cast<const uint4*>(row) + lane);
                        v[0] = t.x;
                        v[1 % RW] = t.y;
                        v[2 % RW] = t.z;
                        v[3 % RW] = t.w;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < RW; ++j) v[j] = kSentinel;
                }
            }
            // (h) visited filter + compaction (slot s = lane*RW + j; rows carry
            // no duplicate ids, see adj_relayout_kernel)
            bool keep[RW];
#pragma unroll
            for (int j = 0; j < RW; ++j) {
                if (REL && j > 0 && j % SPL == 0) __syncwarp();  // next picked row sees this one's marks
                const uint32_t id = v[j];
                bool k2 = id != kSentinel;
                if (k2) {
                    if (xbits) {
                        const uint32_t bit = 1u << (id & 31);
                        k2 = (atomicOr(xbits + (id >> 5), bit) & bit) == 0;
                    } else {
                        k2 = vis_insert(id);
                    }
                }
                keep[j] = k2;
            }
            uint32_t pos = 0, slots = 0;
            n = 0;
#pragma unroll
            for (int j = 0; j < RW; ++j) {
                const unsigned b = __ballot_sync(kFull, keep[j]);
                slots += __popc(__ballot_sync(kFull, v[j] != kSentinel));
                pos += __popc(b & lt_mask);
                n += __popc(b);
            }
            c_slots += slots;
            __syncwarp();  // previous readers of cid are done
#pragma unroll
            for (int j = 0; j < RW; ++j)
                if (keep[j]) cid[pos++] = v[j];
            __syncwarp();
            QVG_PH(ph_pick += clock64() - tp3;)
        }
        if (!(SUSP && budget_left == 0)) break;  // the search ended
        // end of a unit (the loop stopped at the top of an iteration): save the
        // state and hand the query to the FIFO; a full FIFO lets this warp finish it
        {
            uint32_t slot = 0;
            if (lane == 0) slot = atomicAdd(a.susp_ctl, 1u);
            slot = __shfl_sync(kFull, slot, 0);
            if (slot < a.susp_cap) {
                uint4* sstate = a.susp_state + (size_t)(q - a.susp_from) * a.susp_stride16;
                const uint32_t blob16 = (susp_end - L.pk) / 16u;
                const uint4* src = reinterpret_cast<const uint4*>(base + L.pk);
                for (uint32_t i = lane; i < blob16; i += 32) __stcg(sstate + 4 + i, src[i]);
                for (int off = 16; off > 0; off >>= 1) c_drop += __shfl_xor_sync(kFull, c_drop, off);
                if (lane == 0) {
                    __stcg(sstate, make_uint4(np, tn, tdist, hint));
                    __stcg(sstate + 1, make_uint4(n, c_exp, c_tie, c_eval));
                    __stcg(sstate + 2, make_uint4(c_drop, c_slots, c_maxtie, overflow ? 1u : 0u));
                }
                __threadfence();
                __syncwarp();
                if (lane == 0)
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.susp_list + slot), "r"((uint32_t)q + 1u) : "memory");
                break;
            }
            budget_left = kNoBudget;
        }
        }

        if (SUSP && budget_left == 0) continue;
        // ---- outputs ------------------------------------------------------------
        const long long t_search = kTimers ? clock64() : 0;
        for (int off = 16; off > 0; off >>= 1) c_drop += __shfl_xor_sync(kFull, c_drop, off);
        if (a.pool_ids) {
            for (uint32_t i = lane; i < ef; i += 32) {
                a.pool_ids[q * ef + i] = i < np ? (uint32_t)pk[i] : kSentinel;
                a.pool_dists[q * ef + i] = i < np ? kdist(pk[i]) : kSentinel;
            }
            if (lane == 0) a.pool_n[q] = np;
        }
        if (!LEAN && a.exp_out && lane == 0) a.exp_n[q] = min(c_exp, a.exp_cap);
        const int32_t qstatus = overflow ? QVG_Q_TIE_OVERFLOW : QVG_Q_OK;
        if (lane == 0 && overflow && a.flags) atomicOr(a.flags, 1u << QVG_Q_TIE_OVERFLOW);
        if (lane == 0) {
            if (a.out_status) a.out_status[q] = qstatus;
            if (a.qctr) {
                uint32_t* c = a.qctr + q * 8;
                c[0] = c_exp;
                c[1] = c_tie;
                c[2] = c_eval;
                c[3] = c_drop;
                c[4] = c_slots;
                c[5] = np;
                c[6] = c_maxtie;
                c[7] = (uint32_t)qstatus;
            }
        }
        QVG_PH(if (lane == 0 && a.qctr) {
            uint32_t* c = a.qctr + q * 8;  // phases build only: cycles >> 4
            c[2] = (uint32_t)(ph_tma >> 4);
            c[3] = (uint32_t)((ph_issue - ph_tma) >> 4);
            c[4] = (uint32_t)(ph_wait >> 4);
            c[5] = (uint32_t)((ph_dist - ph_wait) >> 4);
            c[6] = (uint32_t)(ph_merge >> 4);
            c[7] = (uint32_t)(ph_pick >> 4);
        })
        if (a.do_rerank) {
            // rerank the NR best scored keys pk[0, NR) (P, then A when XA)
            const uint32_t NR = min(np + na, a.depth);
            if (lane == 0 && a.qctr && NR != np) a.qctr[q * 8 + 5] = NR;  // rows reranked
            // rerank: one lane per pool entry, 4 sequential double chains
            const float* qv = a.qn + q * ix.Dp;
            __syncwarp();
            // (R = 32 / W = 6 geometry, D <= 384: the rows are short and mostly in L2;
            // one lane streaming each row measured 4.6 % faster than the TMA slices
            // (e2e +8.7 %): profiles/r5_cfg1_ldg_rerank.txt, r5_ldg6_ab.txt)
            constexpr bool kLdgRerank = WC == 6;
            if (!kLdgRerank && (LEAN || SL)) {
                // TMA column slices: round t stages slice (t % nsl) of the 32 pool
                // rows of group (t / nsl) — 4 rows x SL floats per gather4 —
                // into a stage half; lane r owns row 32g + r and advances its 4
                // chains slice by slice, i.e. in ascending element order, which
                // keeps every chain's rounding sequence identical to dot_f32.
                const uint32_t dim = GEO ? 768u : ix.dim;  // GEO is dispatched for D = 768 only
                const uint32_t main4 = dim & ~3u;
                const uint32_t nsl = (dim + SL - 1) / SL;
                // t / nsl == __umulhi(t, nsl_m) for nsl > 1 (nsl == 1: 2^32 does
                // not fit; D <= SL takes the plain path)
                const uint32_t nsl_m = 0xFFFFFFFFu / nsl + 1u;
                const uint32_t rounds = ((NR + 31) / 32) * nsl;
                const uint32_t cgs = (16u * SL + 127u) & ~127u;  // bytes per 4-row group
                auto rr_issue = [&](uint32_t t) {
                    const uint32_t g = nsl == 1u ? t : __umulhi(t, nsl_m), s = t - g * nsl, h = t & 1u;
                    const uint32_t rows = min(32u, NR - 32u * g);
                    const uint32_t ng4 = (rows + 3u) >> 2;
                    // the query slice rides in the same transaction (16-B multiple,
                    // clipped to the padded row so the last query never overreads)
                    const uint32_t qbytes = 4u * min(SL, ix.Dp - s * SL);
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        mbar_expect_tx(&bars[h], ng4 * 16u * SL + qbytes);
                        bulk_row(qsl + h * 48u, qv + s * SL, qbytes, &bars[h]);
                    }
                    __syncwarp();
                    if (lane < ng4) {
                        const uint32_t j = 32u * g + 4u * lane;
                        const uint32_t i0 = (uint32_t)pk[j];
                        const uint32_t i1 = 4u * lane + 1u < rows ? (uint32_t)pk[j + 1] : i0;
                        const uint32_t i2 = 4u * lane + 2u < rows ? (uint32_t)pk[j + 2] : i0;
                        const uint32_t i3 = 4u * lane + 3u < rows ? (uint32_t)pk[j + 3] : i0;
                        tma_gather4_col(stage0 + h * stage_delta + lane * cgs, &cmap, s * SL, i0, i1,
                                        i2, i3, &bars[h]);
                    }
                };
                // (a bulk L2 prefetch of all NR rows here measured neutral-to-worse)
                if (rounds > 0) rr_issue(0);
                if (rounds > 1) rr_issue(1);
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                for (uint32_t t = 0; t < rounds; ++t) {
                    const uint32_t g = nsl == 1u ? t : __umulhi(t, nsl_m), s = t - g * nsl, h = t & 1u;
                    // the round's query slice -> registers in one batch of
                    // independent loads, issued before the stage wait (qn is
                    // L2-resident; L1 is mostly carved out for shared memory)
                    constexpr uint32_t kMaxSL4 = 12;  // rerank_slice() caps SL at 48
                    const uint32_t i0 = s * SL;
                    const uint32_t lim = min(SL, dim - i0);
                    const float4* qr = reinterpret_cast<const float4*>(qsl) + h * (kMaxSL4);
                    mbar_wait(&bars[h], (phs >> h) & 1u);
                    phs ^= 1u << h;
                    if (s == 0) s0 = s1 = s2 = s3 = 0.0;
                    const uint32_t row = 32u * g + lane;
                    if constexpr (GEO) {
                        // D = 768: every slice is a full 48 floats of 4-element
                        // groups.  The float -> double conversions share the
                        // FP64 pipe with the chains: the query's are done once
                        // per warp (two per lane) instead of 48 per lane.
                        if (lane < 24) {
                            const float2 f = reinterpret_cast<const float2*>(qr)[lane];
                            reinterpret_cast<double2*>(qd)[lane] = make_double2((double)f.x, (double)f.y);
                        }
                        __syncwarp();
                        if (row < NR) {
                            const float4* rp = reinterpret_cast<const float4*>(
                                stage0 + h * stage_delta + (lane >> 2) * cgs + (lane & 3u) * SL * 4u);
                            const double2* q2 = reinterpret_cast<const double2*>(qd);
#pragma unroll
                            for (uint32_t u = 0; u < kMaxSL4; ++u) {
                                const float4 v = rp[u];
                                const double2 qa = q2[2 * u], qb = q2[2 * u + 1];
                                s0 = __fma_rn(qa.x, (double)v.x, s0);
                                s1 = __fma_rn(qa.y, (double)v.y, s1);
                                s2 = __fma_rn(qb.x, (double)v.z, s2);
                                s3 = __fma_rn(qb.y, (double)v.w, s3);
                            }
                            if (s == nsl - 1)
                                sc[row] = __double2float_rn(__dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3)));
                        }
                        __syncwarp();  // qd is rewritten by the next round
                    } else {
                        // the query slice as doubles, converted once per warp
                        // (the slice buffer holds 48 floats; values past `lim`
                        // are never used)
                        if (lane < 24) {
                            const float2 f = reinterpret_cast<const float2*>(qr)[lane];
                            reinterpret_cast<double2*>(qd)[lane] = make_double2((double)f.x, (double)f.y);
                        }
                        __syncwarp();
                        const double2* q2 = reinterpret_cast<const double2*>(qd);
                        if ((ONE || PRO) && row < NR && lim == 4u * kMaxSL4 && i0 + 4u * kMaxSL4 <= main4) {
                            // a full 48-float slice of 4-element groups (every slice when
                            // D is a multiple of 48): no per-group bounds checks.  cfg 3
                            // 3.79 -> 3.61 ms, cfg 1 e2e +2.5 %; left out of the R = 32
                            // device-query kernels, where it measured -0.7 %
                            // (profiles/r4_rrfull_*_ab.txt)
                            const float4* rp = reinterpret_cast<const float4*>(
                                stage0 + h * stage_delta + (lane >> 2) * cgs + (lane & 3u) * SL * 4u);
#pragma unroll
                            for (uint32_t u = 0; u < kMaxSL4; ++u) {
                                const float4 v = rp[u];
                                const double2 qa = q2[2 * u], qb = q2[2 * u + 1];
                                s0 = __fma_rn(qa.x, (double)v.x, s0);
                                s1 = __fma_rn(qa.y, (double)v.y, s1);
                                s2 = __fma_rn(qb.x, (double)v.z, s2);
                                s3 = __fma_rn(qb.y, (double)v.w, s3);
                            }
                            if (s == nsl - 1)
                                sc[row] = __double2float_rn(__dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3)));
                        } else if (row < NR) {
                            const float4* rp = reinterpret_cast<const float4*>(
                                stage0 + h * stage_delta + (lane >> 2) * cgs + (lane & 3u) * SL * 4u);
#pragma unroll
                            for (uint32_t u = 0; u < kMaxSL4; ++u) {
                                if (4u * u >= lim) break;
                                const uint32_t i = i0 + 4u * u;
                                const float4 v = rp[u];
                                const double2 qa = q2[2 * u], qb = q2[2 * u + 1];
                                const double qx = qa.x, qy = qa.y, qz = qb.x, qw = qb.y;
                                if (i + 4 <= main4) {
                                    s0 = __fma_rn(qx, (double)v.x, s0);
                                    s1 = __fma_rn(qy, (double)v.y, s1);
                                    s2 = __fma_rn(qz, (double)v.z, s2);
                                    s3 = __fma_rn(qw, (double)v.w, s3);
                                } else {  // tail elements >= 4*floor(D/4) all go to s0
                                    if (i < dim) s0 = __fma_rn(qx, (double)v.x, s0);
                                    if (i + 1 < dim) s0 = __fma_rn(qy, (double)v.y, s0);
                                    if (i + 2 < dim) s0 = __fma_rn(qz, (double)v.z, s0);
                                }
                            }
                            if (s == nsl - 1)
                                sc[row] = __double2float_rn(__dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3)));
                        }
                        __syncwarp();  // qd is rewritten by the next round
                    }
                    if (t + 2 < rounds) rr_issue(t + 2);
                }
            } else if (kLdgRerank && (ix.dim % 48u) == 0u) {
                // one lane per pool entry streaming its row from global, 48 elements
                // at a time; the query chunk is converted to doubles once per warp
                // (two conversions per lane) and read back by 16-B broadcast loads
                for (uint32_t idx = lane; idx < NR; idx += 32)
                    prefetch_l2(ix.cold + (size_t)(uint32_t)pk[idx] * ix.Dp, ix.Dp * 4u);
                const double2* q2 = reinterpret_cast<const double2*>(qd);
                for (uint32_t g0 = 0; g0 < NR; g0 += 32) {
                    const uint32_t idx = g0 + lane;
                    const float4* r4 = reinterpret_cast<const float4*>(
                        ix.cold + (size_t)(uint32_t)pk[idx < NR ? idx : g0] * ix.Dp);
                    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                    for (uint32_t c0 = 0; c0 < ix.dim; c0 += 48) {
                        __syncwarp();  // the previous chunk's doubles are consumed
                        if (lane < 24) {
                            const float2 f = __ldg(reinterpret_cast<const float2*>(qv + c0) + lane);
                            reinterpret_cast<double2*>(qd)[lane] = make_double2((double)f.x, (double)f.y);
                        }
                        __syncwarp();
#pragma unroll
                        for (int hb = 0; hb < 2; ++hb) {
                            float4 b[6];
#pragma unroll
                            for (int u = 0; u < 6; ++u) b[u] = __ldg(r4 + c0 / 4 + hb * 6 + u);
#pragma unroll
                            for (int u = 0; u < 6; ++u) {
                                const double2 qa = q2[2 * (hb * 6 + u)], qb = q2[2 * (hb * 6 + u) + 1];
                                s0 = __fma_rn(qa.x, (double)b[u].x, s0);
                                s1 = __fma_rn(qa.y, (double)b[u].y, s1);
                                s2 = __fma_rn(qb.x, (double)b[u].z, s2);
                                s3 = __fma_rn(qb.y, (double)b[u].w, s3);
                            }
                        }
                    }
                    if (idx < NR)
                        sc[idx] = __double2float_rn(__dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3)));
                }
            } else {
                // fallback: one lane per pool entry streaming its row from global
                if (!(a.variant & 1u))
                    for (uint32_t idx = lane; idx < NR; idx += 32)
                        prefetch_l2(ix.cold + (size_t)(uint32_t)pk[idx] * ix.Dp, ix.Dp * 4u);
                for (uint32_t idx = lane; idx < NR; idx += 32) {
                    const uint32_t id = (uint32_t)pk[idx];
                    const float* row = ix.cold + (size_t)id * ix.Dp;
                    sc[idx] = (a.variant & 4u) ? dot4_exact<true>(qv, row, ix.dim)
                                               : dot4_exact<false>(qv, row, ix.dim);
                }
            }
            __syncwarp();
            const long long t_dots = kTimers ? clock64() : 0;
            if (kTimers && (a.variant & 16u) && lane == 0 && a.qctr) {
                a.qctr[q * 8 + 0] = (uint32_t)((t_search - t_start) >> 4);
                a.qctr[q * 8 + 1] = (uint32_t)((t_dots - t_search) >> 4);
            }
            // rank by (score desc, id asc) and emit the first k
            for (uint32_t idx = lane; idx < NR; idx += 32) {
                const float si = sc[idx];
                const uint32_t ii = (uint32_t)pk[idx];
                uint32_t rank = 0;
                for (uint32_t j = 0; j < NR; ++j) {
                    const float sj = sc[j];
                    const uint32_t ij = (uint32_t)pk[j];
                    rank += (sj > si) | ((sj == si) & (ij < ii));
                }
                if (rank < a.k) {
                    a.out_ids[q * a.k + rank] = ii;
                    a.out_scores[q * a.k + rank] = si;
                }
            }
            for (uint32_t r = NR + lane; r < a.k; r += 32) {
                a.out_ids[q * a.k + r] = kSentinel;
                a.out_scores[q * a.k + r] = __int_as_float(0x7fc00000);
            }
            if (lane == 0 && a.out_count) a.out_count[q] = NR < a.k ? NR : a.k;
#ifndef QVG_PHASES  // slot 2 carries the TMA-issue time in the phases build
            if (kTimers && (a.variant & 16u) && lane == 0 && a.qctr)
                a.qctr[q * 8 + 2] = (uint32_t)((clock64() - t_dots) >> 4);
#endif
        }
#ifdef QVG_TAIL
        if (lane == 0 && a.qctr) {
            unsigned long long tg1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tg1));
            a.qctr[q * 8 + 0] = (uint32_t)tg0;
            a.qctr[q * 8 + 1] = (uint32_t)tg1;
            a.qctr[q * 8 + 2] = (uint32_t)gwarp;
            a.qctr[q * 8 + 3] = blockIdx.x;
            a.qctr[q * 8 + 4] = c_mtot;
        }
#endif
        if (SUSP && a.susp_ctl && q >= a.susp_from && lane == 0) {  // (the FIFO servers exit on this count)
            __threadfence();
            atomicAdd(a.susp_ctl + 2, 1u);
        }
        __syncwarp();
    }
}

// one thread per pair, plain loop over W chunks
__global__ void pair_distance_kernel(const DevIndex ix, const uint4* __restrict__ qchunks,
                                     const uint32_t* __restrict__ ids, uint64_t npairs,
                                     uint32_t* __restrict__ out) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= npairs) return;
    const uint4* a = qchunks + t * ix.W;
    const uint4* b = ix.codes + (size_t)ids[t] * ix.W;
    uint32_t d = 0;
    for (uint32_t w = 0; w < ix.W; ++w) d += sm2_chunk(a[w], b[w]);
    out[t] = d;
}

// LEAN instantiations compile out the exact-visited and LDG-rerank paths
// (QVG_LEAN=0: never, for A/B)
bool geo_allowed(const SearchLaunch& a) {
    static const bool env_ok = [] {
        const char* e = getenv("QVG_LEAN");
        return !(e && e[0] == '0');
    }();
    return env_ok && !a.exact_bits && !(a.variant & 8u) && !a.tie_spill && !a.qmap && !a.exp_out;
}

uint32_t pow2ceil(uint32_t x) {
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

uint32_t stage_half_bytes() {
    static uint32_t v = [] {
        const char* e = getenv("QVG_STAGE_HALF_BYTES");
        const long x = e ? atol(e) : 6144;
        return (uint32_t)(x < 64 ? 64 : x);
    }();
    return v;
}

struct Plan {
    void* fn;
    uint32_t rw, SR, warp_bytes, block_bytes;
    bool geo = false;               // the headline-geometry instantiation (GEO)
    bool one = false;               // one block per SM (ONE) without the GEO layout
    uint32_t wpb = kWarpsPerBlock;  // warps per block (GEO: one block per SM, as many as fit)
};

// split rows over lanes when a stage half holds at most this many rows
// (QVG_SPLIT_MAX_ROWS; 0 = never).  cfg3 (16 rows/half): 6.38 -> 5.62 ms;
// cfg4 (8 rows/half): 18.8 -> 9.9 ms; cfg1/cfg2 (32 rows/half): not split.
uint32_t split_max_rows() {
    static uint32_t v = [] {
        const char* e = getenv("QVG_SPLIT_MAX_ROWS");
        return e ? (uint32_t)atol(e) : 16u;
    }();
    return v;
}

template <int RW>
void* pick_kernel(bool xa, bool split) {
    if (xa) return split ? (void*)search_kernel<RW, true, true> : (void*)search_kernel<RW, true, false>;
    return split ? (void*)search_kernel<RW, false, true> : (void*)search_kernel<RW, false, false>;
}

// relaxed variant: RW = capacity of `relax` picked rows
void* pick_relaxed(uint32_t rw, uint32_t relax, bool split) {
    if (relax == 2 && rw == 2) return split ? (void*)search_kernel<2, false, true, 2> : (void*)search_kernel<2, false, false, 2>;
    if (relax == 2 && rw == 4) return split ? (void*)search_kernel<4, false, true, 2> : (void*)search_kernel<4, false, false, 2>;
    if (relax == 4 && rw == 4) return split ? (void*)search_kernel<4, false, true, 4> : (void*)search_kernel<4, false, false, 4>;
    return nullptr;
}

}  // namespace

// row-slot capacity per lane of the relaxed variant (0 = unsupported geometry)
uint32_t relaxed_rw(uint32_t R, uint32_t relax) {
    const uint32_t per = (R + 31) / 32;  // slots per lane of one row
    if (relax == 2 && per == 1) return 2;
    if (relax == 2 && per == 2) return 4;
    if (relax == 4 && per == 1) return 4;
    return 0;
}

namespace {

// QVG_ONEBLK=0: the wide-row kernels keep 2-warp blocks (A/B measurement)
bool one_block_ok() {
    static const bool ok = [] {
        const char* e = getenv("QVG_ONEBLK");
        return !(e && e[0] == '0');
    }();
    return ok;
}

Plan make_plan(const DevIndex& ix, uint32_t ef, uint32_t vis_log2, uint32_t tie_cap,
               uint32_t xa, uint32_t relax = 0, bool geo_ok = true, bool fused = true) {
    Plan p;
    p.rw = relax ? relaxed_rw(ix.R, relax) : pow2ceil((ix.R + 31) / 32);
    p.SR = stage_rows_for(ix.W, p.rw * 32, stage_half_bytes());
    const bool split = p.SR * 2u <= 32u && p.SR <= split_max_rows();
    if (relax) p.fn = pick_relaxed(p.rw, relax, split);
    else if (geo_ok && p.rw == 2 && !xa && !split && ix.W == 12 && ix.dim == 768 && p.SR == 32 &&
             stage_half_bytes() == 6144 && vis_tag_bytes(ix.n, vis_log2) <= 2u)
    {
        p.fn = fused ? (void*)search_kernel<2, false, false, 0, 12, true, true>
                     : (void*)search_kernel<2, false, false, 0, 12, true, false>;
        p.geo = true;
    }
    else if (p.rw == 2 && !xa && !split && ix.W == 12)
        p.fn = !geo_ok ? (void*)search_kernel<2, false, false, 0, 12>
             : fused   ? (void*)search_kernel<2, false, false, 0, 12, false, true, true>
                       : (void*)search_kernel<2, false, false, 0, 12, false, false, true>;
    else if (p.rw == 1 && !xa && !split && ix.W == 6)
        p.fn = !geo_ok ? (void*)search_kernel<1, false, false, 0, 6>
             : fused   ? (void*)search_kernel<1, false, false, 0, 6, false, true, true>
                       : (void*)search_kernel<1, false, false, 0, 6, false, false, true>;
    // (wide-row LEAN instantiations measured 3.6 % slower at W = 48: not used)
    else if (p.rw == 2 && !xa && split && ix.W == 24) {
        p.one = one_block_ok();
        p.fn = p.one ? (void*)search_kernel<2, false, true, 0, 24, false, true, false, true>
                     : (void*)search_kernel<2, false, true, 0, 24>;
    } else if (p.rw == 2 && !xa && split && ix.W == 48) {
        p.one = one_block_ok();
        p.fn = p.one ? (void*)search_kernel<2, false, true, 0, 48, false, true, false, true>
                     : (void*)search_kernel<2, false, true, 0, 48>;
    }
    else if (p.rw == 1) p.fn = pick_kernel<1>(xa != 0, split);
    else if (p.rw == 2) p.fn = pick_kernel<2>(xa != 0, split);
    else p.fn = pick_kernel<4>(xa != 0, split);
    const SmemLayout L = smem_layout((ef + xa + 31) & ~31u, p.rw * 32, ix.W, tie_cap,
                                     (1u << vis_log2) * (p.geo ? 2u : vis_tag_bytes(ix.n, vis_log2)),
                                     p.SR, xa, true, p.geo);
    p.warp_bytes = L.total;
    if (p.geo || p.one) {
        // one block per SM with as many warps as its shared memory holds (the
        // 1 KB per-block reservation is paid once instead of per 2-warp block)
        static const uint32_t sm_smem = [] {
            int d = 0, v = 0, r = 0;
            cudaGetDevice(&d);
            cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, d);
            cudaDeviceGetAttribute(&r, cudaDevAttrReservedSharedMemoryPerBlock, d);
            return (uint32_t)(v > r ? v - r : 0);
        }();
        static const uint32_t blk_smem = [] {
            int d = 0, v = 0;
            cudaGetDevice(&d);
            cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
            return (uint32_t)v;
        }();
        uint32_t w = sm_smem / p.warp_bytes;
        if (w * p.warp_bytes > blk_smem) w = blk_smem / p.warp_bytes;
        if (w > (uint32_t)kGeoMaxWarps) w = kGeoMaxWarps;
        p.wpb = w < 1 ? 1 : w;
    }
    p.block_bytes = p.warp_bytes * p.wpb;
    return p;
}

}  // namespace

// 2-D row-gather descriptor: `cols` elements per row, `n` rows, box {box_cols, 1}
static bool encode_rows_map(CUtensorMap* map, CUtensorMapDataType dt, uint32_t esize,
                            const void* base, uint64_t cols, uint64_t n, uint32_t box_cols) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult qres;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qres) !=
                cudaSuccess ||
            !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)n};
    cuuint64_t gstride[1] = {(cuuint64_t)(cols * esize)};
    cuuint32_t box[2] = {box_cols, 1};
    cuuint32_t es[2] = {1, 1};
    const CUresult r = encode(map, dt, 2, const_cast<void*>(base), gdim, gstride, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_code_tmap(CUtensorMap* map, const void* codes, uint64_t n, uint32_t W) {
    if (2 * W > 256) return false;  // TMA box dimension limit
    return encode_rows_map(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 8, codes, 2 * W, n, 2 * W);
}

// cold-store slice width (floats) for the rerank: 8 four-row groups of a
// stage half, each 128-B aligned; 0 = no TMA rerank
static uint32_t rerank_slice(uint32_t half_bytes) {
    uint32_t sl = (half_bytes / 8u) / 16u;  // floats per row slice
    sl &= ~7u;                                // 16*sl multiple of 128
    if (sl > 48) sl = 48;                     // query slice held in 12 float4 registers
    return sl >= 8 ? sl : 0u;
}

// opt-in dynamic shared memory per block on this device
static uint32_t max_dyn_smem(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    return (uint32_t)v;
}

// Raise a kernel's dynamic-smem cap to the device maximum (monotone, so a
// cached plan of any size stays launchable whatever was planned after it).
static bool allow_max_smem(void* fn, int device) {
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)max_dyn_smem(device)) == cudaSuccess;
}

uint32_t search_stage_bytes(const DevIndex& ix) {
    const uint32_t rw = pow2ceil((ix.R + 31) / 32);
    const uint32_t sr = stage_rows_for(ix.W, rw * 32, stage_half_bytes());
    return 2u * (sr / 4u) * group_stride(ix.W);
}

uint32_t auto_visited_log2(const DevIndex& ix, uint32_t ef, uint32_t tie_cap, int device,
                           uint32_t xa, uint32_t relax) {
    uint32_t min_log = 7;  // 128 slots
    while ((1u << min_log) < ((ef + xa + 31u) & ~31u)) ++min_log;  // rerank scores alias it
    uint32_t best_log = min_log;
    int best_blocks = -1;
    for (uint32_t lg = min_log; lg <= 15 || lg == min_log; ++lg) {
        const Plan p = make_plan(ix, ef, lg, tie_cap, xa, relax);
        if (p.block_bytes > max_dyn_smem(device) || !allow_max_smem(p.fn, device)) {
            break;
        }
        int blocks = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, p.fn, p.wpb * 32,
                                                          p.block_bytes) != cudaSuccess) {
            cudaGetLastError();
            break;
        }
        blocks *= (int)p.wpb;         // resident warps
        if (blocks >= best_blocks) {  // ties go to the larger table
            best_blocks = blocks;
            best_log = lg;
        }
    }
    (void)device;
    return best_log;
}

qvg_status plan_search(const SearchLaunch& a, int device, uint64_t* grid_out, PlanInfo* info) {
    const uint32_t xa = extra_depth(a.ef, a.depth);
    if ((1u << a.vis_log2) < ((a.ef + xa + 31u) & ~31u)) {
        set_error("search: visited_slots must be >= ef + extra rerank depth (rounded to 32)");
        return QVG_INVALID_ARGUMENT;
    }
    const Plan p = make_plan(a.ix, a.ef, a.vis_log2, a.tie_cap, xa, a.relax, geo_allowed(a),
                             a.qraw != nullptr);
    if (p.block_bytes > max_dyn_smem(device)) {
        set_error("search: per-warp shared memory too large (reduce visited_slots / tie_capacity)");
        return QVG_INVALID_ARGUMENT;
    }
    if (!allow_max_smem(p.fn, device)) return cuda_status(cudaGetLastError(), "cudaFuncSetAttribute");
    cudaError_t e;
    int per_sm = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p.fn, p.wpb * 32,
                                                      p.block_bytes);
    if (e != cudaSuccess) return cuda_status(e, "occupancy(search)");
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (per_sm < 1) {
        set_error("search: per-warp shared memory too large (reduce visited_slots / tie_capacity)");
        return QVG_INVALID_ARGUMENT;
    }
    uint64_t want = (a.nq + p.wpb - 1) / p.wpb;
    uint64_t grid = (uint64_t)per_sm * sms;
    if (want < grid) grid = want;
    if (grid < 1) grid = 1;
    *grid_out = grid;
    if (info) {
        info->warps_per_block = p.wpb;
        info->smem_per_block = p.block_bytes;
        info->resident_warps_per_sm = (uint32_t)per_sm * p.wpb;
        info->sms = (uint32_t)sms;
        if ((p.geo || p.one) && !xa && !a.relax) {  // pool .. visited table: a suspended query's state
            const SmemLayout L =
                smem_layout((a.ef + 31) & ~31u, p.rw * 32, a.ix.W, a.tie_cap,
                            (1u << a.vis_log2) * (p.geo ? 2u : vis_tag_bytes(a.ix.n, a.vis_log2)),
                            p.SR, 0, true, p.geo);
            info->susp_blob_bytes = (p.geo ? L.qd : L.qsl) - L.pk;
        }
    }
    return QVG_OK;
}

qvg_status launch_search(const SearchLaunch& a, const CUtensorMap* tmap, uint64_t grid,
                         cudaStream_t s) {
    const Plan p0 = make_plan(a.ix, a.ef, a.vis_log2, a.tie_cap, extra_depth(a.ef, a.depth), a.relax, false);
    alignas(64) CUtensorMap dummy;
    memset(&dummy, 0, sizeof(dummy));
    const CUtensorMap* m = tmap ? tmap : &dummy;
    int use_tmap = tmap != nullptr;
    // cold-store slice map (per launch: the slice width follows the stage size)
    alignas(64) CUtensorMap cmap;
    uint32_t SL = 0;
    if (a.do_rerank && !(a.variant & 8u)) {
        const uint32_t half = (p0.SR / 4u) * group_stride(a.ix.W);
        SL = rerank_slice(half);
        if (SL && !encode_rows_map(&cmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.ix.cold, a.ix.Dp,
                                   a.ix.n, SL))
            SL = 0;
    }
    if (!SL) memset(&cmap, 0, sizeof(cmap));
    // the headline-geometry kernel assumes both tensor maps
    const Plan p = make_plan(a.ix, a.ef, a.vis_log2, a.tie_cap, extra_depth(a.ef, a.depth), a.relax,
                             geo_allowed(a) && use_tmap && (!a.do_rerank || SL != 0),
                             a.qraw != nullptr);
    void* args[] = {(void*)m,     (void*)&cmap,     (void*)&a, (void*)&p.warp_bytes,
                    (void*)&p.SR, (void*)&use_tmap, (void*)&SL};
    cudaError_t e = cudaLaunchKernel(p.fn, dim3((unsigned)grid), dim3(p.wpb * 32),
                                     args, p.block_bytes, s);
    if (e != cudaSuccess) return cuda_status(e, "launch(search)");
    return QVG_OK;
}

void launch_pair_distance(const DevIndex& ix, const uint4* qchunks, const uint32_t* ids,
                          uint64_t npairs, uint32_t* out, cudaStream_t s) {
    if (!npairs) return;
    pair_distance_kernel<<<(unsigned)((npairs + 255) / 256), 256, 0, s>>>(ix, qchunks, ids,
                                                                          npairs, out);
}

}  // namespace qvg

// Latency mode: one CTA of kCoopWarps warps per query (small batches).
//
// The throughput kernel (search.cu) gives each query one warp, which is the
// right trade when thousands of queries keep every SM busy; with a handful of
// queries the GPU is idle and a query's latency is its serial chain of ~80
// expansions.  Here the per-expansion work that parallelises is spread over
// the CTA, and the leader's bookkeeping is taken off the memory round trip:
//   * three helper warps TMA-gather and score a third of the expansion's rows
//     each (<= 24 of 64) in one round trip, into a shared distance array, and
//     copy the adjacency row of their slice's smallest row in the background;
//   * the leader warp runs the unchanged state machine of search.cu — the same
//     contender test, prefix admission, in-place merge, tie stack, pick,
//     visited table and compaction, on the same distances in the same row
//     order — so pools, ids and scores are identical (search.cpp:27-81).  It
//     takes the next pick right after the contender test (min of the predicted
//     pick and the smallest contender, which is always admitted), publishes its
//     surviving neighbours, and merges the contenders while the helpers already
//     gather the next rows;
//   * the rerank spreads the pool over all lanes, four lanes per row: lane c
//     accumulates chain c (elements i = c mod 4, ascending) and lane 0 of the
//     group folds the tail and combines (s0 + s1) + (s2 + s3) — the reference's
//     dot_f32 order (vec_math.hpp:13-26), hence bit-identical scores.
// Not used with exact-visited bitmaps, a rerank depth above ef, or the fused
// encode prologue (the throughput kernel covers those).
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "bq_device.cuh"
#include "qvg_internal.cuh"
#include "search_common.cuh"

namespace qvg {

namespace {

// per-phase cycle counters (variant build: build.py --variant cphases -DQVG_COOP_PHASES)
#ifdef QVG_COOP_PHASES
#define QVG_CP(...) __VA_ARGS__
// per-step event timestamps (SM clock cycles) of the block serving query 0:
// [step][event]; events: 0 step start (leader), 1 leader phase C done, 2 S1
// passed (leader), 3 combine done, 4 adjacency row ready, 5 filter done,
// 8 helper 0 step start, 9 gather landed, 10 scored, 11 bar 1 passed,
// 12 contender test done
__device__ unsigned long long g_coop_trace[1024][16];
__device__ __forceinline__ void coop_ev(uint64_t q, uint32_t iter_q, int ev) {
    if (q != 0 || iter_q >= 1024 || (threadIdx.x & 31) != 0) return;
    g_coop_trace[iter_q][ev] = (unsigned long long)clock64();  // one SM: one clock
}
#else
#define QVG_CP(...)
#endif

__host__ __device__ inline uint32_t coop_vis_log2(uint32_t lg) { return lg < 12u ? lg : 12u; }

struct CoopLayout {
    uint32_t bars, stages, stage_bytes, pk, ctd, evk, crp, csrp, cid, stg, dsh, spec, smin, scop, hctd,
        hcrp, hcnt, hdrop, qc, tie, vis, qn, ctl, total;
};

// block carve-up; SRW = rows per warp (multiple of 4)
__host__ __device__ inline CoopLayout coop_layout(uint32_t EFM, uint32_t RM, uint32_t W,
                                                  uint32_t tie_cap, uint32_t vis_slots,
                                                  uint32_t Dp, uint32_t SRW) {
    CoopLayout L;
    uint32_t o = 0;
    auto take = [&](uint32_t bytes, uint32_t align) {
        o = (o + align - 1) & ~(align - 1);
        const uint32_t at = o;
        o += bytes;
        return at;
    };
    L.bars = take(8 * 2 * kCoopWarps, 16);         // gather + adjacency mbarrier per helper
    L.stage_bytes = (SRW / 4) * group_stride(W);  // multiple of 128
    L.stages = take((kCoopWarps - 1) * L.stage_bytes, 128);  // helpers only
    L.pk = take(8 * EFM, 16);
    L.ctd = take(8 * RM, 16);
    L.evk = L.ctd;
    L.crp = take(4 * RM, 16);
    L.csrp = take(4 * RM, 16);
    L.cid = take(4 * RM, 16);
    L.stg = L.crp;
    L.dsh = take(4 * RM, 16);     // row distances, row order
    // per helper: the adjacency row of its slice's smallest (dist, id) row,
    // bulk-copied in the background (the next pick whenever a contender beats
    // the predicted one), and that row's key
    L.spec = take((kCoopWarps - 1) * 4 * RM, 16);
    L.smin = take((kCoopWarps - 1) * 8, 16);
    L.scop = take((kCoopWarps - 1) * 8, 16);  // key whose adjacency row was copied
    // per helper: its slice's contenders (keys, ranks in P, row order), count,
    // and visited-table-miss drops
    L.hctd = take((kCoopWarps - 1) * 8 * SRW, 16);
    L.hcrp = take((kCoopWarps - 1) * 4 * SRW, 16);
    L.hcnt = take((kCoopWarps - 1) * 4, 16);
    L.hdrop = take((kCoopWarps - 1) * 4, 16);
    L.qc = take(16 * W, 16);
    L.tie = take(4 * tie_cap, 16);
    L.vis = take(4 * vis_slots, 16);  // rerank scores alias it (vis_slots >= EFM)
    L.qn = take(4 * Dp, 16);          // normalised query (rerank)
    L.ctl = take(32, 16);             // query index (u64), row count, done flag, np, guess key
    L.total = (o + 127u) & ~127u;
    return L;
}

template <int RW>
__global__ void __launch_bounds__(kCoopWarps * 32) coop_kernel(
    const __grid_constant__ CUtensorMap tmap, const SearchLaunch a, const uint32_t SRW) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr uint32_t RM = RW * 32;
    const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const DevIndex ix = a.ix;
    const uint32_t W = ix.W;
    const uint32_t rowb = 16u * W;
    const uint32_t gstride = group_stride(W);
    // the block's own visited table: full ids, at most 4096 slots (the
    // per-warp kernel's table size may be chosen for byte tags)
    const uint32_t vlg = coop_vis_log2(a.vis_log2);
    const uint32_t VS = 1u << vlg;
    const uint32_t ef = a.ef;
    const uint32_t EFM = (ef + 31u) & ~31u;
    const CoopLayout L = coop_layout(EFM, RM, W, a.tie_cap, VS, ix.Dp, SRW);
    unsigned char* base = smem_raw;
    // helper h = w - 1 gathers and scores rows [h*SRW, (h+1)*SRW) of an expansion
    const uint32_t h = w - 1;  // (meaningless for the leader, w == 0)
    uint64_t* bar = reinterpret_cast<uint64_t*>(base + L.bars) + (w ? h : 0);
    uint64_t* abar = reinterpret_cast<uint64_t*>(base + L.bars) + kCoopWarps;  // [helper]
    unsigned char* const stage = base + L.stages + (w ? h : 0) * L.stage_bytes;
    uint64_t* pk = reinterpret_cast<uint64_t*>(base + L.pk);
    uint64_t* ctd = reinterpret_cast<uint64_t*>(base + L.ctd);
    uint64_t* evk = reinterpret_cast<uint64_t*>(base + L.evk);
    uint32_t* crp = reinterpret_cast<uint32_t*>(base + L.crp);
    uint32_t* csrp = reinterpret_cast<uint32_t*>(base + L.csrp);
    uint32_t* cid = reinterpret_cast<uint32_t*>(base + L.cid);
    uint32_t* stg = reinterpret_cast<uint32_t*>(base + L.stg);
    uint32_t* dsh = reinterpret_cast<uint32_t*>(base + L.dsh);
    uint32_t* adjw = reinterpret_cast<uint32_t*>(base + L.spec);  // [helper][RM]
    uint64_t* smin = reinterpret_cast<uint64_t*>(base + L.smin);  // [helper]
    uint64_t* scop = reinterpret_cast<uint64_t*>(base + L.scop);  // [helper]
    uint64_t* hctd = reinterpret_cast<uint64_t*>(base + L.hctd);  // [helper][SRW]
    uint32_t* hcrp = reinterpret_cast<uint32_t*>(base + L.hcrp);  // [helper][SRW]
    uint32_t* hcnt = reinterpret_cast<uint32_t*>(base + L.hcnt);  // [helper]
    uint32_t* hdrop = reinterpret_cast<uint32_t*>(base + L.hdrop);  // [helper]
    uint4* qc = reinterpret_cast<uint4*>(base + L.qc);
    uint32_t* tie = reinterpret_cast<uint32_t*>(base + L.tie);
    uint32_t* vis = reinterpret_cast<uint32_t*>(base + L.vis);
    float* sc = reinterpret_cast<float*>(base + L.vis);
    float* qn = reinterpret_cast<float*>(base + L.qn);
    unsigned long long* ctl_q = reinterpret_cast<unsigned long long*>(base + L.ctl);
    volatile uint32_t* ctl_n = reinterpret_cast<volatile uint32_t*>(base + L.ctl + 8);
    volatile uint32_t* ctl_done = reinterpret_cast<volatile uint32_t*>(base + L.ctl + 12);
    // pool size published by the leader for the helpers' contender tests
    volatile uint32_t& np_sh = *reinterpret_cast<volatile uint32_t*>(base + L.ctl + 16);
    // the predicted pick's key, published with it
    volatile uint64_t& gkey_sh = *reinterpret_cast<volatile uint64_t*>(base + L.ctl + 24);

    if (w > 0 && lane == 0) {
        mbar_init(bar);
        mbar_init(abar + h);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t phase = 0;
    uint32_t iter = 0;  // expansions issued by this block (adjacency mbarrier parity)
    // lanes per row for this warp's slice (SRW rows): largest 2^k with 2^k*SRW <= 32
    uint32_t lpr_log = 0;
    while ((SRW << (lpr_log + 1)) <= 32u) ++lpr_log;
    const uint32_t LPR = 1u << lpr_log;
    const uint32_t rot = lane % W;
    __syncthreads();

    for (;;) {
        if (tid == 0) *ctl_q = atomicAdd(a.counter, 1ull);
        __syncthreads();
        const uint64_t q = *ctl_q;
        __syncthreads();
        if (q >= a.nq) break;
        const int32_t qst = a.qstatus ? a.qstatus[q] : 0;
        if (qst != 0) {  // block-uniform
            if (w == 0) {
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
                }
            }
            continue;
        }

        // ---- per-query init ----------------------------------------------------
        for (uint32_t i = tid; i < W; i += blockDim.x) qc[i] = a.qcodes[q * W + i];
        for (uint32_t i = tid; i < VS; i += blockDim.x) vis[i] = kSentinel;
        for (uint32_t i = tid; i < ix.Dp; i += blockDim.x) qn[i] = a.qn[q * ix.Dp + i];
        const uint32_t entry = a.entry;
        __syncthreads();
        if (tid == 0) {
            vis[vhash(entry, vlg)] = entry;
            cid[0] = entry;
            *ctl_n = 1;
            *ctl_done = 0;
        }
        // leader state (meaningful in warp 0 only)
        uint32_t np = 0, tn = 0, tdist = 0, hint = 0;
        uint32_t c_exp = 0, c_tie = 0, c_eval = 0, c_drop = 0, c_slots = 0, c_maxtie = 0;
        bool overflow = false;
        uint32_t spec_u = kSentinel;
        uint32_t spec_v[RW];
#pragma unroll
        for (int j = 0; j < RW; ++j) spec_v[j] = kSentinel;
        __syncthreads();

        // ---- best-first loop ------------------------------------------------------
        // Iteration i: the helpers gather and score the rows of expansion i
        // (phase A) while the leader finishes expansion i-1's bookkeeping —
        // rank / merge / tie stack / expanded mark, then the speculative scan
        // for the next pick (phase C).  Once the leader signals the pool final
        // (named barrier 1), each helper runs the contender test of its rows
        // against it and keeps its contenders in row order, their smallest key,
        // and a background copy of that node's adjacency row.  After the block
        // barrier the leader concatenates the slices, takes the next pick —
        // min(predicted pick, smallest contender: always admitted), or the top
        // of the tie stack — and compacts its surviving neighbours (phase B);
        // the merge of these contenders is left for phase C of the next
        // iteration, where it overlaps the next gather.  Same state machine and
        // the same order of every decision as search.cu (search.cpp:27-81).
        uint32_t guess_idx = kSentinel;  // predicted pick's index in P
        uint64_t spec_key = kInfKey;     // its key (then lowered to the pick's)
        uint32_t pend_m = 0;             // contenders of the last expansion, to merge
        bool pend_pick = false;          // the last pick came from P: mark it expanded
        uint32_t h_drop = 0;             // helper: visited-table misses dropped
        QVG_CP(uint32_t it_q = 0;)
        for (;;) {
            QVG_CP(coop_ev(q, it_q, w == 0 ? 0 : (w == 1 ? 8 : 15));)
            const uint32_t n = *ctl_n;
            if (w > 0) {
                // ---- phase A (helpers): gather + score this helper's slice
                const uint32_t r0 = h * SRW;
                const uint32_t cnt = n > r0 ? min(SRW, n - r0) : 0u;
                uint64_t rmin = kInfKey;  // the slice's smallest scored key
                if (cnt) {
                    const uint32_t ng = (cnt + 3u) >> 2;
                    TMA_WAR_FENCE();
                    __syncwarp();
                    if (lane == 0) mbar_expect_tx(bar, ng * 4u * rowb);
                    __syncwarp();
                    for (uint32_t g = lane; g < ng; g += 32) {
                        const uint32_t j = r0 + 4u * g;
                        const uint32_t i0 = cid[j];
                        const uint32_t i1 = 4u * g + 1u < cnt ? cid[j + 1] : i0;
                        const uint32_t i2 = 4u * g + 2u < cnt ? cid[j + 2] : i0;
                        const uint32_t i3 = 4u * g + 3u < cnt ? cid[j + 3] : i0;
                        dev::tma_gather4(stage + g * gstride, &tmap, 0, i0, i1, i2, i3, bar);
                    }
                    mbar_wait(bar, phase);
                    phase ^= 1u;
                    QVG_CP(if (w == 1) coop_ev(q, it_q, 9);)
                    const uint4* st = reinterpret_cast<const uint4*>(stage);
                    const uint32_t part = lane & (LPR - 1u);
                    for (uint32_t j0 = 0; j0 < cnt; j0 += 32u >> lpr_log) {
                        const uint32_t j = j0 + (lane >> lpr_log);
                        uint32_t d = 0;
                        if (j < cnt) {
                            const uint4* rowp = st + ((j >> 2) * gstride + (j & 3u) * rowb) / 16u;
                            // (wide rows: compile-time code width and lanes per row)
                            if (W == 24u && LPR == 2u) d = row_sm2_fixed<24, 2>(qc, rowp, lane);
                            else if (W == 48u && LPR == 2u) d = row_sm2_fixed<48, 2>(qc, rowp, lane);
                            else if (W == 12u && LPR == 2u) d = row_sm2_fixed_alt<12, 2>(qc, rowp, lane);
                            else d = row_sm2(qc, rowp, W, rot, part, LPR);
                        }
                        for (uint32_t o = 1; o < LPR; o <<= 1) d += __shfl_xor_sync(kFull, d, o);
                        const bool lead = j < cnt && part == 0;
                        if (lead) dsh[r0 + j] = d;
                        const uint32_t id = lead ? cid[r0 + j] : ~0u;
                        const uint32_t dm = __reduce_min_sync(kFull, lead ? d : ~0u);
                        const uint32_t im = __reduce_min_sync(kFull, (lead && d == dm) ? id : ~0u);
                        if (dm != ~0u && mkkey(dm, im) < rmin) rmin = mkkey(dm, im);
                    }
                }
                QVG_CP(if (w == 1) coop_ev(q, it_q, 10);)
                // background copy of the adjacency row of the slice's smallest
                // row, issued before the contender test: whenever the next pick
                // is a contender that beats the prediction it is the smallest
                // contender, almost always the smallest row of its slice.  One
                // copy per iteration keeps the mbarrier parity = iter & 1.
                if (lane == 0) {
                    if (iter > 0) mbar_wait(abar + h, (iter - 1) & 1u);  // buffer / barrier free
                    scop[h] = rmin;
                    const uint32_t src = rmin != kInfKey ? (uint32_t)rmin : a.entry;
                    mbar_expect_tx(abar + h, 4u * ix.RS);
                    bulk_row(adjw + h * RM, ix.adj + (size_t)src * ix.RS, 4u * ix.RS, abar + h);
                }
                __syncwarp();
                // contender test of the slice against the final pool
                asm volatile("bar.sync 1, %0;" ::"r"(kCoopWarps * 32) : "memory");
                QVG_CP(if (w == 1) coop_ev(q, it_q, 11);)
                const uint64_t worst = np_sh == ef ? ordk(pk[ef - 1]) : kInfKey;
                const uint32_t npv = np_sh;
                uint32_t m = 0;
                uint64_t kmin = kInfKey;
                for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
                    const uint32_t jr = i0 + lane;
                    const bool valid = jr < cnt;
                    const uint64_t key = valid ? mkkey(dsh[r0 + jr], cid[r0 + jr]) : kInfKey;
                    bool c = valid && key < worst;
                    uint32_t rp = 0;
                    if (c) {
                        rp = lower_bound_key(pk, npv, key);
                        if (rp < npv && ordk(pk[rp]) == key) {
                            c = false;  // already pooled (visited-table miss)
                            ++h_drop;
                        }
                    }
                    const unsigned bal = __ballot_sync(kFull, c);
                    if (c) {
                        const uint32_t pos = m + __popc(bal & lt_mask);
                        hctd[h * SRW + pos] = key;
                        hcrp[h * SRW + pos] = rp;
                    }
                    m += __popc(bal);
                    const uint32_t dm = __reduce_min_sync(kFull, c ? kdist(key) : ~0u);
                    const uint32_t im = __reduce_min_sync(kFull, (c && kdist(key) == dm) ? (uint32_t)key : ~0u);
                    if (dm != ~0u && mkkey(dm, im) < kmin) kmin = mkkey(dm, im);
                }
                if (lane == 0) {
                    hcnt[h] = m;
                    smin[h] = kmin;  // the slice's smallest contender
                }
                QVG_CP(if (w == 1) coop_ev(q, it_q, 12);)
            } else {
                // ---- phase C (leader) of the previous expansion
                uint32_t ins_lo = kSentinel;
                if (pend_m > 0) {
                    const uint32_t m = pend_m;
                    {  // the helpers' contenders of the last expansion, in row order
                        uint32_t off[kCoopWarps - 1];
                        uint32_t mm = 0;
#pragma unroll
                        for (int hh = 0; hh < kCoopWarps - 1; ++hh) {
                            off[hh] = mm;
                            mm += hcnt[hh];
                        }
                        for (uint32_t i = lane; i < m; i += 32) {
                            uint32_t k2 = i;  // slot in the helper segments (constant indices
#pragma unroll                                // only: a runtime index would spill off[])
                            for (int t = 1; t < kCoopWarps - 1; ++t)
                                if (i >= off[t]) k2 = t * SRW + (i - off[t]);
                            ctd[i] = hctd[k2];
                            crp[i] = hcrp[k2];
                        }
                        __syncwarp();
                    }
                    // (c) contender ranks (key order) and prefix counts (row order)
                    uint64_t y[RW];
                    uint32_t rk[RW], pre[RW], rpv[RW];
#pragma unroll
                    for (int i = 0; i < RW; ++i) {
                        const uint32_t idx = lane + 32u * i;
                        y[i] = idx < m ? ctd[idx] : kInfKey;
                        rpv[i] = idx < m ? crp[idx] : 0u;
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
#pragma unroll
                    for (int i = 0; i < RW; ++i)
                        if (lane + 32u * i < m) csrp[rk[i]] = rpv[i];
                    __syncwarp();
                    // (d) in-place merge of P's tail, backwards
                    const uint32_t lo = csrp[0];
                    ins_lo = lo;
                    const uint32_t total = np + m;
                    if (lo < np) {
                        for (int cb = (int)((np - 1) & ~31u); cb >= (int)(lo & ~31u); cb -= 32) {
                            const uint32_t idx = (uint32_t)cb + lane;
                            const bool mv = idx < np && idx >= lo;
                            uint64_t p = 0;
                            uint32_t npos = 0;
                            if (mv) {
                                p = pk[idx];
                                npos = idx + upper_bound_u32(csrp, m, idx);
                            }
                            __syncwarp();
                            if (mv) {
                                if (npos < ef) pk[npos] = p;
                                else evk[npos - ef] = p;
                            }
                            __syncwarp();
                        }
                    }
#pragma unroll
                    for (int i = 0; i < RW; ++i) {
                        if (lane + 32u * i < m) {
                            const uint32_t npos = rk[i] + rpv[i];
                            if (npos < ef) pk[npos] = y[i];
                            else evk[npos - ef] = (rpv[i] + pre[i]) < ef ? y[i] : (y[i] | kExp);
                        }
                    }
                    __syncwarp();
                    if (lo < hint) hint = lo;
                    // (e) tie stack
                    if (total > ef) {
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
                            const uint32_t room = a.tie_cap - tn;
                            if (adds > room) overflow = true;
                            const uint32_t put = adds < room ? adds : room;
                            for (uint32_t r = lane; r < put; r += 32) tie[tn + put - 1 - r] = stg[r];
                            tn += put;
                            if (tn > c_maxtie) c_maxtie = tn;
                        }
                    }
                    np = total < ef ? total : ef;
                    __syncwarp();
                }
                // (f') the last pick's expanded mark at its index in P': entries
                // before the first insertion point are unchanged, so it is the
                // predicted pick's index unless the smallest contender came first
                if (pend_pick) {
                    const uint32_t pick = ins_lo < guess_idx ? ins_lo : guess_idx;
                    __syncwarp();
                    if (lane == 0) pk[pick] = spec_key | kExp;
                    hint = pick + 1;
                }
                // speculative scan: the best unexpanded entry of the pool (the
                // next pick unless a contender of this expansion beats it)
                uint32_t guess = kSentinel;
                guess_idx = kSentinel;
                spec_key = kInfKey;
                for (uint32_t b0 = hint & ~31u; b0 < np; b0 += 32) {
                    const uint32_t idx = b0 + lane;
                    const uint64_t pv = idx < np ? pk[idx] : kExp;
                    const bool un = idx >= hint && !(pv & kExp);
                    const unsigned bal = __ballot_sync(kFull, un);
                    if (bal) {
                        const uint32_t src = __ffs(bal) - 1;
                        guess_idx = b0 + src;
                        spec_key = __shfl_sync(kFull, pv, src);
                        guess = (uint32_t)spec_key;
                        break;
                    }
                }
                if (guess == kSentinel && tn > 0) guess = tie[tn - 1];
                spec_u = guess;
                if (lane == 0) {
                    np_sh = np;
                    gkey_sh = spec_key;
                }
                __syncwarp();
                // the pool is final for this expansion's contender tests
                asm volatile("bar.arrive 1, %0;" ::"r"(kCoopWarps * 32) : "memory");
                // the predicted pick's adjacency row, and its neighbours' code
                // rows warmed in L2 (the next gather whenever the prediction holds)
                if (guess != kSentinel) {
#pragma unroll
                    for (int j = 0; j < RW; ++j) {
                        const uint32_t sl = lane * RW + j;
                        spec_v[j] = sl < ix.RS ? __ldg(ix.adj + (size_t)guess * ix.RS + sl) : kSentinel;
                    }
#pragma unroll
                    for (int j = 0; j < RW; ++j)
                        if (spec_v[j] != kSentinel)
                            prefetch_lines_l2(ix.codes + (size_t)spec_v[j] * W, rowb);
                }
                QVG_CP(coop_ev(q, it_q, 1);)
            }
            __syncthreads();  // S1: this expansion's contenders found, P final
            QVG_CP(if (w == 0) coop_ev(q, it_q, 2);)
            if (w > 0) {
                // while the leader picks: a slice whose smallest contender beats
                // the prediction holds a likely next pick — warm L2 with its
                // neighbours' code rows (its adjacency row is the background copy)
                const uint64_t km = smin[h];
                if (km < gkey_sh && scop[h] == km) {
                    mbar_wait(abar + h, iter & 1u);
                    for (uint32_t sl = lane; sl < ix.RS; sl += 32) {
                        const uint32_t id = adjw[h * RM + sl];
                        if (id != kSentinel) prefetch_lines_l2(ix.codes + (size_t)id * W, rowb);
                    }
                }
            }

            if (w == 0) {
                // ---- phase B (leader): the helpers' contenders in row order
                c_eval += n;
                uint32_t m = 0;
                uint64_t kmin = kInfKey;
                int hsrc = -1;
#pragma unroll
                for (int hh = 0; hh < kCoopWarps - 1; ++hh) {
                    m += hcnt[hh];
                    const uint64_t km = smin[hh];
                    if (km < kmin) {
                        kmin = km;
                        hsrc = hh;
                    }
                }
                // (the slices are concatenated into ctd / crp at the start of
                // the next phase C, off the critical path: the helpers rewrite
                // them only after that phase's barrier)
                QVG_CP(coop_ev(q, it_q, 3);)
                // (f) pick: the smallest contender is always admitted, so the
                // best unexpanded entry of P' is min(predicted pick, kmin); with
                // none, the top of the tie stack (m == 0 then: the stack is final)
                uint32_t u = kSentinel;
                bool from_p = false;
                const bool retarget = kmin < spec_key;
                if (retarget) spec_key = kmin;
                if (spec_key != kInfKey) {
                    u = (uint32_t)spec_key;
                    from_p = true;
                } else if (tn > 0) {
                    u = tie[tn - 1];
                    --tn;
                    ++c_tie;
                    hint = np;
                }
                pend_m = m;
                pend_pick = from_p;
                if (u == kSentinel) {
                    if (lane == 0) *ctl_done = 1;
                } else {
                    ++c_exp;
                    // (g) adjacency row: the predicted pick's (loaded in phase
                    // C), else the background copy of the winning slice's
                    uint32_t v[RW];
                    if (!retarget && u == spec_u) {
#pragma unroll
                        for (int j = 0; j < RW; ++j) v[j] = spec_v[j];
                    } else if (scop[hsrc] == kmin) {
                        mbar_wait(abar + hsrc, iter & 1u);
#pragma unroll
                        for (int j = 0; j < RW; ++j) {
                            const uint32_t sl = lane * RW + j;
                            v[j] = sl < ix.RS ? adjw[hsrc * RM + sl] : kSentinel;
                        }
                    } else {  // the slice's smallest row was no contender (rare)
#pragma unroll
                        for (int j = 0; j < RW; ++j) {
                            const uint32_t sl = lane * RW + j;
                            v[j] = sl < ix.RS ? __ldg(ix.adj + (size_t)u * ix.RS + sl) : kSentinel;
                        }
                    }
                    QVG_CP(coop_ev(q, it_q, 4);)
                    // (h) visited filter + compaction (the helpers have read
                    // this expansion's cid)
                    bool keep[RW];
#pragma unroll
                    for (int j = 0; j < RW; ++j) {
                        const uint32_t id = v[j];
                        bool k2 = id != kSentinel;
                        if (k2) {
                            const uint32_t sidx = vhash(id, vlg);
                            if (vis[sidx] == id) k2 = false;
                            else vis[sidx] = id;
                        }
                        keep[j] = k2;
                    }
                    uint32_t pos = 0, slots = 0, nn = 0;
#pragma unroll
                    for (int j = 0; j < RW; ++j) {
                        const unsigned b = __ballot_sync(kFull, keep[j]);
                        slots += __popc(__ballot_sync(kFull, v[j] != kSentinel));
                        pos += __popc(b & lt_mask);
                        nn += __popc(b);
                    }
                    c_slots += slots;
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < RW; ++j)
                        if (keep[j]) cid[pos++] = v[j];
                    if (lane == 0) *ctl_n = nn;
                    QVG_CP(coop_ev(q, it_q, 5);)
                }
                fence_proxy_async();  // adjw reads before the helpers' next bulk copies
            }
            ++iter;
            __syncthreads();  // F1: next rows published (or done)
            QVG_CP(++it_q;)
            if (*ctl_done) break;
        }
        if (w > 0 && lane == 0) hdrop[h] = h_drop;
        // every helper's last background copy has landed before smem is reused
        if (w > 0 && lane == 0 && iter > 0) mbar_wait(abar + h, (iter - 1) & 1u);

        // ---- outputs (leader) --------------------------------------------------------
        __syncthreads();  // the helpers' drop counts
        if (w == 0) {
            for (int hh = 0; hh < kCoopWarps - 1; ++hh) c_drop += hdrop[hh];
            if (a.pool_ids) {
                for (uint32_t i = lane; i < ef; i += 32) {
                    a.pool_ids[q * ef + i] = i < np ? (uint32_t)pk[i] : kSentinel;
                    a.pool_dists[q * ef + i] = i < np ? kdist(pk[i]) : kSentinel;
                }
                if (lane == 0) a.pool_n[q] = np;
            }
            const int32_t qs = overflow ? QVG_Q_TIE_OVERFLOW : QVG_Q_OK;
            if (lane == 0) {
                if (overflow && a.flags) atomicOr(a.flags, 1u << QVG_Q_TIE_OVERFLOW);
                if (a.out_status) a.out_status[q] = qs;
                if (a.qctr) {
                    uint32_t* c = a.qctr + q * 8;
                    c[0] = c_exp;
                    c[1] = c_tie;
                    c[2] = c_eval;
                    c[3] = c_drop;
                    c[4] = c_slots;
                    c[5] = np;
                    c[6] = c_maxtie;
                    c[7] = (uint32_t)qs;
                }
                *ctl_n = np;  // pool size for the rerank
            }
        }
        __syncthreads();
        if (a.do_rerank) {
            const uint32_t NR = *ctl_n;
            // four lanes per row: lane c of a group owns chain c
            const uint32_t dim = ix.dim, main4 = dim & ~3u;
            const uint32_t ch = tid & 3u;
            for (uint32_t i = tid; i < NR; i += blockDim.x)  // warm L2 with the rows
                prefetch_l2(ix.cold + (size_t)(uint32_t)pk[i] * ix.Dp, ix.Dp * 4u);
            for (uint32_t r0 = 0; r0 < NR; r0 += blockDim.x / 4) {
                const uint32_t r = r0 + (tid >> 2);
                double s = 0.0;
                if (r < NR) {
                    const float* x = ix.cold + (size_t)(uint32_t)pk[r] * ix.Dp;
                    uint32_t i = ch;
                    for (; i + 28 < main4; i += 32) {  // 8 loads in flight per lane
                        float xv[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) xv[u] = __ldg(x + i + 4 * u);
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            s = __fma_rn((double)qn[i + 4 * u], (double)xv[u], s);
                    }
                    for (; i < main4; i += 4) s = __fma_rn((double)qn[i], (double)__ldg(x + i), s);
                    if (ch == 0)  // tail elements >= 4*floor(D/4) all go to chain 0
                        for (uint32_t t = main4; t < dim; ++t)
                            s = __fma_rn((double)qn[t], (double)__ldg(x + t), s);
                }
                const double s1 = __shfl_down_sync(kFull, s, 1);
                const double s2 = __shfl_down_sync(kFull, s, 2);
                const double s3 = __shfl_down_sync(kFull, s, 3);
                if (r < NR && ch == 0)
                    sc[r] = __double2float_rn(__dadd_rn(__dadd_rn(s, s1), __dadd_rn(s2, s3)));
            }
            __syncthreads();
            if (w == 0) {  // rank by (score desc, id asc), emit the first k
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
            }
        }
        __syncthreads();  // smem reused by the next query
    }
}

uint32_t pow2ceil_c(uint32_t x) {
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

struct CoopPlan {
    void* fn;
    uint32_t rw, SRW, block_bytes;
};

CoopPlan coop_plan(const DevIndex& ix, uint32_t ef, uint32_t vis_log2, uint32_t tie_cap) {
    CoopPlan p;
    p.rw = pow2ceil_c((ix.R + 31) / 32);
    p.fn = p.rw == 1 ? (void*)coop_kernel<1> : (p.rw == 2 ? (void*)coop_kernel<2> : (void*)coop_kernel<4>);
    const uint32_t RM = p.rw * 32;
    // rows per helper warp (the leader scores none): a multiple of 4
    p.SRW = (((RM + kCoopWarps - 2) / (kCoopWarps - 1)) + 3u) & ~3u;
    p.block_bytes =
        coop_layout((ef + 31) & ~31u, RM, ix.W, tie_cap, 1u << coop_vis_log2(vis_log2), ix.Dp,
                    p.SRW).total;
    return p;
}

}  // namespace

// resident CTAs per SM of a coop instantiation at a shared-memory size, cached
// (the occupancy query and the attribute call cost host time on every small-
// batch call, where the GPU would otherwise wait for the launch)
static int coop_per_sm(void* fn, uint32_t block_bytes, int device) {
    struct Key {
        void* fn;
        uint32_t bytes;
        int dev;
        bool operator<(const Key& o) const {
            if (fn != o.fn) return fn < o.fn;
            return bytes != o.bytes ? bytes < o.bytes : dev < o.dev;
        }
    };
    static std::mutex mu;
    static std::map<Key, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    const Key k{fn, block_bytes, device};
    auto it = cache.find(k);
    if (it != cache.end()) return it->second;
    int maxs = 0, per_sm = 0;
    cudaDeviceGetAttribute(&maxs, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (block_bytes > (uint32_t)maxs ||
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, maxs) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kCoopWarps * 32, block_bytes) !=
            cudaSuccess) {
        cudaGetLastError();
        per_sm = 0;
    }
    cache.emplace(k, per_sm);
    return per_sm;
}

// resident CTAs (= concurrently served queries) of the latency kernel for
// this launch, 0 when it cannot run it
// (geometry only: the caller also excludes exact-visited, fused / pipelined
// encode and rerank depths other than ef, which the throughput kernel serves)
uint64_t coop_capacity(const SearchLaunch& a, int device) {
    if (extra_depth(a.ef, a.depth)) return 0;
    if ((1u << a.vis_log2) < ((a.ef + 31u) & ~31u)) return 0;
    const CoopPlan p = coop_plan(a.ix, a.ef, a.vis_log2, a.tie_cap);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return (uint64_t)coop_per_sm(p.fn, p.block_bytes, device) * sms;
}

qvg_status launch_coop(const SearchLaunch& a, const CUtensorMap* tmap, cudaStream_t s,
                       int device, uint64_t* grid_out) {
    const CoopPlan p = coop_plan(a.ix, a.ef, a.vis_log2, a.tie_cap);
    static int sms = [device] {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
        return v;
    }();
    const int per_sm = coop_per_sm(p.fn, p.block_bytes, device);
    if (per_sm < 1) {
        set_error("coop: the latency kernel does not fit");
        return QVG_INVALID_ARGUMENT;
    }
    uint64_t grid = (uint64_t)per_sm * sms;
    if (a.nq < grid) grid = a.nq;
    if (grid < 1) grid = 1;
    alignas(64) CUtensorMap dummy;
    memset(&dummy, 0, sizeof(dummy));
    const CUtensorMap* m = tmap ? tmap : &dummy;
    uint32_t srw = p.SRW;
    void* args[] = {(void*)m, (void*)&a, (void*)&srw};
    const cudaError_t e =
        cudaLaunchKernel(p.fn, dim3((unsigned)grid), dim3(kCoopWarps * 32), args, p.block_bytes, s);
    if (grid_out) *grid_out = grid;
    return e == cudaSuccess ? QVG_OK : cuda_status(e, "launch(coop)");
}

}  // namespace qvg

#ifdef QVG_COOP_PHASES
// instrumented build only: the trace of query 0's block (tools/coop_phases.py)
extern "C" int qvg_debug_coop_trace(unsigned long long* out, int rows) {
    return cudaMemcpyFromSymbol(out, qvg::g_coop_trace, sizeof(unsigned long long) * 16 * rows) ==
                   cudaSuccess
               ? 0
               : 1;
}
#endif

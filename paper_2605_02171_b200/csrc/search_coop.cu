// Latency mode: one CTA of kCoopWarps warps per query (small batches).
//
// The throughput kernel (search.cu) gives each query one warp, which is the
// right trade when thousands of queries keep every SM busy; with a handful of
// queries the GPU is idle and a query's latency is its serial chain of ~80
// expansions.  Here the per-expansion work that parallelises is spread over
// the CTA:
//   * every warp TMA-gathers and scores its slice of the expansion's rows
//     (<= 16 of 64) in one round trip, into a shared distance array;
//   * the leader warp then runs the unchanged state machine of search.cu —
//     the same contender test, prefix admission, in-place merge, tie stack,
//     pick, visited table and compaction, on the same distances in the same
//     row order — so pools, ids and scores are identical (search.cpp:27-81);
//   * the rerank spreads the pool over all lanes, four lanes per row: lane c
//     accumulates chain c (elements i = c mod 4, ascending) and lane 0 of the
//     group folds the tail and combines (s0 + s1) + (s2 + s3) — the reference's
//     dot_f32 order (vec_math.hpp:13-26), hence bit-identical scores.
// Not used with exact-visited bitmaps, a rerank depth above ef, or the fused
// encode prologue (the throughput kernel covers those).
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "bq_device.cuh"
#include "qvg_internal.cuh"
#include "search_common.cuh"

namespace qvg {

namespace {

struct CoopLayout {
    uint32_t bars, stages, stage_bytes, pk, ctd, evk, crp, csrp, cid, stg, dsh, spec, qc, tie, vis,
        qn, ctl, total;
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
    L.bars = take(8 * kCoopWarps, 16);
    L.stage_bytes = (SRW / 4) * group_stride(W);  // multiple of 128
    L.stages = take(kCoopWarps * L.stage_bytes, 128);
    L.pk = take(8 * EFM, 16);
    L.ctd = take(8 * RM, 16);
    L.evk = L.ctd;
    L.crp = take(4 * RM, 16);
    L.csrp = take(4 * RM, 16);
    L.cid = take(4 * RM, 16);
    L.stg = L.crp;
    L.dsh = take(4 * RM, 16);     // row distances, row order
    L.spec = take(4 * RM, 16);    // predicted next pick's adjacency row (L2 prefetch)
    L.qc = take(16 * W, 16);
    L.tie = take(4 * tie_cap, 16);
    L.vis = take(4 * vis_slots, 16);  // rerank scores alias it (vis_slots >= EFM)
    L.qn = take(4 * Dp, 16);          // normalised query (rerank)
    L.ctl = take(32, 16);             // query index (u64), row count, done flag
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
    const uint32_t VS = 1u << a.vis_log2;
    const uint32_t ef = a.ef;
    const uint32_t EFM = (ef + 31u) & ~31u;
    const CoopLayout L = coop_layout(EFM, RM, W, a.tie_cap, VS, ix.Dp, SRW);
    unsigned char* base = smem_raw;
    uint64_t* bar = reinterpret_cast<uint64_t*>(base + L.bars) + w;
    unsigned char* const stage = base + L.stages + w * L.stage_bytes;
    uint64_t* pk = reinterpret_cast<uint64_t*>(base + L.pk);
    uint64_t* ctd = reinterpret_cast<uint64_t*>(base + L.ctd);
    uint64_t* evk = reinterpret_cast<uint64_t*>(base + L.evk);
    uint32_t* crp = reinterpret_cast<uint32_t*>(base + L.crp);
    uint32_t* csrp = reinterpret_cast<uint32_t*>(base + L.csrp);
    uint32_t* cid = reinterpret_cast<uint32_t*>(base + L.cid);
    uint32_t* stg = reinterpret_cast<uint32_t*>(base + L.stg);
    uint32_t* dsh = reinterpret_cast<uint32_t*>(base + L.dsh);
    uint32_t* spec = reinterpret_cast<uint32_t*>(base + L.spec);
    uint4* qc = reinterpret_cast<uint4*>(base + L.qc);
    uint32_t* tie = reinterpret_cast<uint32_t*>(base + L.tie);
    uint32_t* vis = reinterpret_cast<uint32_t*>(base + L.vis);
    float* sc = reinterpret_cast<float*>(base + L.vis);
    float* qn = reinterpret_cast<float*>(base + L.qn);
    unsigned long long* ctl_q = reinterpret_cast<unsigned long long*>(base + L.ctl);
    volatile uint32_t* ctl_n = reinterpret_cast<volatile uint32_t*>(base + L.ctl + 8);
    volatile uint32_t* ctl_done = reinterpret_cast<volatile uint32_t*>(base + L.ctl + 12);

    if (lane == 0) {
        mbar_init(bar);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t phase = 0;
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
            vis[vhash(entry, a.vis_log2)] = entry;
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
        for (;;) {
            const uint32_t n = *ctl_n;
            // (a) this warp's slice of the rows: one gather, one round trip
            const uint32_t r0 = w * SRW;
            const uint32_t cnt = n > r0 ? min(SRW, n - r0) : 0u;
            if (cnt) {
                const uint32_t ng = (cnt + 3u) >> 2;
                TMA_WAR_FENCE();
                __syncwarp();
                if (lane == 0) mbar_expect_tx(bar, ng * 4u * rowb);
                __syncwarp();
                if (lane < ng) {
                    const uint32_t j = r0 + 4u * lane;
                    const uint32_t i0 = cid[j];
                    const uint32_t i1 = 4u * lane + 1u < cnt ? cid[j + 1] : i0;
                    const uint32_t i2 = 4u * lane + 2u < cnt ? cid[j + 2] : i0;
                    const uint32_t i3 = 4u * lane + 3u < cnt ? cid[j + 3] : i0;
                    dev::tma_gather4(stage + lane * gstride, &tmap, 0, i0, i1, i2, i3, bar);
                }
            }
            if (w == 0) {  // speculative adjacency of the current best unexpanded entry
                uint32_t guess = kSentinel;
                for (uint32_t b0 = hint & ~31u; b0 < np; b0 += 32) {
                    const uint32_t idx = b0 + lane;
                    const bool un = idx < np && idx >= hint && !(pk[idx] & kExp);
                    const unsigned bal = __ballot_sync(kFull, un);
                    if (bal) {
                        guess = (uint32_t)pk[b0 + __ffs(bal) - 1];
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
#pragma unroll
                for (int j = 0; j < RW; ++j)  // published for the helpers' L2 prefetch
                    spec[lane * RW + j] = guess != kSentinel ? spec_v[j] : kSentinel;
            }
            if (cnt) {
                mbar_wait(bar, phase);
                phase ^= 1u;
                const uint4* st = reinterpret_cast<const uint4*>(stage);
                const uint32_t j = lane >> lpr_log;
                const uint32_t part = lane & (LPR - 1u);
                uint32_t d = 0;
                if (j < cnt) {
                    const uint4* rowp = st + ((j >> 2) * gstride + (j & 3u) * rowb) / 16u;
                    d = row_sm2(qc, rowp, W, rot, part, LPR);
                }
                for (uint32_t o = 1; o < LPR; o <<= 1) d += __shfl_xor_sync(kFull, d, o);
                if (j < cnt && part == 0) dsh[r0 + j] = d;
            }
            __syncthreads();  // all slices scored

            if (w > 0) {
                // helpers are idle while the leader merges: warm L2 with the code
                // rows of the predicted next pick (its rows are gathered next
                // whenever the prediction holds)
                for (uint32_t sl = (w - 1) * 32 + lane; sl < RM; sl += (kCoopWarps - 1) * 32) {
                    const uint32_t id = spec[sl];
                    if (id != kSentinel) prefetch_l2(ix.codes + (size_t)id * W, rowb);
                }
            }
            if (w == 0) {
                c_eval += n;
                const uint64_t worst = np == ef ? ordk(pk[ef - 1]) : kInfKey;
                uint32_t m = 0;
                // (b) contender test + row-order compaction
                for (uint32_t i0 = 0; i0 < n; i0 += 32) {
                    const uint32_t jr = i0 + lane;
                    const bool valid = jr < n;
                    const uint64_t key = valid ? mkkey(dsh[jr], cid[jr]) : kInfKey;
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
                }
                __syncwarp();
                if (m > 0) {
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
                // (f) pick
                uint32_t u = kSentinel;
                for (uint32_t b0 = hint & ~31u; b0 < np; b0 += 32) {
                    const uint32_t idx = b0 + lane;
                    const bool un = idx < np && idx >= hint && !(pk[idx] & kExp);
                    const unsigned bal = __ballot_sync(kFull, un);
                    if (bal) {
                        const uint32_t pick = b0 + __ffs(bal) - 1;
                        u = (uint32_t)pk[pick];
                        __syncwarp();
                        if (lane == 0) pk[pick] |= kExp;
                        hint = pick + 1;
                        break;
                    }
                }
                bool done = false;
                if (u == kSentinel) {
                    hint = np;
                    if (tn == 0) {
                        done = true;
                    } else {
                        u = tie[tn - 1];
                        --tn;
                        ++c_tie;
                    }
                }
                if (done) {
                    if (lane == 0) *ctl_done = 1;
                } else {
                    ++c_exp;
                    // (g) adjacency row (speculative hit or fresh load)
                    uint32_t v[RW];
                    if (u == spec_u) {
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
                    // (h) visited filter + compaction
                    bool keep[RW];
#pragma unroll
                    for (int j = 0; j < RW; ++j) {
                        const uint32_t id = v[j];
                        bool k2 = id != kSentinel;
                        if (k2) {
                            const uint32_t s = vhash(id, a.vis_log2);
                            if (vis[s] == id) k2 = false;
                            else vis[s] = id;
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
                }
            }
            __syncthreads();  // next rows (or done) published
            if (*ctl_done) break;
        }

        // ---- outputs (leader) --------------------------------------------------------
        if (w == 0) {
            for (int off = 16; off > 0; off >>= 1) c_drop += __shfl_xor_sync(kFull, c_drop, off);
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
    p.SRW = (((RM + kCoopWarps - 1) / kCoopWarps) + 3u) & ~3u;  // <= 32 rows per warp
    p.block_bytes =
        coop_layout((ef + 31) & ~31u, RM, ix.W, tie_cap, 1u << vis_log2, ix.Dp, p.SRW).total;
    return p;
}

}  // namespace

// resident CTAs (= concurrently served queries) of the latency kernel for
// this launch, 0 when it cannot run it
// (geometry only: the caller also excludes exact-visited, fused / pipelined
// encode and rerank depths other than ef, which the throughput kernel serves)
uint64_t coop_capacity(const SearchLaunch& a, int device) {
    if (extra_depth(a.ef, a.depth)) return 0;
    if ((1u << a.vis_log2) < ((a.ef + 31u) & ~31u)) return 0;
    const CoopPlan p = coop_plan(a.ix, a.ef, a.vis_log2, a.tie_cap);
    int maxs = 0, sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&maxs, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (p.block_bytes > (uint32_t)maxs) return 0;
    if (cudaFuncSetAttribute(p.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, maxs) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p.fn, kCoopWarps * 32,
                                                      p.block_bytes) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return (uint64_t)per_sm * sms;
}

qvg_status launch_coop(const SearchLaunch& a, const CUtensorMap* tmap, cudaStream_t s,
                       int device, uint64_t* grid_out) {
    const CoopPlan p = coop_plan(a.ix, a.ef, a.vis_log2, a.tie_cap);
    int maxs = 0, sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&maxs, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaError_t e = cudaFuncSetAttribute(p.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, maxs);
    if (e != cudaSuccess) return cuda_status(e, "coop: smem attribute");
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p.fn, kCoopWarps * 32,
                                                      p.block_bytes);
    if (e != cudaSuccess || per_sm < 1) return cuda_status(e, "coop: occupancy");
    uint64_t grid = (uint64_t)per_sm * sms;
    if (a.nq < grid) grid = a.nq;
    if (grid < 1) grid = 1;
    alignas(64) CUtensorMap dummy;
    memset(&dummy, 0, sizeof(dummy));
    const CUtensorMap* m = tmap ? tmap : &dummy;
    uint32_t srw = p.SRW;
    void* args[] = {(void*)m, (void*)&a, (void*)&srw};
    e = cudaLaunchKernel(p.fn, dim3((unsigned)grid), dim3(kCoopWarps * 32), args, p.block_bytes, s);
    if (grid_out) *grid_out = grid;
    return e == cudaSuccess ? QVG_OK : cuda_status(e, "launch(coop)");
}

}  // namespace qvg

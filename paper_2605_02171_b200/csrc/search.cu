// K2/K3/K4 — exact BQ beam search fused with the float32 rerank, one warp per
// query, persistent grid with an atomic query counter.
//
// Reference behaviour reproduced (paths under /root/reference/proj/core):
//   beam_search_words  search.cpp:27-81   dual-heap best-first search
//   candidate_less     graph.hpp:28-30    (dist, id) order == u64 key order
//   sm2_distance_words encoding.hpp:169-176
//   rerank             search.cpp:96-120  4-chain double dot (vec_math.hpp:13-26),
//                                         sort (score desc, id asc), take k
//
// The dual heap is replaced by the equivalent sorted-list state machine of
// SURVEY §8.A.3 (validated against the reference: tests/test_oracle_pins.py and
// the GPU parity tests):
//   P   sorted pool of <= ef u64 keys (dist<<32 | id) + expanded flags (smem,
//       double-buffered)
//   T   tie stack: keys evicted from P while unexpanded whose dist equals the
//       pool's worst dist.  Worst dist never increases once P is full, so every
//       live T entry shares one dist (tdist) and new entries (always smaller
//       keys) are pushed on top; a drop of the worst dist kills all of T.
//   vis lossy direct-mapped visited table (smem).  A forgotten node that is
//       scored again is either already in P (found by exact lookup, dropped) or
//       has key > max(P) and is rejected, so results are unchanged
//       (SURVEY §8.A.4b); misses cost only bandwidth.
// Admission of a row is the exact parallel form of the sequential loop: the
// i-th surviving neighbour c_i is admitted iff
//   #{p in P : p < c_i} + #{j < i : c_j < c_i} < ef
// and P' = first ef of merge(P, admitted).  Only "contenders" (c < max(P), or
// any c while P is not full) can matter, so the per-row sort/merge work scales
// with the few contenders, not with the row length.
#include <cuda_runtime.h>

#include "qvg_internal.cuh"

namespace qvg {

namespace {

constexpr uint64_t kInfKey = ~0ull;
constexpr unsigned kFull = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t vhash(uint32_t id, uint32_t lg) {
    return (id * 0x9E3779B1u) >> (32 - lg);
}

// SM2 distance contribution of one 16-B chunk {pos word, strong word}
// (encoding.hpp:169-176): popc(x) + popc(x & (sa|sb)) + 2*popc(x & sa & sb)
__device__ __forceinline__ uint32_t sm2_chunk(const uint4 q, const uint4 v) {
    const uint32_t x0 = q.x ^ v.x, x1 = q.y ^ v.y;
    const uint32_t o0 = x0 & (q.z | v.z), o1 = x1 & (q.w | v.w);
    const uint32_t a0 = x0 & q.z & v.z, a1 = x1 & q.w & v.w;
    return __popc(x0) + __popc(x1) + __popc(o0) + __popc(o1) + 2u * (__popc(a0) + __popc(a1));
}

__device__ __forceinline__ uint4 ldg_chunk(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ uint32_t lower_bound_u64(const uint64_t* a, uint32_t n, uint64_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// 4 strided double chains combined as (s0+s1)+(s2+s3) (vec_math.hpp:13-26).
// Products of floats are exact in double, so FMA == mul+add here.
__device__ __forceinline__ float dot4_exact(const float* __restrict__ q,
                                            const float* __restrict__ v, uint32_t dim) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const float4* q4 = reinterpret_cast<const float4*>(q);
    const float4* v4 = reinterpret_cast<const float4*>(v);
    const uint32_t n4 = dim >> 2;
    uint32_t t = 0;
    for (; t + 8 <= n4; t += 8) {
        float4 b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) b[u] = __ldg(v4 + t + u);
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
    uint32_t pk0, pk1, cand, ctd, cid, stg, pf0, pf1, qc, tie, vis, misc, total;
};

// Per-warp shared-memory carve-up (bytes, every region 16-B aligned).
__host__ __device__ inline SmemLayout smem_layout(uint32_t EFM, uint32_t RM, uint32_t W,
                                                  uint32_t tie_cap, uint32_t vis_slots) {
    SmemLayout L;
    uint32_t o = 0;
    auto take = [&](uint32_t bytes) {
        const uint32_t at = o;
        o += (bytes + 15u) & ~15u;
        return at;
    };
    L.pk0 = take(8 * EFM);
    L.pk1 = take(8 * EFM);
    L.cand = take(8 * RM);  // candidate keys in row order; later sorted contenders
    L.ctd = take(8 * RM);   // contenders in row order; later evicted keys
    L.cid = take(4 * RM);   // compacted row ids; later eviction flags
    L.stg = take(4 * RM);   // tie-stack additions, ascending
    L.pf0 = take(EFM);
    L.pf1 = take(EFM);
    L.qc = take(16 * W);
    L.tie = take(4 * tie_cap);
    L.vis = take(4 * vis_slots);  // rerank scores alias this region (vis_slots >= EFM)
    L.misc = take(16);
    L.total = o;
    return L;
}

template <int EFW, int RW, int PB>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    search_kernel(const SearchLaunch a, const uint32_t warp_bytes, const uint32_t G) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr uint32_t EFM = EFW * 32;
    constexpr uint32_t RM = RW * 32;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t wib = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const DevIndex ix = a.ix;
    const uint32_t W = ix.W;
    const uint32_t VS = 1u << a.vis_log2;
    const SmemLayout L = smem_layout(EFM, RM, W, a.tie_cap, VS);
    unsigned char* base = smem_raw + (size_t)wib * warp_bytes;
    uint64_t* pk = reinterpret_cast<uint64_t*>(base + L.pk0);
    uint64_t* pk2 = reinterpret_cast<uint64_t*>(base + L.pk1);
    uint8_t* pf = base + L.pf0;
    uint8_t* pf2 = base + L.pf1;
    uint64_t* cand = reinterpret_cast<uint64_t*>(base + L.cand);
    uint64_t* cs = cand;  // alias: sorted contenders
    uint64_t* ctd = reinterpret_cast<uint64_t*>(base + L.ctd);
    uint64_t* evk = ctd;  // alias: evicted keys by (newpos - ef)
    uint32_t* cid = reinterpret_cast<uint32_t*>(base + L.cid);
    uint8_t* evf = reinterpret_cast<uint8_t*>(base + L.cid);  // alias: eviction flags
    uint4* qc = reinterpret_cast<uint4*>(base + L.qc);
    uint32_t* tie = reinterpret_cast<uint32_t*>(base + L.tie);
    uint32_t* vis = reinterpret_cast<uint32_t*>(base + L.vis);
    float* sc = reinterpret_cast<float*>(base + L.vis);

    const uint32_t ef = a.ef;
    const uint32_t RPP = 32u / G;  // code rows per pass
    const uint32_t sub = lane & (G - 1u);
    const uint32_t grp = lane / G;
    const uint32_t cpl = (W + G - 1u) / G;
    const uint64_t gwarp = (uint64_t)blockIdx.x * kWarpsPerBlock + wib;
    uint32_t* xbits = a.exact_bits ? a.exact_bits + gwarp * a.exact_words : nullptr;

    // Score the n compacted ids in cid[0..n) into cand[0..n) (row order).
    auto gather = [&](uint32_t n) {
        for (uint32_t b0 = 0; b0 < n; b0 += RPP * PB) {
            uint32_t acc[PB];
#pragma unroll
            for (int b = 0; b < PB; ++b) acc[b] = 0;
            for (uint32_t c0 = 0; c0 < cpl; c0 += 3) {
                uint4 qv[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const uint32_t w = sub + (c0 + c) * G;
                    qv[c] = (c0 + c < cpl && w < W) ? qc[w] : make_uint4(0, 0, 0, 0);
                }
                uint4 buf[PB][3];
#pragma unroll
                for (int b = 0; b < PB; ++b) {
                    const uint32_t r = b0 + b * RPP + grp;
                    const uint32_t id = r < n ? cid[r] : 0u;
                    const uint4* row = ix.codes + (size_t)id * W;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const uint32_t w = sub + (c0 + c) * G;
                        buf[b][c] = (r < n && c0 + c < cpl && w < W) ? ldg_chunk(row + w) : qv[c];
                    }
                }
#pragma unroll
                for (int b = 0; b < PB; ++b)
#pragma unroll
                    for (int c = 0; c < 3; ++c) acc[b] += sm2_chunk(qv[c], buf[b][c]);
            }
#pragma unroll
            for (int b = 0; b < PB; ++b) {
                for (uint32_t off = G >> 1; off > 0; off >>= 1)
                    acc[b] += __shfl_xor_sync(kFull, acc[b], off);
                const uint32_t r = b0 + b * RPP + grp;
                if (sub == 0 && r < n) cand[r] = ((uint64_t)acc[b] << 32) | cid[r];
            }
        }
    };

    for (;;) {
        unsigned long long qq = 0;
        if (lane == 0) qq = atomicAdd(a.counter, 1ull);
        qq = __shfl_sync(kFull, qq, 0);
        if (qq >= a.nq) break;
        const uint64_t q = qq;

        const int32_t qst = a.qstatus ? a.qstatus[q] : 0;
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
            }
            continue;
        }

        // ---- per-query init --------------------------------------------------
        for (uint32_t w = lane; w < W; w += 32) qc[w] = a.qcodes[q * W + w];
        if (xbits) {
            uint4* xb4 = reinterpret_cast<uint4*>(xbits);
            for (uint64_t i = lane; i < a.exact_words / 4; i += 32) xb4[i] = make_uint4(0, 0, 0, 0);
            __syncwarp();
        } else {
            for (uint32_t i = lane; i < VS; i += 32) vis[i] = kSentinel;
        }
        uint32_t entry = a.entry;
        if (lane == 0) {
            cid[0] = entry;
            if (xbits) atomicOr(xbits + (entry >> 5), 1u << (entry & 31));
            else vis[vhash(entry, a.vis_log2)] = entry;
        }
        __syncwarp();
        gather(1);
        __syncwarp();
        if (lane == 0) {
            pk[0] = cand[0];
            pf[0] = 0;
        }
        __syncwarp();
        uint32_t np = 1, tn = 0, tdist = 0;
        uint32_t c_exp = 0, c_tie = 0, c_eval = 1, c_drop = 0, c_slots = 0, c_maxtie = 0;
        bool overflow = false;

        // ---- best-first loop ----------------------------------------------------
        for (;;) {
            // 1. pick: first unexpanded pool entry, else the top of the tie stack
            int pick = -1;
#pragma unroll
            for (int e = 0; e < EFW; ++e) {
                const uint32_t idx = lane + 32u * e;
                const bool un = idx < np && pf[idx] == 0;
                const unsigned bal = __ballot_sync(kFull, un);
                if (bal) {
                    pick = 32 * e + __ffs(bal) - 1;
                    break;
                }
            }
            uint32_t u;
            if (pick >= 0) {
                u = (uint32_t)pk[pick];
                __syncwarp();
                if (lane == 0) pf[pick] = 1;
            } else if (tn > 0) {
                // every live tie entry has dist == worst(P).dist: the reference's
                // stop test (search.cpp:48, dist-only, strict) does not fire
                u = tie[tn - 1];
                --tn;
                ++c_tie;
            } else {
                break;
            }
            ++c_exp;

            // 2. adjacency row (stored order), vectorised, sentinel = unused slot
            uint32_t v[RW];
            {
                const uint32_t* row = ix.adj + (size_t)u * ix.RS;
                if (lane * RW < ix.RS) {
                    if (RW == 1) {
                        v[0] = __ldg(row + lane);
                    } else if (RW == 2) {
                        const uint2 t = __ldg(reinterpret_cast<const uint2*>(row) + lane);
                        v[0] = t.x;
                        v[1] = t.y;
                    } else {
                        const uint4 t = __ldg(reinterpret_cast<const uint4*>(row) + lane);
                        v[0] = t.x;
                        v[1] = t.y;
                        if (RW > 2) {
                            v[2 % RW] = t.z;
                            v[3 % RW] = t.w;
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < RW; ++j) v[j] = kSentinel;
                }
            }
            // 3. visited filter (slot s = lane*RW + j; rows carry no duplicates)
            bool keep[RW];
            unsigned deg_bal = 0;
#pragma unroll
            for (int j = 0; j < RW; ++j) {
                const uint32_t id = v[j];
                bool k2 = id != kSentinel;
                deg_bal += __popc(__ballot_sync(kFull, k2));
                if (k2) {
                    if (xbits) {
                        const uint32_t bit = 1u << (id & 31);
                        k2 = (atomicOr(xbits + (id >> 5), bit) & bit) == 0;
                    } else {
                        const uint32_t s = vhash(id, a.vis_log2);
                        if (vis[s] == id) k2 = false;
                        else vis[s] = id;
                    }
                }
                keep[j] = k2;
            }
            c_slots += deg_bal;
            uint32_t n = 0, pos = 0;
#pragma unroll
            for (int j = 0; j < RW; ++j) {
                const unsigned b = __ballot_sync(kFull, keep[j]);
                pos += __popc(b & lt_mask);
                n += __popc(b);
            }
#pragma unroll
            for (int j = 0; j < RW; ++j)
                if (keep[j]) cid[pos++] = v[j];
            __syncwarp();
            if (n == 0) continue;
            c_eval += n;

            // 4. gather codes + SM2 distances -> cand[r] (row order)
            gather(n);
            __syncwarp();

            // 5. contenders: c < max(P) (or P not full), not already in P
            const uint64_t worst = np == ef ? pk[ef - 1] : kInfKey;
            uint64_t x[RW];
            bool isc[RW];
#pragma unroll
            for (int i = 0; i < RW; ++i) {
                const uint32_t r = lane + 32u * i;
                x[i] = r < n ? cand[r] : kInfKey;
                bool c2 = x[i] < worst;
                if (c2) {
                    const uint32_t rp = lower_bound_u64(pk, np, x[i]);
                    if (rp < np && pk[rp] == x[i]) {
                        c2 = false;
                        ++c_drop;  // per-lane count, reduced at the end
                    }
                }
                isc[i] = c2;
            }
            uint32_t m = 0;
            pos = 0;
#pragma unroll
            for (int i = 0; i < RW; ++i) {
                const unsigned b = __ballot_sync(kFull, isc[i]);
                // row order r = lane + 32 i  ->  order by (i, lane)
                const uint32_t before = m + __popc(b & lt_mask);
                if (isc[i]) ctd[before] = x[i];
                m += __popc(b);
            }
            __syncwarp();
            if (m == 0) continue;

            // 6. contender ranks (among contenders) and prefix counts (row order)
            uint64_t y[RW];
            uint32_t rk[RW], pre[RW], rp[RW];
#pragma unroll
            for (int i = 0; i < RW; ++i) {
                const uint32_t idx = lane + 32u * i;
                y[i] = idx < m ? ctd[idx] : kInfKey;
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
            for (int i = 0; i < RW; ++i) {
                const uint32_t idx = lane + 32u * i;
                rp[i] = idx < m ? lower_bound_u64(pk, np, y[i]) : 0u;
                if (idx < m) cs[rk[i]] = y[i];  // sorted contenders
            }
            __syncwarp();

            // 7. merge into the other pool buffer; evicted keys -> evk/evf
            const uint32_t total = np + m;
            const uint32_t newnp = total < ef ? total : ef;
            uint64_t wkey = 0;
            bool haveW = false;
            for (uint32_t idx = lane; idx < np; idx += 32) {
                const uint64_t p = pk[idx];
                const uint8_t f = pf[idx];
                const uint32_t npos = idx + lower_bound_u64(cs, m, p);
                if (npos < ef) {
                    pk2[npos] = p;
                    pf2[npos] = f;
                } else {
                    evk[npos - ef] = p;
                    evf[npos - ef] = f == 0;  // unexpanded -> tie candidate
                }
                if (npos == ef - 1) {
                    wkey = p;
                    haveW = true;
                }
            }
#pragma unroll
            for (int i = 0; i < RW; ++i) {
                const uint32_t idx = lane + 32u * i;
                if (idx < m) {
                    const uint32_t npos = rk[i] + rp[i];
                    if (npos < ef) {
                        pk2[npos] = y[i];
                        pf2[npos] = 0;
                    } else {
                        evk[npos - ef] = y[i];
                        evf[npos - ef] = (rp[i] + pre[i]) < ef;  // admitted, then evicted
                    }
                    if (npos == ef - 1) {
                        wkey = y[i];
                        haveW = true;
                    }
                }
            }
            {
                const unsigned hb = __ballot_sync(kFull, haveW);
                if (hb) wkey = __shfl_sync(kFull, wkey, __ffs(hb) - 1);
            }
            __syncwarp();

            // 8. tie stack maintenance
            if (total > ef) {
                const uint32_t wd = (uint32_t)(wkey >> 32);
                if (tn == 0 || wd < tdist) {
                    tn = 0;
                    tdist = wd;
                }
                const uint32_t nev = total - ef;
                uint32_t* stg = reinterpret_cast<uint32_t*>(base + L.stg);
                uint32_t adds = 0;
                for (uint32_t b0 = 0; b0 < nev; b0 += 32) {
                    const uint32_t e = b0 + lane;
                    uint32_t idv = kSentinel;
                    if (e < nev) {
                        const uint64_t kk = evk[e];
                        if (evf[e] && (uint32_t)(kk >> 32) == wd) idv = (uint32_t)kk;
                    }
                    const unsigned b = __ballot_sync(kFull, idv != kSentinel);
                    if (idv != kSentinel) stg[adds + __popc(b & lt_mask)] = idv;
                    adds += __popc(b);
                }
                __syncwarp();
                const uint32_t room = a.tie_cap - tn;
                if (adds > room) overflow = true;
                const uint32_t put = adds < room ? adds : room;
                // smallest key on top of the stack
                for (uint32_t r = lane; r < put; r += 32) tie[tn + put - 1 - r] = stg[r];
                tn += put;
                if (tn > c_maxtie) c_maxtie = tn;
                __syncwarp();
            }
            // swap pool buffers
            {
                uint64_t* t1 = pk;
                pk = pk2;
                pk2 = t1;
                uint8_t* t2 = pf;
                pf = pf2;
                pf2 = t2;
            }
            np = newnp;
        }

        // ---- outputs ------------------------------------------------------------
        // reduce per-lane in-pool drop counts
        for (int off = 16; off > 0; off >>= 1) c_drop += __shfl_xor_sync(kFull, c_drop, off);
        if (a.pool_ids) {
            for (uint32_t i = lane; i < ef; i += 32) {
                a.pool_ids[q * ef + i] = i < np ? (uint32_t)pk[i] : kSentinel;
                a.pool_dists[q * ef + i] = i < np ? (uint32_t)(pk[i] >> 32) : kSentinel;
            }
            if (lane == 0) a.pool_n[q] = np;
        }
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
        if (a.do_rerank) {
            // rerank: one lane per pool entry, 4 sequential double chains
            const float* qv = a.qn + q * ix.Dp;
            __syncwarp();
            for (uint32_t idx = lane; idx < np; idx += 32) {
                const uint32_t id = (uint32_t)pk[idx];
                sc[idx] = dot4_exact(qv, ix.cold + (size_t)id * ix.Dp, ix.dim);
            }
            __syncwarp();
            // rank by (score desc, id asc) and emit the first k
            for (uint32_t idx = lane; idx < np; idx += 32) {
                const float si = sc[idx];
                const uint32_t ii = (uint32_t)pk[idx];
                uint32_t rank = 0;
                for (uint32_t j = 0; j < np; ++j) {
                    const float sj = sc[j];
                    const uint32_t ij = (uint32_t)pk[j];
                    rank += (sj > si) | ((sj == si) & (ij < ii));
                }
                if (rank < a.k) {
                    a.out_ids[q * a.k + rank] = ii;
                    a.out_scores[q * a.k + rank] = si;
                }
            }
            for (uint32_t r = np + lane; r < a.k; r += 32) {
                a.out_ids[q * a.k + r] = kSentinel;
                a.out_scores[q * a.k + r] = __int_as_float(0x7fc00000);
            }
            if (lane == 0 && a.out_count) a.out_count[q] = np < a.k ? np : a.k;
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

template <int EFW, int RW>
using KernelPtr = void (*)(const SearchLaunch, const uint32_t, const uint32_t);

constexpr int kPB = 4;

template <int RW>
void* pick_kernel_ef(uint32_t efw) {
    switch (efw) {
        case 1: return (void*)search_kernel<1, RW, kPB>;
        case 2: return (void*)search_kernel<2, RW, kPB>;
        case 4: return (void*)search_kernel<4, RW, kPB>;
        case 8: return (void*)search_kernel<8, RW, kPB>;
        case 16: return (void*)search_kernel<16, RW, kPB>;
        default: return (void*)search_kernel<32, RW, kPB>;
    }
}

void* pick_kernel(uint32_t efw, uint32_t rw) {
    if (rw == 1) return pick_kernel_ef<1>(efw);
    if (rw == 2) return pick_kernel_ef<2>(efw);
    return pick_kernel_ef<4>(efw);
}

uint32_t pow2ceil(uint32_t x) {
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

struct Plan {
    void* fn;
    uint32_t efw, rw, G, warp_bytes, block_bytes;
};

Plan make_plan(const DevIndex& ix, uint32_t ef, uint32_t vis_log2, uint32_t tie_cap) {
    Plan p;
    p.efw = pow2ceil((ef + 31) / 32);
    p.rw = pow2ceil((ix.R + 31) / 32);
    p.G = pow2ceil((ix.W + 2) / 3);
    if (p.G > 32) p.G = 32;
    p.fn = pick_kernel(p.efw, p.rw);
    // the tie-add staging area lives in the cid region beyond RM/4 words: needs
    // RM u32 more -> cid region is 4*RM bytes; staging uses [RM/4, RM/4 + RM)
    const SmemLayout L = smem_layout(p.efw * 32, p.rw * 32, ix.W, tie_cap, 1u << vis_log2);
    p.warp_bytes = L.total;
    p.block_bytes = p.warp_bytes * kWarpsPerBlock;
    return p;
}

}  // namespace

qvg_status plan_search(const SearchLaunch& a, int device, uint64_t* grid_out) {
    const Plan p = make_plan(a.ix, a.ef, a.vis_log2, a.tie_cap);
    cudaError_t e = cudaFuncSetAttribute(p.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)p.block_bytes);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(search)");
    int per_sm = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p.fn, kWarpsPerBlock * 32,
                                                      p.block_bytes);
    if (e != cudaSuccess) return cuda_status(e, "occupancy(search)");
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (per_sm < 1) {
        set_error("search: per-warp shared memory too large (reduce visited_slots / tie_capacity)");
        return QVG_INVALID_ARGUMENT;
    }
    uint64_t want = (a.nq + kWarpsPerBlock - 1) / kWarpsPerBlock;
    uint64_t grid = (uint64_t)per_sm * sms;
    if (want < grid) grid = want;
    if (grid < 1) grid = 1;
    *grid_out = grid;
    return QVG_OK;
}

qvg_status launch_search(const SearchLaunch& a, uint64_t grid, cudaStream_t s) {
    const Plan p = make_plan(a.ix, a.ef, a.vis_log2, a.tie_cap);
    void* args[] = {(void*)&a, (void*)&p.warp_bytes, (void*)&p.G};
    cudaError_t e = cudaLaunchKernel(p.fn, dim3((unsigned)grid), dim3(kWarpsPerBlock * 32),
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

// K5 — GPU batched BQ-space Vamana construction (secondary path ★(2),
// BASELINE config 5).  Reference: build_index / stage0_preinstall /
// select_entry_point / link_node (builder.cpp:59-155), robust_prune and
// insert_bidirectional (graph.hpp:162-227).
//
// Stage 0 (exact w.r.t. the reference): every row is normalised and encoded by
// the query-path encode kernel (normalize_l2 + encode_sm2, bit-exact); the entry
// point is the approximate medoid — centroid summed in double in row order,
// normalised, argmax of the 4-chain dot with smallest-id ties
// (builder.cpp:90-120).  The insertion order is the reference's own
// std::shuffle(mt19937_64(seed)).
//
// Stage 1 (batched; the reference inserts one node at a time under per-slot
// spinlocks, which is nondeterministic with threads > 1): batches
// of prefix-doubling size (1, 1, 2, 4, ... up to `batch`), per batch
//   1. beam search (ef_c) from the entry for every batch node with the search
//      kernel (pool output, no rerank) over the graph as it stands;
//   2. RobustPrune(node, pool \ {node} [∪ N_out(node) on later passes], alpha, R)
//      — greedy over (dist,id)-sorted candidates, keep c iff for every kept s
//      !(float(c.dist) > alpha * float(d(c, s))) (graph.hpp:162-183);
//   3. reverse edges grouped by target (CUB radix sort): if the union of the
//      target's row and its new sources fits in R they are appended in order,
//      otherwise the target is re-pruned over the union (graph.hpp:207-226).
// Two passes give alpha = 1.0 then `alpha`.  The result is deterministic.
// Candidate and selected code rows are staged in shared memory by TMA gather4.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <numeric>
#include <random>
#include <vector>

#include "bq_device.cuh"
#include "qvg_internal.cuh"

namespace qvg {

qvg_status make_handle_from_device(int device, uint64_t n, uint32_t dim, uint32_t R,
                                   uint32_t entry, qvg_index** out);
void destroy_handle(qvg_index* h);

namespace {

using namespace dev;
constexpr unsigned kFull = 0xFFFFFFFFu;
// candidates a prune task holds: the kMaxCand closest by (dist, id) of its
// existing row and new candidates (streamed in chunks of 32; kCandBuf is the
// bitonic-sort capacity of kMaxCand + 32 rounded to a power of two)
constexpr uint32_t kMaxCand = 480;
constexpr uint32_t kCandBuf = 512;

// ---- stage 0: entry point (builder.cpp:90-120) --------------------------------
__global__ void centroid_kernel(const float* __restrict__ cold, uint64_t n, uint32_t dim,
                                uint32_t Dp, double* __restrict__ c) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= dim) return;
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s = __dadd_rn(s, (double)__ldg(cold + i * Dp + j));
    c[j] = s;
}

__global__ void center_kernel(const double* __restrict__ c, uint32_t dim, float* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double norm = 0.0;
    for (uint32_t j = 0; j < dim; ++j) norm = __fma_rn(c[j], c[j], norm);
    norm = __dsqrt_rn(norm);
    for (uint32_t j = 0; j < dim; ++j) out[j] = norm > 0.0 ? __double2float_rn(__ddiv_rn(c[j], norm)) : 0.0f;
}

__device__ __forceinline__ uint32_t orderable(float f) {
    if (f == 0.0f) f = 0.0f;  // -0 == +0 under the reference's `>`
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// argmax of dot_f32(row, center) with smallest-id ties (strict > scan)
__global__ void entry_kernel(const float* __restrict__ cold, uint64_t n, uint32_t dim, uint32_t Dp,
                             const float* __restrict__ center, unsigned long long* best) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* v = cold + i * Dp;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    uint32_t t = 0;
    for (; t + 4 <= dim; t += 4) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(v + t));
        const float4 b = __ldg(reinterpret_cast<const float4*>(center + t));
        s0 = __fma_rn((double)a.x, (double)b.x, s0);
        s1 = __fma_rn((double)a.y, (double)b.y, s1);
        s2 = __fma_rn((double)a.z, (double)b.z, s2);
        s3 = __fma_rn((double)a.w, (double)b.w, s3);
    }
    for (; t < dim; ++t) s0 = __fma_rn((double)v[t], (double)center[t], s0);
    const float f = __double2float_rn(__dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3)));
    const unsigned long long key = ((unsigned long long)orderable(f) << 32) | (0xFFFFFFFFu - (uint32_t)i);
    atomicMax(best, key);
}

// ---- stage 1 helpers ------------------------------------------------------------
__global__ void gather_codes_kernel(const uint4* __restrict__ codes, uint32_t W,
                                    const uint32_t* __restrict__ ids, uint32_t nb,
                                    uint4* __restrict__ out) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= (uint64_t)nb * W) return;
    out[t] = codes[(uint64_t)ids[t / W] * W + (t % W)];
}

// (target, source) pairs of the batch's new forward edges; empty = sentinel key
__global__ void reverse_pairs_kernel(const uint32_t* __restrict__ adj, uint32_t RS, uint32_t R,
                                     const uint32_t* __restrict__ batch, uint32_t nb,
                                     uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= (uint64_t)nb * R) return;
    const uint32_t u = batch[t / R];
    const uint32_t v = adj[(uint64_t)u * RS + (t % R)];
    keys[t] = v;
    vals[t] = u;
}

__global__ void segment_flags_kernel(const uint32_t* __restrict__ keys, uint32_t n,
                                     uint8_t* __restrict__ flags) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    flags[i] = keys[i] != kSentinel && (i == 0 || keys[i] != keys[i - 1]);
}

// After DeviceSelect wrote the segment starts seg[0..nseg): seg[nseg] = index
// of the first sentinel key (end of the valid pairs) and tg[i] = keys[seg[i]].
__global__ void segment_tail_kernel(const uint32_t* __restrict__ keys, uint32_t n,
                                    const uint32_t* __restrict__ nseg, uint32_t* __restrict__ seg,
                                    uint32_t* __restrict__ tg) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t ns = *nseg;
    if (i < ns) tg[i] = keys[seg[i]];
    const bool valid = keys[i] != kSentinel;
    const bool next_invalid = i + 1 == n || keys[i + 1] == kSentinel;
    if (valid && next_invalid) seg[ns] = i + 1;
    if (i == 0 && !valid) seg[ns] = 0;
}

// Prune tasks.  Task t: target v = targets[t]; new candidates cand_ids[lo,hi)
// with optional known distances; optionally the target's current row.
struct PruneArgs {
    DevIndex ix;
    uint32_t* adj;                 // rows rewritten in place (one task per row)
    uint32_t ntasks;
    const uint32_t* targets;
    const uint32_t* cand_ids;
    const uint32_t* cand_dists;    // nullable: distances d(target, c) aligned with cand_ids
    const uint32_t* seg;           // nullable: task t uses [seg[t], seg[t+1]) (seg[ntasks] = end)
    uint32_t stride;               // else task t uses [t*stride, t*stride + counts[t])
    const uint32_t* counts;
    int include_existing;
    int append_if_fits;
    float alpha;
    uint32_t R;
    unsigned long long* reprunes;
    unsigned long long* counter;   // task queue
    // function-level mode (qvg_robust_prune): task t's selection goes to
    // out_sel[t*R ...) and its size to out_cnt[t] instead of the adjacency row;
    // targets may be null (no target: every distance is given)
    uint32_t* out_sel;
    uint32_t* out_cnt;
    // extra candidates with known distances (the build search's expanded-node
    // list, Vamana's visited set V): keys dist<<33 | id, ext_n[t] of them at
    // ext_keys[t * ext_stride ...]; nullable
    const uint64_t* ext_keys;
    const uint32_t* ext_n;
    uint32_t ext_stride;
};

constexpr int kPruneWarps = 2;

struct PruneSmem {
    uint32_t keys_off, sel_ids, sel_codes, stage, vcode, bar, total;
};

__host__ __device__ inline PruneSmem prune_layout(uint32_t W, uint32_t R) {
    PruneSmem L;
    uint32_t o = 0;
    auto take = [&](uint32_t b, uint32_t al) {
        o = (o + al - 1) & ~(al - 1);
        const uint32_t at = o;
        o += b;
        return at;
    };
    const uint32_t gs = (64u * W + 127u) & ~127u;  // 4-row TMA group
    L.bar = take(16, 16);
    L.keys_off = take(8 * kCandBuf, 16);
    L.sel_ids = take(4 * R, 16);
    L.sel_codes = take(16 * W * R, 16);
    L.stage = take(8 * gs, 128);  // 32 candidate rows per TMA round
    L.vcode = take(16 * W, 16);
    L.total = (o + 127u) & ~127u;
    return L;
}

__global__ void __launch_bounds__(kPruneWarps * 32)
    prune_kernel(const __grid_constant__ CUtensorMap tmap, const PruneArgs a, const uint32_t warp_bytes) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const DevIndex ix = a.ix;
    const uint32_t W = ix.W, rowb = 16u * W, gs = (64u * W + 127u) & ~127u;
    const PruneSmem L = prune_layout(W, a.R);
    unsigned char* base = smem_raw + (size_t)wib * warp_bytes;
    uint64_t* bar = reinterpret_cast<uint64_t*>(base + L.bar);
    uint64_t* keys = reinterpret_cast<uint64_t*>(base + L.keys_off);
    uint32_t* sel = reinterpret_cast<uint32_t*>(base + L.sel_ids);
    uint4* selc = reinterpret_cast<uint4*>(base + L.sel_codes);
    unsigned char* stage = base + L.stage;
    uint4* vc = reinterpret_cast<uint4*>(base + L.vcode);
    if (lane == 0) {
        mbar_init(bar);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t phase = 0;
    const uint32_t lt_mask = (1u << lane) - 1u;

    // stage rows ids[r0..r0+cnt) (cnt <= 32) into `stage` (row j at (j/4)*gs + (j%4)*rowb)
    auto fetch = [&](const uint32_t* ids_smem_or_null, const uint64_t* key_src, uint32_t r0,
                     uint32_t cnt) {
        const uint32_t ng = (cnt + 3u) >> 2;
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_expect_tx(bar, ng * 4u * rowb);
        __syncwarp();
        if (lane < ng) {
            uint32_t id[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t r = 4u * lane + j < cnt ? 4u * lane + j : 4u * lane;
                id[j] = ids_smem_or_null ? ids_smem_or_null[r0 + r] : (uint32_t)key_src[r0 + r];
            }
            tma_gather4(stage + lane * gs, &tmap, 0, id[0], id[1], id[2], id[3], bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1u;
    };
    auto srow = [&](uint32_t j) {
        return reinterpret_cast<const uint4*>(stage + (j >> 2) * gs + (j & 3u) * rowb);
    };

    for (;;) {
        unsigned long long tt = 0;
        if (lane == 0) tt = atomicAdd(a.counter, 1ull);
        tt = __shfl_sync(kFull, tt, 0);
        if (tt >= a.ntasks) break;
        const uint32_t t = (uint32_t)tt;
        const uint32_t v = a.targets ? a.targets[t] : kSentinel;
        uint32_t lo, hi;
        if (a.seg) {
            lo = a.seg[t];
            hi = a.seg[t + 1];
        } else {
            lo = t * a.stride;
            hi = lo + a.counts[t];
        }
        uint32_t* vrow = v != kSentinel ? a.adj + (size_t)v * ix.RS : nullptr;
        if (v != kSentinel)
            for (uint32_t w = lane; w < W; w += 32) vc[w] = ix.codes[(size_t)v * W + w];
        // existing row (kept in registers: slot lane*... up to R <= 128)
        uint32_t ex[4];
        uint32_t nex = 0;
        if (a.include_existing) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t s = lane + 32u * j;
                ex[j] = s < a.R ? vrow[s] : kSentinel;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) nex += __popc(__ballot_sync(kFull, ex[j] != kSentinel));
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) ex[j] = kSentinel;
        }
        const uint32_t nnew = hi - lo;
        // reverse fast path: existing + new (not already present) fit -> append
        if (a.append_if_fits) {
            // count new sources not already in the row (rows hold no duplicates;
            // sources within a segment are distinct: one forward edge per pair)
            uint32_t add = 0;
            for (uint32_t i = lane; i < nnew; i += 32) {
                const uint32_t u = a.cand_ids[lo + i];
                bool present = false;
                for (uint32_t s = 0; s < nex; ++s) present |= vrow[s] == u;
                add += !present;
            }
            for (int off = 16; off > 0; off >>= 1) add += __shfl_xor_sync(kFull, add, off);
            if (nex + add <= a.R) {
                uint32_t pos = nex;
                for (uint32_t i0 = 0; i0 < nnew; i0 += 32) {
                    const uint32_t i = i0 + lane;
                    bool keep = false;
                    uint32_t u = 0;
                    if (i < nnew) {
                        u = a.cand_ids[lo + i];
                        keep = true;
                        for (uint32_t s = 0; s < nex; ++s) keep &= vrow[s] != u;
                    }
                    const unsigned b = __ballot_sync(kFull, keep);
                    if (keep) vrow[pos + __popc(b & lt_mask)] = u;
                    pos += __popc(b);
                }
                __syncwarp();
                continue;
            }
            if (lane == 0) atomicAdd(a.reprunes, 1ull);
        }
        // d(v, c) for the keys in [b, e) whose distance is unknown (TMA-staged
        // rows, lane per row)
        auto score_unknown = [&](uint32_t b, uint32_t e) {
            for (uint32_t r0 = b; r0 < e; r0 += 32) {
                const uint32_t cnt = min(32u, e - r0);
                bool unknown = false;
                if (lane < cnt) unknown = (keys[r0 + lane] >> 32) == kSentinel;
                if (!__any_sync(kFull, unknown)) continue;
                fetch(nullptr, keys, r0, cnt);
                if (unknown) {
                    const uint4* rp = srow(lane);
                    uint32_t d = 0;
                    for (uint32_t w = 0; w < W; ++w) d += sm2_chunk(vc[w], rp[w]);
                    keys[r0 + lane] = ((uint64_t)d << 32) | (uint32_t)keys[r0 + lane];
                }
                __syncwarp();
            }
        };
        // ascending (dist, id) order of keys[0, cnt) (bitonic over the next power of two)
        auto sort_keys = [&](uint32_t cnt) {
            uint32_t np2 = 1;
            while (np2 < cnt) np2 <<= 1;
            for (uint32_t i = cnt + lane; i < np2; i += 32) keys[i] = ~0ull;
            __syncwarp();
            for (uint32_t size = 2; size <= np2; size <<= 1) {
                for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                    for (uint32_t i = lane; i < np2; i += 32) {
                        const uint32_t j = i ^ stride;
                        if (j > i) {
                            const uint64_t x = keys[i], y = keys[j];
                            const bool up = (i & size) == 0;
                            if ((x > y) == up) {
                                keys[i] = y;
                                keys[j] = x;
                            }
                        }
                    }
                    __syncwarp();
                }
            }
        };
        // ---- candidate keys (dist<<32 | id): the existing row, then the new
        // candidates in chunks of 32.  Whenever more than kMaxCand are held the
        // unknown distances are computed and only the kMaxCand closest keys by
        // (dist, id) are kept, so a hub target that receives thousands of
        // reverse edges in one batch still re-prunes over its closest
        // candidates (graph.hpp:207-226 re-prunes over row + node)
        uint32_t nc = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool have = ex[j] != kSentinel;
            const unsigned b = __ballot_sync(kFull, have);
            if (have) keys[nc + __popc(b & lt_mask)] = ((uint64_t)kSentinel << 32) | ex[j];
            nc += __popc(b);
        }
        for (uint32_t i0 = 0; i0 < nnew; i0 += 32) {
            const uint32_t i = i0 + lane;
            if (i < nnew) {
                const uint32_t c = a.cand_ids[lo + i];
                const uint32_t d = a.cand_dists ? a.cand_dists[lo + i] : kSentinel;
                keys[nc + lane] = ((uint64_t)d << 32) | c;
            }
            nc += min(32u, nnew - i0);
            __syncwarp();
            if (nc > kMaxCand) {
                score_unknown(0, nc);
                sort_keys(nc);
                nc = kMaxCand;
            }
        }
        // Vamana's visited set (expanded nodes) as further candidates; a node
        // also in the pool gives an identical key, dropped after the sort
        const uint32_t next = a.ext_keys ? a.ext_n[t] : 0u;
        for (uint32_t i0 = 0; i0 < next; i0 += 32) {
            const uint32_t i = i0 + lane;
            if (i < next) {
                const uint64_t k = a.ext_keys[(size_t)t * a.ext_stride + i];
                keys[nc + lane] = ((k >> 33) << 32) | (uint32_t)k;
            }
            nc += min(32u, next - i0);
            __syncwarp();
            if (nc > kMaxCand) {
                score_unknown(0, nc);
                sort_keys(nc);
                nc = kMaxCand;
            }
        }
        __syncwarp();
        score_unknown(0, nc);
        sort_keys(nc);
        // ---- greedy RobustPrune (graph.hpp:162-183)
        uint32_t ns = 0;
        for (uint32_t r0 = 0; r0 < nc && ns < a.R; r0 += 32) {
            const uint32_t cnt = min(32u, nc - r0);
            fetch(nullptr, keys, r0, cnt);
            for (uint32_t j = 0; j < cnt && ns < a.R; ++j) {
                const uint64_t kk = keys[r0 + j];
                const uint32_t cid = (uint32_t)kk;
                if (cid == v) continue;                                       // self
                if (r0 + j > 0 && (uint32_t)keys[r0 + j - 1] == cid) continue;  // duplicate
                const float cd = (float)(uint32_t)(kk >> 32);
                const uint4* crow = srow(j);
                bool violate = false;
                for (uint32_t s = lane; s < ns; s += 32) {
                    const uint4* sr = selc + (size_t)s * W;
                    uint32_t d = 0;
                    for (uint32_t w = 0; w < W; ++w) d += sm2_chunk(crow[w], sr[w]);
                    violate |= cd > __fmul_rn(a.alpha, (float)d);
                }
                if (__any_sync(kFull, violate)) continue;
                for (uint32_t w = lane; w < W; w += 32) selc[(size_t)ns * W + w] = crow[w];
                if (lane == 0) sel[ns] = cid;
                ++ns;
                __syncwarp();
            }
        }
        __syncwarp();
        if (a.out_sel) {
            for (uint32_t s = lane; s < ns; s += 32) a.out_sel[(size_t)t * a.R + s] = sel[s];
            if (lane == 0) a.out_cnt[t] = ns;
        } else {
            for (uint32_t s = lane; s < ix.RS; s += 32) vrow[s] = s < ns ? sel[s] : kSentinel;
        }
        __syncwarp();
    }
}

__global__ void degree_kernel(const uint32_t* __restrict__ adj, uint64_t n, uint32_t RS,
                              unsigned long long* sum, uint32_t* mn, uint32_t* mx) {
    const uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (u >= n) return;
    uint32_t d = 0;
    for (uint32_t s = 0; s < RS; ++s) d += adj[u * RS + s] != kSentinel;
    atomicAdd(sum, (unsigned long long)d);
    atomicMin(mn, d);
    atomicMax(mx, d);
}

}  // namespace
}  // namespace qvg

using namespace qvg;

extern "C" qvg_status qvg_build(const float* data, uint64_t n, uint32_t dim,
                                const qvg_build_params* p, int device, qvg_index** out,
                                qvg_build_stats* stats) {
    if (out) *out = nullptr;
    if (!data || !p || !out) {
        set_error("qvg_build: null argument");
        return QVG_INVALID_ARGUMENT;
    }
    // BuildParams::validate (graph.hpp:41-46) + stage0 checks (builder.cpp:61-66)
    if (p->m < 1) { set_error("BuildParams: m must be >= 1"); return QVG_INVALID_ARGUMENT; }
    if (p->ef_c < 1) { set_error("BuildParams: ef_c must be >= 1"); return QVG_INVALID_ARGUMENT; }
    if (!(p->alpha >= 1.0f)) { set_error("BuildParams: alpha must be >= 1.0"); return QVG_INVALID_ARGUMENT; }
    if (n == 0) { set_error("stage0_preinstall: no vectors"); return QVG_INVALID_ARGUMENT; }
    if (dim == 0) { set_error("stage0_preinstall: zero dimension"); return QVG_INVALID_ARGUMENT; }
    const uint32_t R = 2 * p->m;
    if (R > kMaxDegree) { set_error("qvg_build: 2m exceeds the supported max degree"); return QVG_NOT_IMPLEMENTED; }
    if (p->ef_c > kMaxEf) { set_error("qvg_build: ef_c too large"); return QVG_NOT_IMPLEMENTED; }
    const auto t_start = std::chrono::steady_clock::now();
    qvg_index* h = nullptr;
    qvg_status st = make_handle_from_device(device, n, dim, R, 0, &h);
    if (st != QVG_OK) return st;
    h->m = p->m;
    h->alpha = p->alpha;
    DevIndex& ix = h->ix;
    cudaStream_t s = h->stream;
    std::vector<void*> tmp;
    auto dalloc = [&](size_t bytes) -> void* {
        void* q = nullptr;
        if (cudaMalloc(&q, bytes) != cudaSuccess) return nullptr;
        tmp.push_back(q);
        return q;
    };
    auto fail = [&](qvg_status code) {
        for (void* q : tmp) cudaFree(q);
        destroy_handle(h);
        return code;
    };
    cudaError_t e;
    // ---- stage 0: normalise + encode straight into the cold / code stores
    float* d_x = static_cast<float*>(dalloc(n * (size_t)dim * 4));
    int32_t* d_st = static_cast<int32_t*>(dalloc(n * 4));
    uint32_t* d_flags = static_cast<uint32_t*>(dalloc(64));
    if (!d_x || !d_st || !d_flags) return fail(cuda_status(cudaErrorMemoryAllocation, "qvg_build"));
    e = cudaMemcpyAsync(d_x, data, n * (size_t)dim * 4, cudaMemcpyDefault, s);
    if (e != cudaSuccess) return fail(cuda_status(e, "qvg_build: upload"));
    cudaMemsetAsync(d_flags, 0, 64, s);
    launch_encode(d_x, n, dim, ix.Dp, const_cast<float*>(ix.cold), const_cast<uint4*>(ix.codes),
                  nullptr, d_st, d_flags, s);
    uint32_t hflags = 0;
    cudaMemcpyAsync(&hflags, d_flags, 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (hflags) {
        set_error("normalize_l2: zero or non-finite norm (or non-finite coordinate) in build data");
        return fail(QVG_INVALID_ARGUMENT);
    }
    cudaFree(d_x);
    tmp.erase(std::find(tmp.begin(), tmp.end(), (void*)d_x));
    // entry point
    double* d_c = static_cast<double*>(dalloc(dim * 8ull));
    float* d_center = static_cast<float*>(dalloc(((dim + 3) & ~3u) * 4ull));
    unsigned long long* d_best = static_cast<unsigned long long*>(dalloc(8));
    if (!d_c || !d_center || !d_best) return fail(cuda_status(cudaErrorMemoryAllocation, "qvg_build"));
    cudaMemsetAsync(d_center, 0, ((dim + 3) & ~3u) * 4ull, s);
    cudaMemsetAsync(d_best, 0, 8, s);
    centroid_kernel<<<(dim + 127) / 128, 128, 0, s>>>(ix.cold, n, dim, ix.Dp, d_c);
    center_kernel<<<1, 32, 0, s>>>(d_c, dim, d_center);
    entry_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(ix.cold, n, dim, ix.Dp, d_center, d_best);
    unsigned long long best = 0;
    cudaMemcpyAsync(&best, d_best, 8, cudaMemcpyDeviceToHost, s);
    // empty graph
    cudaMemsetAsync(const_cast<uint32_t*>(ix.adj), 0xFF, n * (size_t)ix.RS * 4, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(cuda_status(e, "qvg_build: stage0"));
    ix.entry = 0xFFFFFFFFu - (uint32_t)(best & 0xFFFFFFFFu);

    // ---- insertion order: the reference's std::shuffle(mt19937_64(seed))
    std::vector<uint32_t> order(n);
    std::iota(order.begin(), order.end(), 0u);
    std::mt19937_64 rng(p->seed);
    std::shuffle(order.begin(), order.end(), rng);
    uint32_t* d_order = static_cast<uint32_t*>(dalloc(n * 4ull));
    if (!d_order) return fail(cuda_status(cudaErrorMemoryAllocation, "qvg_build"));
    cudaMemcpyAsync(d_order, order.data(), n * 4ull, cudaMemcpyHostToDevice, s);

    // ---- per-batch buffers
    const uint32_t maxb = p->batch ? p->batch : 65536u;
    const uint32_t L = p->ef_c;
    uint4* d_qc = static_cast<uint4*>(dalloc((size_t)maxb * ix.W * 16));
    uint32_t* d_pi = static_cast<uint32_t*>(dalloc((size_t)maxb * L * 4));
    uint32_t* d_pd = static_cast<uint32_t*>(dalloc((size_t)maxb * L * 4));
    uint32_t* d_pn = static_cast<uint32_t*>(dalloc((size_t)maxb * 4));
    // prune candidates: bit 0 / bit 1 = also the expanded-node list V of the
    // first / the final (alpha) pass's searches (qvg.h prune_candidates)
    const uint32_t vmode = p->prune_candidates ? p->prune_candidates : 3u;
    const uint32_t xcap = 2 * L < kMaxCand ? 2 * L : kMaxCand;
    uint64_t* d_ex = static_cast<uint64_t*>(dalloc((size_t)maxb * xcap * 8));
    uint32_t* d_exn = static_cast<uint32_t*>(dalloc((size_t)maxb * 4));
    const size_t npairs = (size_t)maxb * R;
    uint32_t* d_k0 = static_cast<uint32_t*>(dalloc(npairs * 4));
    uint32_t* d_v0 = static_cast<uint32_t*>(dalloc(npairs * 4));
    uint32_t* d_k1 = static_cast<uint32_t*>(dalloc(npairs * 4));
    uint32_t* d_v1 = static_cast<uint32_t*>(dalloc(npairs * 4));
    uint8_t* d_fl = static_cast<uint8_t*>(dalloc(npairs));
    uint32_t* d_seg = static_cast<uint32_t*>(dalloc((npairs + 2) * 4));
    uint32_t* d_nseg = static_cast<uint32_t*>(dalloc(8));
    unsigned long long* d_ctr = static_cast<unsigned long long*>(dalloc(64));
    if (!d_qc || !d_pi || !d_pd || !d_pn || !d_k0 || !d_v0 || !d_k1 || !d_v1 || !d_fl || !d_seg ||
        !d_nseg || !d_ctr || !d_ex || !d_exn)
        return fail(cuda_status(cudaErrorMemoryAllocation, "qvg_build"));
    size_t sort_bytes = 0, sel_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, d_k0, d_k1, d_v0, d_v1, (int)npairs);
    cub::DeviceSelect::Flagged(nullptr, sel_bytes, cub::CountingInputIterator<uint32_t>(0), d_fl,
                               d_seg, d_nseg, (int)npairs);
    void* d_cub = dalloc(std::max(sort_bytes, sel_bytes));
    if (!d_cub) return fail(cuda_status(cudaErrorMemoryAllocation, "qvg_build"));

    // search launch template (pool output, no rerank)
    SearchLaunch sa{};
    sa.ix = ix;
    sa.qcodes = d_qc;
    sa.ef = L;
    sa.k = 1;
    sa.entry = ix.entry;
    sa.tie_cap = ((L < 64 ? 64u : L) + 3u) & ~3u;
    sa.vis_log2 = auto_visited_log2(ix, L, sa.tie_cap, device);
    sa.do_rerank = 0;
    sa.pool_ids = d_pi;
    sa.pool_dists = d_pd;
    sa.pool_n = d_pn;
    sa.counter = d_ctr;
    sa.flags = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(d_ctr) + 32);
    PlanInfo pinfo;
    uint64_t grid_full = 0;
    sa.nq = maxb;
    if ((st = plan_search(sa, device, &grid_full, &pinfo)) != QVG_OK) return fail(st);

    // prune kernel setup
    const PruneSmem PL = prune_layout(ix.W, R);
    const uint32_t pwb = PL.total, pblock = pwb * kPruneWarps;
    e = cudaFuncSetAttribute(prune_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pblock);
    if (e != cudaSuccess) return fail(cuda_status(e, "qvg_build: prune smem"));
    int prune_per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&prune_per_sm, prune_kernel, kPruneWarps * 32, pblock);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (prune_per_sm < 1) {
        set_error("qvg_build: prune kernel does not fit (code rows too wide)");
        return fail(QVG_NOT_IMPLEMENTED);
    }
    unsigned long long* d_repr = d_ctr + 2;
    auto run_prune = [&](PruneArgs pa) -> qvg_status {
        if (pa.ntasks == 0) return QVG_OK;
        pa.counter = d_ctr + 1;
        cudaMemsetAsync(pa.counter, 0, 8, s);
        uint64_t want = (pa.ntasks + kPruneWarps - 1) / kPruneWarps;
        uint64_t g = (uint64_t)prune_per_sm * sms;
        if (want < g) g = want;
        prune_kernel<<<(unsigned)g, kPruneWarps * 32, pblock, s>>>(h->tmap, pa, pwb);
        const cudaError_t e2 = cudaGetLastError();
        return e2 == cudaSuccess ? QVG_OK : cuda_status(e2, "qvg_build: prune");
    };
    cudaMemsetAsync(d_repr, 0, 8, s);

    const uint32_t passes = p->passes == 2 ? 2u : 1u;
    uint64_t nbatches = 0;
    for (uint32_t pass = 0; pass < passes; ++pass) {
        const float alpha = (passes == 2 && pass == 0) ? 1.0f : p->alpha;
        uint64_t done = 0;
        while (done < n) {
            uint64_t b = pass == 0 ? std::max<uint64_t>(1, std::min<uint64_t>(maxb, done)) : maxb;
            if (done + b > n) b = n - done;
            const uint32_t nb = (uint32_t)b;
            const uint32_t* batch = d_order + done;
            // 1. beam search of every batch node over the current graph
            gather_codes_kernel<<<(unsigned)(((uint64_t)nb * ix.W + 255) / 256), 256, 0, s>>>(
                ix.codes, ix.W, batch, nb, d_qc);
            cudaMemsetAsync(d_ctr, 0, 8, s);
            sa.nq = nb;
            sa.ix = ix;
            const bool use_v = (vmode >> (pass + 1 == passes ? 1u : 0u)) & 1u;
            sa.exp_out = use_v ? d_ex : nullptr;
            sa.exp_n = d_exn;
            sa.exp_cap = xcap;
            const uint64_t wpb = pinfo.warps_per_block ? pinfo.warps_per_block : kWarpsPerBlock;
            uint64_t g = (nb + wpb - 1) / wpb;
            if (g > grid_full) g = grid_full;
            if ((st = launch_search(sa, h->has_tmap ? &h->tmap : nullptr, g, s)) != QVG_OK) return fail(st);
            // 2. forward prune over the pool (+ current row on later passes)
            PruneArgs fa{};
            fa.ix = ix;
            fa.adj = const_cast<uint32_t*>(ix.adj);
            fa.ntasks = nb;
            fa.targets = batch;
            fa.cand_ids = d_pi;
            fa.cand_dists = d_pd;
            fa.stride = L;
            fa.counts = d_pn;
            fa.include_existing = pass > 0;
            fa.append_if_fits = 0;
            fa.alpha = alpha;
            fa.R = R;
            fa.reprunes = d_repr;
            fa.ext_keys = use_v ? d_ex : nullptr;
            fa.ext_n = d_exn;
            fa.ext_stride = xcap;
            if ((st = run_prune(fa)) != QVG_OK) return fail(st);
            // 3. reverse edges grouped by target
            const uint32_t np = nb * R;
            reverse_pairs_kernel<<<(np + 255) / 256, 256, 0, s>>>(ix.adj, ix.RS, R, batch, nb, d_k0, d_v0);
            size_t sb = sort_bytes;
            cub::DeviceRadixSort::SortPairs(d_cub, sb, d_k0, d_k1, d_v0, d_v1, (int)np, 0, 32, s);
            segment_flags_kernel<<<(np + 255) / 256, 256, 0, s>>>(d_k1, np, d_fl);
            size_t sl = sel_bytes;
            cub::DeviceSelect::Flagged(d_cub, sl, cub::CountingInputIterator<uint32_t>(0), d_fl, d_seg,
                                       d_nseg, (int)np, s);
            // close the last segment at the first sentinel key (they sort last)
            // and gather each segment's target id
            uint32_t* d_tg = d_k0;  // free after the sort
            segment_tail_kernel<<<(np + 255) / 256, 256, 0, s>>>(d_k1, np, d_nseg, d_seg, d_tg);
            uint32_t nseg = 0;
            cudaMemcpyAsync(&nseg, d_nseg, 4, cudaMemcpyDeviceToHost, s);
            e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) return fail(cuda_status(e, "qvg_build: batch"));
            PruneArgs ra{};
            ra.ix = ix;
            ra.adj = const_cast<uint32_t*>(ix.adj);
            ra.ntasks = nseg;
            ra.targets = nullptr;
            ra.cand_ids = d_v1;
            ra.cand_dists = nullptr;
            ra.seg = d_seg;
            ra.include_existing = 1;
            ra.append_if_fits = 1;
            ra.alpha = alpha;
            ra.R = R;
            ra.reprunes = d_repr;
            ra.targets = d_tg;
            if ((st = run_prune(ra)) != QVG_OK) return fail(st);
            done += b;
            ++nbatches;
        }
    }
    // ---- stats
    uint32_t* d_mm = static_cast<uint32_t*>(dalloc(16));
    unsigned long long* d_sum = static_cast<unsigned long long*>(dalloc(8));
    if (!d_mm || !d_sum) return fail(cuda_status(cudaErrorMemoryAllocation, "qvg_build"));
    const uint32_t init[2] = {0xFFFFFFFFu, 0u};
    cudaMemcpyAsync(d_mm, init, 8, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(d_sum, 0, 8, s);
    degree_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ix.adj, n, ix.RS, d_sum, d_mm, d_mm + 1);
    unsigned long long hsum = 0, hrep = 0;
    uint32_t hmm[2] = {0, 0};
    cudaMemcpyAsync(&hsum, d_sum, 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(hmm, d_mm, 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&hrep, d_repr, 8, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(cuda_status(e, "qvg_build: finish"));
    for (void* q : tmp) cudaFree(q);
    if (stats) {
        stats->seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
        stats->reprunes = hrep;
        stats->batches = nbatches;
        stats->mean_degree = (double)hsum / (double)n;
        stats->min_degree = hmm[0];
        stats->max_degree = hmm[1];
    }
    *out = h;
    return QVG_OK;
}

// qivr::robust_prune (graph.hpp:162-183) as a batched device call over the
// index's BQ codes: the builder's own prune kernel in function-level mode.
extern "C" qvg_status qvg_robust_prune(qvg_index* h, uint64_t ntasks, const uint64_t* offsets,
                                       const uint32_t* cand_ids, const uint32_t* cand_dists,
                                       uint32_t max_degree, float alpha, uint32_t* out_ids,
                                       uint32_t* out_count) {
    if (!h || !offsets || !out_count || (ntasks && !out_ids)) {
        set_error("qvg_robust_prune: null argument");
        return QVG_INVALID_ARGUMENT;
    }
    if (max_degree < 1 || max_degree > kMaxDegree) {
        set_error("qvg_robust_prune: max_degree must be in [1, 128]");
        return QVG_INVALID_ARGUMENT;
    }
    if (ntasks == 0) return QVG_OK;
    if (!h->has_tmap) {
        set_error("qvg_robust_prune: code rows too wide for the TMA gather (W > 128)");
        return QVG_NOT_IMPLEMENTED;
    }
    std::lock_guard<std::mutex> lock(h->mu);
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
    const DevIndex& ix = h->ix;
    std::vector<uint64_t> off(ntasks + 1);
    e = cudaMemcpy(off.data(), offsets, (ntasks + 1) * 8, cudaMemcpyDefault);
    if (e != cudaSuccess) return cuda_status(e, "qvg_robust_prune: offsets");
    if (off[0] != 0) {
        set_error("qvg_robust_prune: offsets[0] must be 0");
        return QVG_INVALID_ARGUMENT;
    }
    for (uint64_t t = 0; t < ntasks; ++t) {
        if (off[t + 1] < off[t]) {
            set_error("qvg_robust_prune: offsets must be non-decreasing");
            return QVG_INVALID_ARGUMENT;
        }
        if (off[t + 1] - off[t] > kMaxCand) {
            set_error("qvg_robust_prune: more than 480 candidates in one task");
            return QVG_NOT_IMPLEMENTED;
        }
    }
    const uint64_t total = off[ntasks];
    if (total >= 0xFFFFFFFFull) {
        set_error("qvg_robust_prune: too many candidates");
        return QVG_NOT_IMPLEMENTED;
    }
    if (total && (!cand_ids || !cand_dists)) {
        set_error("qvg_robust_prune: null candidates");
        return QVG_INVALID_ARGUMENT;
    }
    std::vector<uint32_t> ids(total), seg(ntasks + 1);
    if (total) {
        e = cudaMemcpy(ids.data(), cand_ids, total * 4, cudaMemcpyDefault);
        if (e != cudaSuccess) return cuda_status(e, "qvg_robust_prune: candidates");
    }
    for (uint64_t i = 0; i < total; ++i)
        if (ids[i] >= ix.n) {
            set_error("qvg_robust_prune: candidate id out of range");
            return QVG_INVALID_ARGUMENT;
        }
    for (uint64_t t = 0; t <= ntasks; ++t) seg[t] = (uint32_t)off[t];
    cudaStream_t s = h->stream;
    std::vector<void*> tmp;
    auto dalloc = [&](size_t bytes) -> void* {
        void* q = nullptr;
        if (cudaMalloc(&q, bytes < 16 ? 16 : bytes) != cudaSuccess) return nullptr;
        tmp.push_back(q);
        return q;
    };
    auto done = [&](qvg_status st) {
        cudaStreamSynchronize(s);
        for (void* q : tmp) cudaFree(q);
        return st;
    };
    uint32_t* d_ids = static_cast<uint32_t*>(dalloc(total * 4));
    uint32_t* d_dst = static_cast<uint32_t*>(dalloc(total * 4));
    uint32_t* d_seg = static_cast<uint32_t*>(dalloc((ntasks + 1) * 4));
    uint32_t* d_sel = static_cast<uint32_t*>(dalloc(ntasks * max_degree * 4));
    uint32_t* d_cnt = static_cast<uint32_t*>(dalloc(ntasks * 4));
    unsigned long long* d_ctr = static_cast<unsigned long long*>(dalloc(16));
    if (!d_ids || !d_dst || !d_seg || !d_sel || !d_cnt || !d_ctr)
        return done(cuda_status(cudaErrorMemoryAllocation, "qvg_robust_prune"));
    e = cudaMemcpyAsync(d_ids, ids.data(), total * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_dst, cand_dists, total * 4, cudaMemcpyDefault, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(d_seg, seg.data(), (ntasks + 1) * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_ctr, 0, 16, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_sel, 0xFF, ntasks * max_degree * 4, s);
    if (e != cudaSuccess) return done(cuda_status(e, "qvg_robust_prune: upload"));
    PruneArgs pa{};
    pa.ix = ix;
    pa.adj = const_cast<uint32_t*>(ix.adj);  // not written in function-level mode
    pa.ntasks = (uint32_t)ntasks;
    pa.targets = nullptr;
    pa.cand_ids = d_ids;
    pa.cand_dists = d_dst;
    pa.seg = d_seg;
    pa.alpha = alpha;
    pa.R = max_degree;
    pa.reprunes = d_ctr + 1;
    pa.counter = d_ctr;
    pa.out_sel = d_sel;
    pa.out_cnt = d_cnt;
    const PruneSmem PL = prune_layout(ix.W, max_degree);
    const uint32_t pwb = PL.total, pblock = pwb * kPruneWarps;
    e = cudaFuncSetAttribute(prune_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pblock);
    if (e != cudaSuccess) return done(cuda_status(e, "qvg_robust_prune: smem"));
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, prune_kernel, kPruneWarps * 32, pblock);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
    if (per_sm < 1) {
        set_error("qvg_robust_prune: prune kernel does not fit (code rows too wide)");
        return done(QVG_NOT_IMPLEMENTED);
    }
    uint64_t g = (ntasks + kPruneWarps - 1) / kPruneWarps;
    if (g > (uint64_t)per_sm * sms) g = (uint64_t)per_sm * sms;
    prune_kernel<<<(unsigned)g, kPruneWarps * 32, pblock, s>>>(h->tmap, pa, pwb);
    e = cudaGetLastError();
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(out_ids, d_sel, ntasks * max_degree * 4, cudaMemcpyDefault, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_count, d_cnt, ntasks * 4, cudaMemcpyDefault, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return done(e == cudaSuccess ? QVG_OK : cuda_status(e, "qvg_robust_prune"));
}

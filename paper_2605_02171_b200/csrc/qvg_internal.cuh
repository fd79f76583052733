// Internal declarations shared by the qvg translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "../../include/qvg.h"

namespace qvg {

constexpr uint32_t kSentinel = 0xFFFFFFFFu;
constexpr uint32_t kMaxEf = 1024;
constexpr uint32_t kMaxDegree = 128;
constexpr int kWarpsPerBlock = 2;
constexpr int kGeoMaxWarps = 16;  // headline-geometry kernel: one block per SM, up to 16 warps

// HBM-resident index.  Layouts:
//   codes : n x W chunks of 16 B, chunk w = {pos word w, strong word w}
//   adj   : n x RS u32 (RS = R rounded up to 4), deduplicated, row order kept,
//           unused slots = kSentinel (degree is implicit)
//   cold  : n x Dp f32 (Dp = dim rounded up to 4, zero pad)
struct DevIndex {
    const uint4* codes;
    const uint32_t* adj;
    const float* cold;
    uint64_t n;
    uint32_t dim, W, R, RS, Dp, entry;
};

struct Buffer {
    void* p = nullptr;
    size_t bytes = 0;
};

struct PlanInfo {
    uint32_t warps_per_block = 0, smem_per_block = 0, resident_warps_per_sm = 0, sms = 0;
    uint64_t coop_cap = 0;  // resident CTAs of the latency kernel (0 = n/a)
    // bytes of per-query search state a warp saves when it suspends a query
    // (0 = the planned kernel cannot suspend)
    uint32_t susp_blob_bytes = 0;
};

}  // namespace qvg

struct qvg_index {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    qvg::DevIndex ix{};
    uint32_t m = 0;       // params.m (R = 2m for reference-built graphs)
    float alpha = 1.2f;
    void* d_codes = nullptr;
    void* d_adj = nullptr;
    void* d_cold = nullptr;
    // scratch, grown on demand
    qvg::Buffer s_in, s_qn, s_qc, s_qst, s_ids, s_sc, s_cnt, s_pool_i, s_pool_d, s_pool_n,
        s_qctr, s_counter, s_exact, s_pair_ids, s_pair_out, s_st, s_susp;
    cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    // pipelined upload of host queries (created on first use): copy stream,
    // its completion event, pinned ready counts published after each chunk
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_copy = nullptr;
    uint32_t* ready_host = nullptr;
    size_t ready_cap = 0;
    uint32_t* host_flags = nullptr;  // pinned: per-call status summary (D2H target)
    // TMA descriptor over the code rows (2-D: 2W u64 columns x n rows, box
    // {2W, 1}) for tile::gather4; valid iff has_tmap (W <= 128)
    alignas(64) CUtensorMap tmap;
    bool has_tmap = false;
    // launch plans keyed by (ef, tie capacity, visited-slot request, extra depth)
    struct PlanKey {
        uint32_t ef, tcap, vreq, xa, relax;
        bool operator<(const PlanKey& o) const {
            if (ef != o.ef) return ef < o.ef;
            if (tcap != o.tcap) return tcap < o.tcap;
            if (relax != o.relax) return relax < o.relax;
            return vreq != o.vreq ? vreq < o.vreq : xa < o.xa;
        }
    };
    std::map<PlanKey, std::pair<uint32_t, qvg::PlanInfo>> plans;  // -> (vis_log2, info)
    // one call at a time per handle: the scratch buffers, plan cache and stream
    // state above are shared by every call on it (concurrent callers serialise)
    std::mutex mu;
};

namespace qvg {

void set_error(const std::string& msg);
qvg_status cuda_status(cudaError_t e, const char* what);
qvg_status grow(Buffer& b, size_t bytes);
bool is_device_ptr(const void* p);

// kernels (encode.cu / search.cu)
// flags (nullable): atomicOr(1 << status) for every rejected query
void launch_encode(const float* x, uint64_t nq, uint32_t dim, uint32_t Dp, float* qn,
                   uint4* qcodes, float* tau, int32_t* status, uint32_t* flags, cudaStream_t s);
void launch_codes_to_chunks(const uint64_t* ref_codes, uint64_t rows, uint32_t W, uint4* out,
                            cudaStream_t s);
void launch_chunks_to_codes(const uint4* chunks, uint64_t rows, uint32_t W, uint64_t* out,
                            cudaStream_t s);

struct SearchLaunch {
    DevIndex ix;
    const uint4* qcodes;
    const float* qn;
    const int32_t* qstatus;
    uint64_t nq;
    uint32_t ef, k, entry;
    uint32_t vis_log2, tie_cap;
    uint32_t do_rerank;
    uint32_t* out_ids;
    float* out_scores;
    uint32_t* out_count;
    int32_t* out_status;
    uint32_t* pool_ids;
    uint32_t* pool_dists;
    uint32_t* pool_n;
    uint32_t* qctr;
    unsigned long long* counter;
    uint32_t* flags;        // atomicOr(1 << QVG_Q_TIE_OVERFLOW) on overflow
    const float* qraw;      // non-null: fused encode prologue (raw queries nq x dim);
    float* qn_out;          //   writes normalised queries here, status to out_status
    uint32_t variant;       // A/B switches (QVG_VARIANT env): bit0 no rerank L2 prefetch,
                            // bit1 unused (was: paired-half distance pass)
    uint32_t* exact_bits;   // nullable: per-warp-slot visited bitmaps
    uint64_t exact_words;   // words per slot
    uint32_t depth;         // rerank depth (>= k): the `depth` best scored keys are
                            // reranked; depth == ef is the reference (search.cpp:138)
    const uint32_t* ready;  // nullable: queries [0, *ready) have landed in qraw
                            // (pipelined upload; the warp waits before its prologue)
    uint32_t relax;         // 0: exact search; 2 / 4: relaxed variant, expansions per step
    // re-run of the queries whose shared-memory tie stack overflowed (non-LEAN
    // per-warp kernels only): the tie stack lives in global memory, tie_spill_cap
    // entries per warp slot, and work item i is query qmap[i]
    uint32_t* tie_spill;
    uint32_t tie_spill_cap;
    const uint32_t* qmap;
    // builder searches (non-LEAN kernels): keys (dist<<33 | id) of the first
    // exp_cap expanded nodes of query q at exp_out[q * exp_cap ...], count exp_n[q]
    uint64_t* exp_out;
    uint32_t* exp_n;
    uint32_t exp_cap;
    // Tail balancing (exact per-warp kernels without extra rerank depth; null =
    // off).  The last
    // queries of a batch (index >= susp_from) run in units of susp_budget
    // expansions: at the end of a unit the warp saves the query's search state
    // (pool, compacted rows, query code, tie stack, visited table, scalars) to
    // susp_state and appends the query to a FIFO that warps serve once the fresh
    // queries are gone.  The batch then ends with every warp on a short unit
    // instead of a fifth of them on a whole query; results are unchanged (the
    // state machine resumes where it stopped).
    uint32_t* susp_ctl;     // [0] pushes reserved, [1] pops reserved, [2] budgeted queries completed
    uint32_t* susp_list;    // susp_cap entries, zeroed per launch; entry = query + 1
    uint4* susp_state;      // susp_stride16 uint4 per budgeted query
    uint32_t susp_from, susp_budget, susp_cap, susp_stride16;
};

// Visited-table entry width (bytes) for n nodes and 2^lg slots.  The table
// hashes id by a bijection on b = bits(n - 1) bits (id * odd mod 2^b): the top
// lg bits pick the slot, the low b - lg bits are the tag, so a tag of <= 7 /
// <= 15 bits fits a byte / a short and slot + tag still identify the id
// exactly (no false "visited"); wider tags keep full 32-bit ids.
__host__ __device__ inline uint32_t vis_id_bits(uint64_t n) {
    uint32_t b = 1;
    while (b < 32 && (1ull << b) < n) ++b;
    return b;
}
__host__ __device__ inline uint32_t vis_tag_bytes(uint64_t n, uint32_t lg) {
    const int tb = (int)vis_id_bits(n) - (int)lg;
    return tb <= 7 ? 1u : (tb <= 15 ? 2u : 4u);
}

// keys kept beyond the pool for a rerank deeper than ef (0 = reference depth)
__host__ __device__ inline uint32_t extra_depth(uint32_t ef, uint32_t depth) { return depth > ef ? depth - ef : 0u; }

// grid = min(resident blocks, ceil(nq / warps per block)); exact-visited
// bitmaps are sized for grid * kWarpsPerBlock warp slots.
// default visited-table size (log2 slots): the largest table (256..4096
// slots, >= ef) among those that keep the maximum number of resident blocks
uint32_t auto_visited_log2(const DevIndex& ix, uint32_t ef, uint32_t tie_cap, int device,
                           uint32_t xa = 0, uint32_t relax = 0);
// per-lane row-slot capacity of the relaxed search kernel for max degree R and
// `relax` expansions per step (0 = geometry not supported)
uint32_t relaxed_rw(uint32_t R, uint32_t relax);
// contiguous bytes of the search kernel's per-warp TMA stage (both halves)
uint32_t search_stage_bytes(const DevIndex& ix);

qvg_status plan_search(const SearchLaunch& a, int device, uint64_t* grid,
                       PlanInfo* info = nullptr);
qvg_status launch_search(const SearchLaunch& a, const CUtensorMap* tmap, uint64_t grid,
                         cudaStream_t s);
// latency mode (search_coop.cu): one CTA of warps per query for small batches
uint64_t coop_capacity(const SearchLaunch& a, int device);  // 0 = not applicable
// (grid_out: the CTAs launched; stats report them with warps_per_block = kCoopWarps)
constexpr int kCoopWarps = 8;  // 1 leader + 7 helper warps
qvg_status launch_coop(const SearchLaunch& a, const CUtensorMap* tmap, cudaStream_t s, int device,
                       uint64_t* grid_out = nullptr);
// encode the gather4 descriptor for a code table (false if W > 128)
bool make_code_tmap(CUtensorMap* map, const void* codes, uint64_t n, uint32_t W);
void launch_pair_distance(const DevIndex& ix, const uint4* qchunks, const uint32_t* ids,
                          uint64_t npairs, uint32_t* out, cudaStream_t s);

}  // namespace qvg

// C-ABI entry points for the query path (qvg.h).  Host side of the boundary:
// argument validation with the reference's error classes, host/device buffer
// handling, kernel sequencing on the handle's stream, counters.
//
// qvg_search mirrors qivr::run_query_batch (eval.cpp:225-247) over
// qivr::query (search.cpp:122-143): validate params (search.hpp:16-19), per
// query finite check, normalise, encode, beam search from the entry point,
// rerank to k.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <unistd.h>  // environ
#include <string>
#include <vector>

#include "qvg_internal.cuh"

namespace qvg {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

qvg_status cuda_status(cudaError_t e, const char* what) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    cudaGetLastError();  // clear sticky-free errors
    return e == cudaErrorMemoryAllocation ? QVG_OUT_OF_MEMORY : QVG_CUDA_ERROR;
}

qvg_status grow(Buffer& b, size_t bytes) {
    if (bytes <= b.bytes && b.p) return QVG_OK;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    size_t want = bytes < 256 ? 256 : bytes;
    cudaError_t e = cudaMalloc(&b.p, want);
    if (e != cudaSuccess) return cuda_status(e, "cudaMalloc(scratch)");
    b.bytes = want;
    return QVG_OK;
}

// a tool that serialises kernel launches is injected (Nsight Compute sets
// NV_NSIGHT_INJECTION_* / NV_TPS_LAUNCH_TOKEN; CUDA_INJECTION64_PATH is the
// generic injection hook; sanitizer variables): the pipelined upload must then
// submit its copies before the launch whatever the buffer type
bool under_tool() {
    static const bool v = [] {
        if (getenv("CUDA_INJECTION64_PATH") || getenv("NV_TPS_LAUNCH_TOKEN") ||
            getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE"))
            return true;
        for (char** e = ::environ; e && *e; ++e)
            if (strstr(*e, "SANITIZER") || strstr(*e, "NSIGHT_INJECTION")) return true;
        return false;
    }();
    return v;
}

// page-locked host memory (cudaHostAlloc / cudaHostRegister)
bool is_pinned_host_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

namespace {

const char* qstatus_message(int32_t s) {
    switch (s) {
        case QVG_Q_NONFINITE_COORD: return "query: non-finite coordinate";
        case QVG_Q_BAD_NORM: return "normalize_l2: zero or non-finite norm";
        case QVG_Q_NONFINITE_CODE: return "encode: non-finite coordinate";
        case QVG_Q_TIE_OVERFLOW: return "search: tie stack overflow (raise tie_capacity)";
        default: return "ok";
    }
}

uint32_t log2_floor(uint32_t x) {
    uint32_t l = 0;
    while ((1u << (l + 1)) <= x) ++l;
    return l;
}

// Output buffer: the user's device pointer, or a scratch buffer copied back to
// the user's host pointer at the end.
struct Out {
    void* user = nullptr;
    void* dev = nullptr;
    size_t bytes = 0;
    bool copy_back = false;
};

// `mapped_ok`: a pinned host buffer is written by the kernel itself through
// its device alias (posted PCIe writes as each query finishes) instead of a
// device scratch buffer plus a D2H copy after the launch — only for the small
// per-query results (k ids / scores, count, status)
qvg_status bind_out(Out& o, void* user, Buffer& scratch, size_t bytes, bool needed,
                    bool mapped_ok = false) {
    o.user = user;
    o.bytes = bytes;
    if (!user && !needed) return QVG_OK;
    if (user) {
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, user) != cudaSuccess) {
            cudaGetLastError();
        } else if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
            o.dev = user;
            return QVG_OK;
        } else if (mapped_ok && at.type == cudaMemoryTypeHost && at.devicePointer) {
            o.dev = at.devicePointer;
            return QVG_OK;
        }
    }
    qvg_status st = grow(scratch, bytes);
    if (st != QVG_OK) return st;
    o.dev = scratch.p;
    o.copy_back = user != nullptr;
    return QVG_OK;
}

struct Mode {
    bool encode;   // queries are float vectors (else reference-layout code words)
    bool rerank;
};

// copy stream, its event and `chunks` pinned ready slots for the pipelined upload
qvg_status ensure_copy_stream(qvg_index* h, uint64_t chunks) {
    cudaError_t e;
    if (!h->copy_stream) {
        if ((e = cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_status(e, "cudaStreamCreate(copy)");
        if ((e = cudaEventCreateWithFlags(&h->ev_copy, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_status(e, "cudaEventCreate(copy)");
    }
    if (h->ready_cap < chunks) {
        if (h->ready_host) cudaFreeHost(h->ready_host);
        h->ready_host = nullptr;
        h->ready_cap = 0;
        if ((e = cudaMallocHost(&h->ready_host, chunks * 4)) != cudaSuccess)
            return cuda_status(e, "cudaMallocHost(ready)");
        h->ready_cap = chunks;
    }
    return QVG_OK;
}

qvg_status run(qvg_index* h, const float* queries, const uint64_t* qcodes, uint64_t nq,
               uint32_t k, uint32_t ef, const qvg_search_opts* opts, Mode mode,
               uint32_t* out_ids, float* out_scores, uint32_t* out_count,
               int32_t* out_query_status, uint32_t* out_pool_ids, uint32_t* out_pool_dists,
               uint32_t* out_pool_size, uint32_t* out_qctr, qvg_stats* stats) {
    if (!h) {
        set_error("qvg_search: null index");
        return QVG_INVALID_ARGUMENT;
    }
    if (mode.rerank) {
        if (k < 1) {
            set_error("SearchParams: k must be >= 1");
            return QVG_INVALID_ARGUMENT;
        }
        if (ef < k) {
            set_error("SearchParams: ef must be >= k");
            return QVG_INVALID_ARGUMENT;
        }
    } else if (ef < 1) {
        set_error("beam_search: ef must be >= 1");
        return QVG_INVALID_ARGUMENT;
    }
    if (ef > kMaxEf) {
        set_error("search: ef > " + std::to_string(kMaxEf) + " is not supported");
        return QVG_NOT_IMPLEMENTED;
    }
    if (stats) std::memset(stats, 0, sizeof(*stats));
    if (nq == 0) return QVG_OK;
    if (!queries && !qcodes) {
        set_error("qvg_search: null queries");
        return QVG_INVALID_ARGUMENT;
    }
    if (mode.rerank && (!out_ids || !out_scores || !out_count)) {
        set_error("qvg_search: out_ids, out_scores and out_count are required");
        return QVG_INVALID_ARGUMENT;
    }
    std::lock_guard<std::mutex> lock(h->mu);
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
    const DevIndex& ix = h->ix;
    cudaStream_t s = h->stream;
    const uint32_t entry =
        opts && opts->entry_point != kSentinel ? opts->entry_point : ix.entry;
    if (entry >= ix.n) {
        set_error("beam_search: invalid entry point");
        return QVG_INVALID_ARGUMENT;
    }
    // shared-memory tie stack: 64 entries by default at every ef (a deeper
    // stack costs a resident warp at ef 256: 9.90 -> 9.38 ms); a query that
    // overflows it is re-run with the global-memory stack below
    uint32_t tcap = opts && opts->tie_capacity ? opts->tie_capacity : 64u;
    tcap = (tcap + 3) & ~3u;
    // relaxed variant: 0/1 = exact
    uint32_t relax = opts && opts->relaxed_expansions > 1 ? opts->relaxed_expansions : 0u;
    if (relax) {
        if (relax != 2 && relax != 4) {
            set_error("search: relaxed_expansions must be 0, 1, 2 or 4");
            return QVG_INVALID_ARGUMENT;
        }
        if (!relaxed_rw(ix.R, relax)) {
            set_error("search: relaxed_expansions * ceil(max_degree / 32) must be <= 4");
            return QVG_INVALID_ARGUMENT;
        }
        if (opts->rerank_depth && opts->rerank_depth != ef) {
            set_error("search: relaxed_expansions does not combine with rerank_depth");
            return QVG_INVALID_ARGUMENT;
        }
        tcap = 0;  // no tie stack
    }
    const bool do_rerank = mode.rerank && !(opts && opts->no_rerank);
    // rerank depth (GPU-only knob): 0 = ef, the reference
    const uint32_t depth = opts && opts->rerank_depth ? opts->rerank_depth : ef;
    if (mode.rerank && (depth < k || depth > 2 * ef)) {
        set_error("search: rerank_depth must satisfy k <= rerank_depth <= 2*ef");
        return QVG_INVALID_ARGUMENT;
    }
    const uint32_t xa = do_rerank ? extra_depth(ef, depth) : 0u;
    uint32_t vslots = opts && opts->visited_slots ? opts->visited_slots : 0;
    uint32_t vlog;
    auto cached = h->plans.find(qvg_index::PlanKey{ef, tcap, vslots, xa, relax});
    if (cached != h->plans.end()) {
        vlog = cached->second.first;
    } else if (vslots) {
        const uint32_t floor_slots = 32 * ((ef + xa + 31) / 32);  // rerank scores alias it
        if (vslots < floor_slots) vslots = floor_slots;
        vlog = log2_floor(vslots);
        if ((1u << vlog) < vslots) ++vlog;
        if (vlog < 5) vlog = 5;
    } else {
        // largest table that keeps the most resident warps (occupancy-aware)
        vlog = auto_visited_log2(ix, ef, tcap, h->device, xa, relax);
    }
    const bool exact = opts && opts->exact_visited;
    const bool want_ctr = out_qctr != nullptr || (stats && !(opts && opts->timing_only));

    qvg_status st = QVG_OK;
    // ---- inputs -------------------------------------------------------------
    const size_t in_bytes = mode.encode ? nq * (size_t)ix.dim * 4 : nq * 2ull * ix.W * 8;
    const void* user_in = mode.encode ? (const void*)queries : (const void*)qcodes;
    const bool in_dev = is_device_ptr(user_in);
    if ((st = grow(h->s_qn, nq * (size_t)ix.Dp * 4)) != QVG_OK) return st;
    if ((st = grow(h->s_qc, nq * (size_t)ix.W * 16)) != QVG_OK) return st;
    if ((st = grow(h->s_qst, nq * 4 + 16)) != QVG_OK) return st;  // + flag word
    if ((st = grow(h->s_counter, 64)) != QVG_OK) return st;
    if (!in_dev && (st = grow(h->s_in, in_bytes)) != QVG_OK) return st;
    Out o_ids, o_sc, o_cnt, o_st, o_pi, o_pd, o_pn, o_ctr;
    static const bool zc = [] {  // QVG_ZEROCOPY=0: always stage results in HBM (A/B)
        const char* v = getenv("QVG_ZEROCOPY");
        return !(v && v[0] == '0');
    }();
    if ((st = bind_out(o_ids, out_ids, h->s_ids, nq * k * 4ull, do_rerank, zc)) != QVG_OK) return st;
    if ((st = bind_out(o_sc, out_scores, h->s_sc, nq * k * 4ull, do_rerank, zc)) != QVG_OK) return st;
    if ((st = bind_out(o_cnt, out_count, h->s_cnt, nq * 4ull, do_rerank, zc)) != QVG_OK) return st;
    if ((st = bind_out(o_st, out_query_status, h->s_st, nq * 4ull, true, zc)) != QVG_OK) return st;
    if ((st = bind_out(o_pi, out_pool_ids, h->s_pool_i, nq * ef * 4ull, false)) != QVG_OK) return st;
    if ((st = bind_out(o_pd, out_pool_dists, h->s_pool_d, nq * ef * 4ull, o_pi.dev != nullptr)) != QVG_OK) return st;
    if ((st = bind_out(o_pn, out_pool_size, h->s_pool_n, nq * 4ull, o_pi.dev != nullptr)) != QVG_OK) return st;
    if ((st = bind_out(o_ctr, out_qctr, h->s_qctr, nq * 32ull, want_ctr)) != QVG_OK) return st;

    SearchLaunch a{};
    a.ix = ix;
    a.qcodes = static_cast<const uint4*>(h->s_qc.p);
    a.qn = static_cast<const float*>(h->s_qn.p);
    a.qstatus = static_cast<const int32_t*>(h->s_qst.p);
    a.nq = nq;
    a.ef = ef;
    a.k = k;
    a.entry = entry;
    a.vis_log2 = vlog;
    a.tie_cap = tcap;
    a.relax = relax;
    a.do_rerank = do_rerank;
    a.depth = ef + xa;
    if (do_rerank && depth < ef) a.depth = depth;
    a.out_ids = static_cast<uint32_t*>(o_ids.dev);
    a.out_scores = static_cast<float*>(o_sc.dev);
    a.out_count = static_cast<uint32_t*>(o_cnt.dev);
    a.out_status = static_cast<int32_t*>(o_st.dev);
    a.pool_ids = static_cast<uint32_t*>(o_pi.dev);
    a.pool_dists = static_cast<uint32_t*>(o_pd.dev);
    a.pool_n = static_cast<uint32_t*>(o_pn.dev);
    a.qctr = static_cast<uint32_t*>(o_ctr.dev);
    a.counter = static_cast<unsigned long long*>(h->s_counter.p);
    uint64_t grid = 0;
    {
        static const uint32_t variant = [] {
            const char* v = getenv("QVG_VARIANT");
            return v ? (uint32_t)strtoul(v, nullptr, 0) : 0u;
        }();
        a.variant = variant;
    }
    // launch plan, cached per (ef, tie capacity, visited request): occupancy
    // queries cost host time that would otherwise leave the GPU idle per call
    PlanInfo pinfo;
    {
        const uint32_t vreq = opts && opts->visited_slots ? opts->visited_slots : 0u;
        const qvg_index::PlanKey key{ef, tcap, vreq, xa, relax};
        auto it = h->plans.find(key);
        if (it == h->plans.end()) {
            if ((st = plan_search(a, h->device, &grid, &pinfo)) != QVG_OK) return st;
            pinfo.coop_cap = h->has_tmap ? coop_capacity(a, h->device) : 0;
            it = h->plans.emplace(key, std::make_pair(vlog, pinfo)).first;
        }
        pinfo = it->second.second;
        const uint64_t wpb = pinfo.warps_per_block ? pinfo.warps_per_block : kWarpsPerBlock;
        const uint64_t want = (nq + wpb - 1) / wpb;
        const uint64_t full = (uint64_t)pinfo.resident_warps_per_sm / wpb * pinfo.sms;
        grid = want < full ? want : full;
        if (grid < 1) grid = 1;
    }
    if (exact) {
        const uint64_t words = ((ix.n + 31) / 32 + 3) & ~3ull;
        const uint64_t wpb = pinfo.warps_per_block ? pinfo.warps_per_block : kWarpsPerBlock;
        if ((st = grow(h->s_exact, grid * wpb * words * 4)) != QVG_OK) return st;
        a.exact_bits = static_cast<uint32_t*>(h->s_exact.p);
        a.exact_words = words;
    }

    // ---- tail balancing (headline-geometry kernel; see SearchLaunch) ----------
    {
        static const bool susp_env = [] {  // QVG_SUSPEND=0: whole queries only (A/B)
            const char* v = getenv("QVG_SUSPEND");
            return !(v && v[0] == '0');
        }();
        const uint64_t wpb = pinfo.warps_per_block ? pinfo.warps_per_block : kWarpsPerBlock;
        const uint64_t slots = grid * wpb;
        // (small ef: a query is 50-100 us, a hand-off ~3 us, whole queries win:
        // ef 16 -1.7 % on cfg 2, ef 32 0 % on cfg 2 and -5 % on its clustered variant)
        if (susp_env && pinfo.susp_blob_bytes && !exact && !relax && !xa && h->has_tmap &&
            ef >= 48 && nq > slots && nq < (1ull << 31)) {
            // the last round's queries (one per warp slot) run in units of about a
            // quarter of a query
            const uint64_t nb = nq < slots ? nq : slots;
            const uint32_t stride16 = (64u + pinfo.susp_blob_bytes + 15u) / 16u;
            const uint64_t cap = 8 * nb + 64;
            const size_t head = 64 + ((cap * 4 + 15) & ~size_t(15));
            if ((st = grow(h->s_susp, head + nb * stride16 * 16ull)) != QVG_OK) return st;
            char* p = static_cast<char*>(h->s_susp.p);
            a.susp_ctl = reinterpret_cast<uint32_t*>(p);
            a.susp_list = reinterpret_cast<uint32_t*>(p + 64);
            a.susp_state = reinterpret_cast<uint4*>(p + head);
            a.susp_from = (uint32_t)(nq - nb);
            // (cfg 2, ef 64, kernel ms: off 2.080; window of 0.5 / 1 / 1.5 / 2 / 3 / 4
            // rounds at this budget 2.027 / 1.971 / 1.972 / 1.988 / 1.992 / 2.011;
            // budgets of 12 / 16 / 21 / 30 / 40 / 55 expansions at 1 round
            // - / - / 1.971 / 1.985 / 1.987 / 2.022: profiles/r3_susp_tune*.txt)
            a.susp_budget = (3u * ef + 9u) / 10u + 2u;
            if (a.susp_budget < 12u) a.susp_budget = 12u;
            a.susp_cap = (uint32_t)cap;
            a.susp_stride16 = stride16;
            cudaMemsetAsync(p, 0, head, s);
        }
    }

    // ---- pipeline -------------------------------------------------------------
    uint32_t* d_flags = reinterpret_cast<uint32_t*>(static_cast<char*>(h->s_counter.p) + 32);
    uint32_t* d_ready = reinterpret_cast<uint32_t*>(static_cast<char*>(h->s_counter.p) + 48);
    a.flags = d_flags;
    // opt-in: the lane-0 FP64 chains stall the search warp; measured 3.10 ms
    // fused vs 3.02 ms with the separate encode kernel (cfg2, 10k queries)
    static const bool fused_env = [] {
        const char* v = getenv("QVG_FUSED");
        return v && v[0] == '1';
    }();
    // Host queries: pipelined upload (QVG_PIPELINE=0 disables).  One search
    // launch with the fused encode prologue starts first; a copy stream lands
    // the queries chunk by chunk and publishes how many have landed; each
    // warp waits for its query's chunk.  The upload hides under the search
    // (no per-chunk launch tails), also for pageable buffers, since the
    // kernel is already running while the driver stages them.
    static const bool pipe_env = [] {
        const char* v = getenv("QVG_PIPELINE");
        return !(v && v[0] == '0');
    }();
    static const uint64_t kChunk = [] {  // queries per pipelined upload chunk
        const char* v = getenv("QVG_CHUNK");
        const long long c = v ? atoll(v) : 1024;
        return (uint64_t)(c < 32 ? 32 : c);
    }();
    bool launched = false;
    const bool stage_ok = 4ull * ix.dim <= search_stage_bytes(ix);
    const bool pipelined = mode.encode && !in_dev && pipe_env && stage_ok && nq >= 2 * kChunk;
    cudaEventRecord(h->ev[0], s);
    const void* din = user_in;
    if (!in_dev && !pipelined) {
        e = cudaMemcpyAsync(h->s_in.p, user_in, in_bytes, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_status(e, "H2D(queries)");
    }
    if (!in_dev) din = h->s_in.p;
    cudaMemsetAsync(h->s_counter.p, 0, 64, s);  // work counter + flag word + ready count
    cudaEventRecord(h->ev[1], s);
    const bool fused = mode.encode && stage_ok && (fused_env || pipelined);
    if (pipelined && (st = ensure_copy_stream(h, (nq + kChunk - 1) / kChunk + 5)) != QVG_OK) return st;
    if (fused) {
        // K1 runs as the search kernel's per-query prologue
        a.qraw = static_cast<const float*>(din);
        a.qn_out = static_cast<float*>(h->s_qn.p);
        a.qstatus = nullptr;
        if (pipelined) a.ready = d_ready;
    } else if (mode.encode) {
        launch_encode(static_cast<const float*>(din), nq, ix.dim, ix.Dp,
                      static_cast<float*>(h->s_qn.p), static_cast<uint4*>(h->s_qc.p), nullptr,
                      static_cast<int32_t*>(h->s_qst.p), d_flags, s);
    } else {
        launch_codes_to_chunks(static_cast<const uint64_t*>(din), nq, ix.W,
                               static_cast<uint4*>(h->s_qc.p), s);
        cudaMemsetAsync(h->s_qst.p, 0, nq * 4, s);
    }
    cudaEventRecord(h->ev[2], s);
    // small batches: one CTA per query (latency mode, search_coop.cu) when the
    // whole batch fits in one wave of its CTAs (measured: cfg2 batch 1 0.48 ->
    // 0.39 ms, batch 1024 0.69 -> 0.57 ms; beyond one wave the per-warp kernel
    // wins, e.g. batch 2048 0.83 vs 1.03 ms).  QVG_COOP_MAX_NQ overrides the
    // cut-off (0 disables).
    static const int64_t coop_env = [] {
        const char* v = getenv("QVG_COOP_MAX_NQ");
        return v ? (int64_t)strtoll(v, nullptr, 0) : -1ll;
    }();
    bool coop = coop_env != 0 && pinfo.coop_cap > 0 && !a.exact_bits && !a.qraw && !a.ready &&
                !a.tie_spill && !a.qmap &&
                !(a.do_rerank && a.depth != a.ef) && !a.relax;
    if (coop) coop = coop_env > 0 ? nq <= (uint64_t)coop_env : nq <= pinfo.coop_cap;
    // Chunk copies of a PINNED buffer are submitted BEFORE the search launch
    // (pure DMA, submission is cheap): the copy engine still overlaps them with
    // the running kernel, and a tool that serialises launches (ncu kernel
    // replay, compute-sanitizer) drains them before the kernel starts instead
    // of deadlocking it.  A PAGEABLE buffer is staged by the host thread inside
    // each cudaMemcpyAsync, so its chunks are submitted after the launch (the
    // kernel runs while the driver stages them); under such tools use
    // QVG_PIPELINE=0 for pageable host queries.
    // (launching before the copies are queued — only a first chunk of 128 to
    // 1024 queries submitted ahead of the kernel, ramped or not, polling every
    // 256 ns or 2 us — measured 0.4-1.7 % slower end to end than every chunk
    // submitted first: profiles/r2k_e2e_ab.txt, r2w_early_ab.txt)
    const bool copies_first = pipelined && (is_pinned_host_ptr(user_in) || under_tool());
    uint64_t next_c0 = 0, next_c = 0;
    bool chunks_started = false;
    auto submit_chunks = [&](uint64_t max_chunks) -> qvg_status {
        // Each chunk's ready count is a 4-byte copy ordered after its rows on
        // the copy stream; the chunks start after the counter reset (ev[1]).
        cudaStream_t cs = h->copy_stream;
        if (!chunks_started) cudaStreamWaitEvent(cs, h->ev[1], 0);
        chunks_started = true;
        const size_t row = (size_t)ix.dim * 4;
        for (uint64_t done = 0; next_c0 < nq && done < max_chunks; ++done, ++next_c) {
            const uint64_t c0 = next_c0;
            const uint64_t len = kChunk;
            const uint64_t c1 = c0 + len < nq ? c0 + len : nq;
            next_c0 = c1;
            e = cudaMemcpyAsync(static_cast<char*>(h->s_in.p) + c0 * row,
                                static_cast<const char*>(user_in) + c0 * row, (c1 - c0) * row,
                                cudaMemcpyHostToDevice, cs);
            if (e == cudaSuccess) {
                h->ready_host[next_c] = (uint32_t)c1;
                e = cudaMemcpyAsync(d_ready, &h->ready_host[next_c], 4, cudaMemcpyHostToDevice, cs);
            }
            if (e != cudaSuccess) {
                // never leave a running kernel waiting: release every query
                // (a copy-engine write; no SM is free while the search runs)
                if (launched) {
                    h->ready_host[next_c + 1] = (uint32_t)nq;
                    cudaMemcpyAsync(d_ready, &h->ready_host[next_c + 1], 4, cudaMemcpyHostToDevice, cs);
                }
                cudaStreamSynchronize(cs);
                if (launched) cudaStreamSynchronize(s);
                return cuda_status(e, "H2D(queries, pipelined)");
            }
        }
        if (next_c0 >= nq) cudaEventRecord(h->ev_copy, cs);
        return QVG_OK;
    };
    const uint64_t kAll = ~0ull;
    if (copies_first && (st = submit_chunks(kAll)) != QVG_OK) return st;
    if (coop) {
        st = launch_coop(a, &h->tmap, s, h->device, &grid);
        pinfo.warps_per_block = kCoopWarps;  // reported in stats: the latency kernel ran
    } else {
        st = launch_search(a, h->has_tmap ? &h->tmap : nullptr, grid, s);
    }
    if (st != QVG_OK) {
        if (chunks_started) cudaStreamSynchronize(h->copy_stream);  // no copy outlives the call
        return st;
    }
    launched = true;
    if (pipelined && !copies_first && (st = submit_chunks(kAll)) != QVG_OK) return st;
    if (pipelined) cudaStreamWaitEvent(s, h->ev_copy, 0);  // results after every chunk
    cudaEventRecord(h->ev[3], s);
    Out* outs[] = {&o_ids, &o_sc, &o_cnt, &o_st, &o_pi, &o_pd, &o_pn, &o_ctr};
    for (Out* o : outs) {
        if (o->copy_back) {
            e = cudaMemcpyAsync(o->user, o->dev, o->bytes, cudaMemcpyDeviceToHost, s);
            if (e != cudaSuccess) return cuda_status(e, "D2H(results)");
        }
    }
    // 4-byte summary of all per-query statuses
    // the 4-byte status summary lands in a pinned word of the handle: a copy
    // into pageable memory would stage through the driver and stall the call
    if (!h->host_flags) {
        e = cudaMallocHost(&h->host_flags, 16);
        if (e != cudaSuccess) return cuda_status(e, "cudaMallocHost(flags)");
    }
    h->host_flags[0] = 0;
    e = cudaMemcpyAsync(h->host_flags, d_flags, 4, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_status(e, "D2H(flags)");
    const bool counters = out_qctr != nullptr || (stats && !(opts && opts->timing_only));
    std::vector<uint32_t> ctr_host;
    if (stats && counters && !o_ctr.copy_back) {
        ctr_host.resize(nq * 8);
        e = cudaMemcpyAsync(ctr_host.data(), o_ctr.dev, nq * 32, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return cuda_status(e, "D2H(counters)");
    }
    cudaEventRecord(h->ev[4], s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, "search");
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_status(e, "search");
    uint32_t hflags = h->host_flags[0];

    // Queries whose shared-memory tie stack overflowed are re-run at once with
    // the stack in global memory (capacity n: a node enters it at most once),
    // so no valid query ever fails where the reference's unbounded frontier
    // (search.cpp:38-68) answers it.  Rare path: results of the other queries
    // are untouched, the copies back are simply redone.
    uint64_t n_spilled = 0;
    if (hflags & (1u << QVG_Q_TIE_OVERFLOW)) {
        std::vector<int32_t> qs(nq);
        e = cudaMemcpy(qs.data(), o_st.dev, nq * 4, cudaMemcpyDefault);  // (HBM or mapped host)
        if (e != cudaSuccess) return cuda_status(e, "D2H(status)");
        std::vector<uint32_t> redo;
        for (uint64_t i = 0; i < nq; ++i)
            if (qs[i] == QVG_Q_TIE_OVERFLOW) redo.push_back((uint32_t)i);
        n_spilled = redo.size();
        if (!redo.empty()) {
            if (fused) {
                // the fused prologue kept the query codes in shared memory:
                // encode the (device-resident) raw rows for the re-run
                launch_encode(static_cast<const float*>(din), nq, ix.dim, ix.Dp,
                              static_cast<float*>(h->s_qn.p), static_cast<uint4*>(h->s_qc.p),
                              nullptr, static_cast<int32_t*>(h->s_qst.p), nullptr, s);
            }
            SearchLaunch r = a;
            r.susp_ctl = nullptr;
            r.qraw = nullptr;
            r.qn_out = nullptr;
            r.ready = nullptr;
            r.qcodes = static_cast<const uint4*>(h->s_qc.p);
            r.qn = static_cast<const float*>(h->s_qn.p);
            r.qstatus = static_cast<const int32_t*>(h->s_qst.p);
            r.nq = redo.size();
            r.tie_cap = 4;  // shared-memory stack unused (layout minimum)
            r.tie_spill_cap = (uint32_t)(ix.n < 0xFFFFFFF0ull ? ix.n : 0xFFFFFFF0ull);
            uint64_t rgrid = 0;
            PlanInfo rinfo;
            if ((st = plan_search(r, h->device, &rgrid, &rinfo)) != QVG_OK) return st;
            const uint64_t wpb = rinfo.warps_per_block ? rinfo.warps_per_block : kWarpsPerBlock;
            // at most 64 Mi stack entries (256 MB) in flight
            uint64_t slots = (64ull << 20) / r.tie_spill_cap;
            if (slots < wpb) slots = wpb;
            if (rgrid > slots / wpb) rgrid = slots / wpb;
            if (rgrid < 1) rgrid = 1;
            void* spill = nullptr;
            void* qmap = nullptr;
            e = cudaMalloc(&spill, rgrid * wpb * r.tie_spill_cap * 4ull);
            if (e == cudaSuccess) e = cudaMalloc(&qmap, redo.size() * 4);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(qmap, redo.data(), redo.size() * 4, cudaMemcpyHostToDevice, s);
            if (e == cudaSuccess && r.exact_bits) {
                st = grow(h->s_exact, rgrid * wpb * r.exact_words * 4);
                r.exact_bits = static_cast<uint32_t*>(h->s_exact.p);
            }
            if (e == cudaSuccess && st == QVG_OK) {
                r.tie_spill = static_cast<uint32_t*>(spill);
                r.qmap = static_cast<const uint32_t*>(qmap);
                cudaMemsetAsync(h->s_counter.p, 0, 48, s);  // work counter + flag word
                st = launch_search(r, h->has_tmap ? &h->tmap : nullptr, rgrid, s);
                for (Out* o : outs)
                    if (st == QVG_OK && o->copy_back) {
                        e = cudaMemcpyAsync(o->user, o->dev, o->bytes, cudaMemcpyDeviceToHost, s);
                        if (e != cudaSuccess) break;
                    }
                h->host_flags[1] = 0;
                if (e == cudaSuccess && st == QVG_OK)
                    e = cudaMemcpyAsync(h->host_flags + 1, d_flags, 4, cudaMemcpyDeviceToHost, s);
                if (e == cudaSuccess && st == QVG_OK && stats && counters && !o_ctr.copy_back)
                    e = cudaMemcpyAsync(ctr_host.data(), o_ctr.dev, nq * 32, cudaMemcpyDeviceToHost, s);
                if (e == cudaSuccess && st == QVG_OK) e = cudaStreamSynchronize(s);
                hflags = (hflags & ~(1u << QVG_Q_TIE_OVERFLOW)) | h->host_flags[1];
            }
            cudaFree(spill);
            cudaFree(qmap);
            if (st != QVG_OK) return st;
            if (e != cudaSuccess) return cuda_status(e, "search (tie-stack re-run)");
        }
    }

    if (stats) {
        float t = 0;
        cudaEventElapsedTime(&t, h->ev[1], h->ev[2]);
        stats->encode_ms = t;
        cudaEventElapsedTime(&t, h->ev[2], h->ev[3]);
        stats->search_ms = t;
        cudaEventElapsedTime(&t, h->ev[1], h->ev[3]);
        stats->device_ms = t;
        cudaEventElapsedTime(&t, h->ev[0], h->ev[4]);
        stats->total_ms = t;
        stats->grid_blocks = (uint32_t)grid;
        stats->warps_per_block = pinfo.warps_per_block;
        stats->smem_per_block = pinfo.smem_per_block;
        stats->resident_warps_per_sm = pinfo.resident_warps_per_sm;
        stats->queries = nq;
        if (counters) {
            const uint32_t* c = o_ctr.copy_back ? out_qctr : ctr_host.data();
            for (uint64_t i = 0; i < nq; ++i) {
                const uint32_t* r = c + i * 8;
                if (r[7] == QVG_Q_NONFINITE_COORD || r[7] == QVG_Q_BAD_NORM ||
                    r[7] == QVG_Q_NONFINITE_CODE)
                    continue;
                stats->expansions += r[0];
                stats->tie_expansions += r[1];
                stats->dist_evals += r[2];
                stats->inpool_drops += r[3];
                stats->adjacency_slots += r[4];
                stats->cold_accesses += do_rerank ? r[5] : 0;

                if (r[6] > stats->max_tie_depth) stats->max_tie_depth = r[6];
                stats->adjacency_bytes += 4ull * r[0] + 4ull * r[4];
            }
            stats->code_bytes = stats->dist_evals * 16ull * ix.W;
            stats->rerank_bytes = stats->cold_accesses * 4ull * ix.dim;
            stats->io_bytes = nq * (4ull * ix.dim + (do_rerank ? 8ull * k : 0));
        }
        stats->tie_overflows = n_spilled;  // re-run with a global-memory tie stack
    }
    if (hflags == 0) return QVG_OK;
    if (hflags & (1u << 30)) {
        set_error("search: internal error (a suspended query was never handed over)");
        return QVG_RUNTIME_ERROR;
    }
    // rare path: locate the first offending query (the reference's
    // single-threaded batch throws at the first invalid one)
    std::vector<int32_t> qs(nq);
    e = cudaMemcpy(qs.data(), o_st.dev, nq * 4, cudaMemcpyDefault);
    if (e != cudaSuccess) return cuda_status(e, "D2H(status)");
    int64_t first_bad = -1, first_ovf = -1;
    for (uint64_t i = 0; i < nq; ++i) {
        const int32_t v = qs[i];
        if (v == QVG_Q_TIE_OVERFLOW) {
            if (first_ovf < 0) first_ovf = (int64_t)i;
        } else if (v != 0 && first_bad < 0) {
            first_bad = (int64_t)i;
        }
    }
    if (first_bad >= 0) {
        set_error(std::string(qstatus_message(qs[first_bad])) + " (query " +
                  std::to_string(first_bad) + ")");
        return QVG_INVALID_ARGUMENT;
    }
    if (first_ovf >= 0) {
        set_error(std::string(qstatus_message(QVG_Q_TIE_OVERFLOW)) + " (query " +
                  std::to_string(first_ovf) + ")");
        return QVG_CAPACITY_OVERFLOW;
    }
    return QVG_OK;
}

}  // namespace
}  // namespace qvg

using namespace qvg;

extern "C" {

const char* qvg_last_error(void) { return g_last_error.c_str(); }

int qvg_abi_version(void) { return QVG_ABI_VERSION; }

qvg_status qvg_search(qvg_index* index, const float* queries, uint64_t nq, uint32_t k,
                      uint32_t ef, uint32_t* out_ids, float* out_scores, uint32_t* out_count,
                      int32_t* out_query_status, qvg_stats* stats) {
    return run(index, queries, nullptr, nq, k, ef, nullptr, Mode{true, true}, out_ids,
               out_scores, out_count, out_query_status, nullptr, nullptr, nullptr, nullptr,
               stats);
}

qvg_status qvg_search_ex(qvg_index* index, const float* queries, uint64_t nq, uint32_t k,
                         uint32_t ef, const qvg_search_opts* opts, uint32_t* out_ids,
                         float* out_scores, uint32_t* out_count, int32_t* out_query_status,
                         uint32_t* out_pool_ids, uint32_t* out_pool_dists,
                         uint32_t* out_pool_size, uint32_t* out_query_counters,
                         qvg_stats* stats) {
    const bool rr = !(opts && opts->no_rerank);
    return run(index, queries, nullptr, nq, k, ef, opts, Mode{true, rr}, out_ids, out_scores,
               out_count, out_query_status, out_pool_ids, out_pool_dists, out_pool_size,
               out_query_counters, stats);
}

qvg_status qvg_beam_search(qvg_index* index, const uint64_t* query_codes, uint64_t nq,
                           uint32_t ef, uint32_t entry_point, uint32_t* out_pool_ids,
                           uint32_t* out_pool_dists, uint32_t* out_pool_size,
                           qvg_stats* stats) {
    qvg_search_opts o{};
    o.entry_point = entry_point;
    o.no_rerank = 1;
    if (!out_pool_ids || !out_pool_dists || !out_pool_size) {
        set_error("qvg_beam_search: pool outputs are required");
        return QVG_INVALID_ARGUMENT;
    }
    return run(index, nullptr, query_codes, nq, 1, ef, &o, Mode{false, false}, nullptr,
               nullptr, nullptr, nullptr, out_pool_ids, out_pool_dists, out_pool_size, nullptr,
               stats);
}

qvg_status qvg_encode(int device, const float* x, uint64_t nq, uint32_t dim,
                      float* out_normalized, uint64_t* out_codes, float* out_tau,
                      int32_t* out_query_status) {
    if (dim == 0) {
        set_error("compute_threshold: empty vector");
        return QVG_INVALID_ARGUMENT;
    }
    if (nq == 0) return QVG_OK;
    if (!x || !out_normalized || !out_codes || !out_query_status) {
        set_error("qvg_encode: null argument");
        return QVG_INVALID_ARGUMENT;
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
    const uint32_t W = (dim + 63) / 64, Dp = (dim + 3) & ~3u;
    void *d_x = nullptr, *d_qn = nullptr, *d_qc = nullptr, *d_codes = nullptr, *d_tau = nullptr,
         *d_st = nullptr;
    e = cudaMalloc(&d_x, nq * dim * 4ull);
    if (e == cudaSuccess) e = cudaMalloc(&d_qn, nq * Dp * 4ull);
    if (e == cudaSuccess) e = cudaMalloc(&d_qc, nq * W * 16ull);
    if (e == cudaSuccess) e = cudaMalloc(&d_codes, nq * W * 16ull);
    if (e == cudaSuccess) e = cudaMalloc(&d_tau, nq * 4ull);
    if (e == cudaSuccess) e = cudaMalloc(&d_st, nq * 4ull);
    if (e == cudaSuccess) e = cudaMemcpy(d_x, x, nq * dim * 4ull, cudaMemcpyDefault);
    if (e == cudaSuccess) {
        launch_encode(static_cast<const float*>(d_x), nq, dim, Dp, static_cast<float*>(d_qn),
                      static_cast<uint4*>(d_qc), static_cast<float*>(d_tau),
                      static_cast<int32_t*>(d_st), nullptr, 0);
        launch_chunks_to_codes(static_cast<const uint4*>(d_qc), nq, W,
                               static_cast<uint64_t*>(d_codes), 0);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess)
        e = cudaMemcpy2D(out_normalized, dim * 4ull, d_qn, Dp * 4ull, dim * 4ull, nq,
                         cudaMemcpyDefault);
    if (e == cudaSuccess) e = cudaMemcpy(out_codes, d_codes, nq * W * 16ull, cudaMemcpyDefault);
    if (e == cudaSuccess && out_tau) e = cudaMemcpy(out_tau, d_tau, nq * 4ull, cudaMemcpyDefault);
    if (e == cudaSuccess)
        e = cudaMemcpy(out_query_status, d_st, nq * 4ull, cudaMemcpyDefault);
    cudaFree(d_x);
    cudaFree(d_qn);
    cudaFree(d_qc);
    cudaFree(d_codes);
    cudaFree(d_tau);
    cudaFree(d_st);
    if (e != cudaSuccess) return cuda_status(e, "qvg_encode");
    std::vector<int32_t> sts(nq);
    if (is_device_ptr(out_query_status))
        cudaMemcpy(sts.data(), out_query_status, nq * 4, cudaMemcpyDeviceToHost);
    else
        std::memcpy(sts.data(), out_query_status, nq * 4);
    for (uint64_t i = 0; i < nq; ++i)
        if (sts[i] != 0) {
            set_error(std::string(qstatus_message(sts[i])) + " (row " + std::to_string(i) + ")");
            return QVG_INVALID_ARGUMENT;
        }
    return QVG_OK;
}

qvg_status qvg_sm2_distance(qvg_index* h, const uint64_t* query_codes, const uint32_t* ids,
                            uint64_t npairs, uint32_t* out) {
    if (!h || !query_codes || !ids || !out) {
        set_error("qvg_sm2_distance: null argument");
        return QVG_INVALID_ARGUMENT;
    }
    if (npairs == 0) return QVG_OK;
    std::lock_guard<std::mutex> lock(h->mu);
    cudaSetDevice(h->device);
    const DevIndex& ix = h->ix;
    std::vector<uint32_t> hid(npairs);
    cudaError_t e = cudaMemcpy(hid.data(), ids, npairs * 4, cudaMemcpyDefault);
    if (e != cudaSuccess) return cuda_status(e, "qvg_sm2_distance");
    for (uint64_t i = 0; i < npairs; ++i)
        if (hid[i] >= ix.n) {
            set_error("sm2_distance: node id out of range");
            return QVG_INVALID_ARGUMENT;
        }
    qvg_status st;
    if ((st = grow(h->s_in, npairs * 2ull * ix.W * 8)) != QVG_OK) return st;
    if ((st = grow(h->s_qc, npairs * (size_t)ix.W * 16)) != QVG_OK) return st;
    if ((st = grow(h->s_pair_ids, npairs * 4)) != QVG_OK) return st;
    if ((st = grow(h->s_pair_out, npairs * 4)) != QVG_OK) return st;
    cudaStream_t s = h->stream;
    e = cudaMemcpyAsync(h->s_in.p, query_codes, npairs * 2ull * ix.W * 8, cudaMemcpyDefault, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(h->s_pair_ids.p, hid.data(), npairs * 4, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "qvg_sm2_distance");
    launch_codes_to_chunks(static_cast<const uint64_t*>(h->s_in.p), npairs, ix.W,
                           static_cast<uint4*>(h->s_qc.p), s);
    launch_pair_distance(ix, static_cast<const uint4*>(h->s_qc.p),
                         static_cast<const uint32_t*>(h->s_pair_ids.p), npairs,
                         static_cast<uint32_t*>(h->s_pair_out.p), s);
    e = cudaMemcpyAsync(out, h->s_pair_out.p, npairs * 4, cudaMemcpyDefault, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return e == cudaSuccess ? QVG_OK : cuda_status(e, "qvg_sm2_distance");
}

}  // extern "C"

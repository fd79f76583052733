/*
 * qvg.h — C-ABI of the B200-native BQ query path (drop-in for QuIVer `qivr`).
 *
 * One handle = one HBM-resident index on one device + one CUDA stream.  A handle
 * must not be used by two host threads at once; separate handles are
 * independent.  All buffers are caller-owned; no exception crosses this ABI.
 * Pointers named `queries` / `out_*` may be host (pageable or pinned) or device
 * pointers — the library detects which with cudaPointerGetAttributes.
 *
 * Reference interfaces each entry point replaces (paths under
 * /root/reference/proj/core):
 *   qvg_index_create      qivr::Index built by build_index (builder.cpp:137-155)
 *                         or load_index (store_io.cpp:128-169): consumes the
 *                         public raw() layouts SignatureStore::raw
 *                         (encoding.hpp:247-248), AdjacencyTable::raw
 *                         (graph.hpp:135-136), ColdStore::raw (cold_store.hpp:58)
 *   qvg_index_load        qivr::load_index(path, ColdMode) (store_io.hpp:40,
 *                         store_io.cpp:128-169) — .qivr v1 straight into HBM
 *   qvg_index_save        qivr::save_index (store_io.cpp:99-126)
 *   qvg_search            qivr::run_query_batch(index, queries, nq,
 *                         SearchParams{ef,k}, threads) (eval.hpp:42-44,
 *                         eval.cpp:225-247) == per-query qivr::query
 *                         (search.hpp:95-98, search.cpp:122-143)
 *   qvg_search_ex         same, plus the beam-search pool (beam_search_words,
 *                         search.cpp:27-81) and per-query counters
 *   qvg_beam_search       qivr::beam_search / beam_search_words on given code
 *                         words from a given entry (search.hpp:79-86,
 *                         search.cpp:83-94)
 *   qvg_encode            qivr::normalize_l2 + encode_sm2_into
 *                         (vec_math.hpp:37-44, encoding.cpp:23-45)
 *   qvg_sm2_distance      SignatureStore::distance_to / sm2_distance_words
 *                         (encoding.hpp:110-178, 243-245)
 *   qvg_build             qivr::build_index (builder.cpp:137-155) — GPU batched
 *                         BQ-space Vamana insertion with RobustPrune
 *                         (graph.hpp:162-227)
 *   qvg_brute_force_topk  qivr::brute_force_topk (eval.hpp:19-21,
 *                         eval.cpp:81-168) — exact ground truth on the GPU
 *   qvg_compatibility_probe  qivr::compatibility_probe (eval.cpp:196-222)
 *   qvg_strong_bit_rate   qivr::strong_bit_rate (encoding.cpp:132-167)
 *
 * Error mapping: QVG_INVALID_ARGUMENT <-> std::invalid_argument
 * (SearchParams::validate search.hpp:16-19; dim mismatch search.cpp:125-127;
 * non-finite coordinate search.cpp:129-131; zero/non-finite norm
 * vec_math.hpp:39-41); QVG_RUNTIME_ERROR <-> std::runtime_error (store_io.cpp
 * format / I/O errors).  qvg_last_error() returns a thread-local message.
 */
#ifndef QVG_H_
#define QVG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QVG_ABI_VERSION 1

typedef struct qvg_index qvg_index;

typedef enum qvg_status {
    QVG_OK = 0,
    QVG_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    QVG_CUDA_ERROR = 2,
    QVG_OUT_OF_MEMORY = 3,
    QVG_CAPACITY_OVERFLOW = 4, /* reserved: never returned by search (a query whose
                                  shared-memory tie stack fills is re-run with the
                                  stack in global memory, capacity n) */
    QVG_NOT_IMPLEMENTED = 5,
    QVG_RUNTIME_ERROR = 6 /* std::runtime_error in the reference (I/O, format) */
} qvg_status;

/* Per-query status codes written to out_query_status (0 = ok). */
#define QVG_Q_OK 0
#define QVG_Q_NONFINITE_COORD 1 /* "query: non-finite coordinate"        */
#define QVG_Q_BAD_NORM 2        /* "normalize_l2: zero or non-finite norm" */
#define QVG_Q_NONFINITE_CODE 3  /* "encode: non-finite coordinate"        */
#define QVG_Q_TIE_OVERFLOW 4    /* internal: shared-memory tie stack full; the query
                                   is re-run before the call returns, so callers
                                   never see this status */

/* Counters summed over a batch.  "Algorithmic" bytes follow SURVEY §8(d):
 * B_q = sum_exp(4 + 4*deg) + evals*16W + |pool|*4D + 4D + 8k. */
typedef struct qvg_stats {
    uint64_t queries;
    uint64_t expansions;
    uint64_t tie_expansions;   /* expansions of nodes evicted from the pool */
    uint64_t dist_evals;       /* code rows scored (incl. entry) */
    uint64_t inpool_drops;     /* re-scored keys found in the pool (visited-cache misses) */
    uint64_t adjacency_slots;  /* sum of degrees of expanded nodes */
    uint64_t cold_accesses;    /* sum of pool sizes == rerank rows (ColdStore::vec calls) */
    uint64_t tie_overflows;    /* queries whose shared-memory tie stack filled and
                                  were re-run with a global-memory stack */
    uint64_t max_tie_depth;
    uint64_t adjacency_bytes;  /* sum_exp (4 + 4*deg), reference slot layout */
    uint64_t code_bytes;       /* dist_evals * 16W */
    uint64_t rerank_bytes;     /* cold_accesses * 4D */
    uint64_t io_bytes;         /* nq * (4D + 8k) */
    double encode_ms;          /* device time of the encode kernel */
    double search_ms;          /* device time of the fused search+rerank kernel */
    double device_ms;          /* encode + search (device, excl. copies) */
    double total_ms;           /* incl. host<->device copies when host buffers */
    uint32_t grid_blocks;      /* persistent grid of the search kernel */
    uint32_t warps_per_block;
    uint32_t smem_per_block;   /* dynamic shared memory bytes */
    uint32_t resident_warps_per_sm;
} qvg_stats;

/* Search options for qvg_search_ex. */
typedef struct qvg_search_opts {
    uint32_t visited_slots; /* per-query lossy visited table (power of 2; 0 = default) */
    uint32_t tie_capacity;  /* shared-memory tie stack entries per query (0 = default);
                             overflow spills to a global-memory re-run          */
    uint32_t exact_visited; /* 1: exact global visited bitmap (stats / validation)   */
    uint32_t entry_point;   /* UINT32_MAX: the index's entry point                   */
    uint32_t no_rerank;     /* 1: skip rerank (pool only)                            */
    uint32_t timing_only;   /* 1: stats carries device timings only (no counter D2H)  */
    uint32_t rerank_depth;  /* 0 = ef (the reference).  Otherwise k <= depth <= 2*ef:
                             * rerank the `depth` best (dist, id) keys among all
                             * scored nodes.  GPU-only knob (BASELINE config 4), no
                             * reference counterpart; depth <= ef reranks a pool
                             * prefix. */
    uint32_t relaxed_expansions; /* 0 or 1: exact search (the reference).  2 or 4: the
                             * RELAXED variant — expand that many best unexpanded pool
                             * entries per step, merge-then-truncate admission, no
                             * tie stack; NOT result-identical to the reference
                             * (reported separately).  Needs relaxed * ceil(R/32) <= 4
                             * and rerank_depth == 0. */
} qvg_search_opts;

const char* qvg_last_error(void);
int qvg_abi_version(void);

/* Create an HBM-resident index from the reference's raw layouts:
 *   codes : n x 2*ceil(dim/64) u64, per node W pos words then W strong words
 *   adj   : n x (max_degree+1) u32, [degree, id_0 .. id_{R-1}], unused = 0
 *   cold  : n x dim f32, unit-normalised rows
 * Host buffers may be freed after return.  Validates degree <= max_degree,
 * ids < n and entry < n (QVG_INVALID_ARGUMENT otherwise). */
qvg_status qvg_index_create(const uint64_t* codes, uint64_t n, uint32_t dim,
                            const uint32_t* adj_slots, uint32_t max_degree, const float* cold,
                            uint32_t entry_point, int device, qvg_index** out);

/* Load a .qivr v1 file (store_io.hpp:17-30 layout) straight into HBM.
 * Fail-closed like load_index: bad magic / version / offsets / truncation ->
 * QVG_RUNTIME_ERROR, never a partial index. */
qvg_status qvg_index_load(const char* path, int device, qvg_index** out);

/* Write the index as a .qivr v1 file readable by qivr::load_index. */
qvg_status qvg_index_save(const qvg_index* index, const char* path);

void qvg_index_destroy(qvg_index* index);

qvg_status qvg_index_info(const qvg_index* index, uint64_t* n, uint32_t* dim,
                          uint32_t* max_degree, uint32_t* entry_point);

/* Use a caller-owned CUDA stream (cudaStream_t as void*; NULL restores the
 * handle's own stream).  All later work on the handle is issued on it. */
qvg_status qvg_index_set_stream(qvg_index* index, void* stream);

/* Copy the index's stores back out in the reference layouts (host buffers of
 * the sizes given to qvg_index_create; any may be NULL). */
qvg_status qvg_index_export(const qvg_index* index, uint64_t* codes, uint32_t* adj_slots,
                            float* cold);

/* Batched query: normalise, encode, exact BQ beam search, float32 rerank.
 * queries: nq x dim f32.  out_ids/out_scores: nq x k (rows past out_count[i]
 * are padded with UINT32_MAX / NaN).  out_count: nq (min(k, |pool|)).
 * out_query_status: nq (nullable).  stats: nullable.
 * Returns QVG_INVALID_ARGUMENT if params are invalid (k < 1, ef < k) or any
 * query is invalid (per-query codes tell which; valid queries are answered). */
qvg_status qvg_search(qvg_index* index, const float* queries, uint64_t nq, uint32_t k,
                      uint32_t ef, uint32_t* out_ids, float* out_scores, uint32_t* out_count,
                      int32_t* out_query_status, qvg_stats* stats);

/* qvg_search plus options, the pool (nq x ef ids / dists, ascending (dist,id),
 * padded with UINT32_MAX) and per-query counters (nq x 8 u32: expansions, tie
 * expansions, evals, in-pool drops, adjacency slots, rows reranked (== pool
 * size at the reference rerank depth or without rerank), max tie depth,
 * status).  Any output may be NULL. */
qvg_status qvg_search_ex(qvg_index* index, const float* queries, uint64_t nq, uint32_t k,
                         uint32_t ef, const qvg_search_opts* opts, uint32_t* out_ids,
                         float* out_scores, uint32_t* out_count, int32_t* out_query_status,
                         uint32_t* out_pool_ids, uint32_t* out_pool_dists,
                         uint32_t* out_pool_size, uint32_t* out_query_counters,
                         qvg_stats* stats);

/* Beam search only, from given code words (nq x 2W u64, reference layout) and
 * an entry point (UINT32_MAX = index entry): beam_search_words' pool. */
qvg_status qvg_beam_search(qvg_index* index, const uint64_t* query_codes, uint64_t nq,
                           uint32_t ef, uint32_t entry_point, uint32_t* out_pool_ids,
                           uint32_t* out_pool_dists, uint32_t* out_pool_size,
                           qvg_stats* stats);

/* Query-path encode on the GPU: out_normalized nq x dim f32, out_codes nq x 2W
 * u64 (reference layout), out_tau nq (nullable), out_query_status nq. */
qvg_status qvg_encode(int device, const float* x, uint64_t nq, uint32_t dim,
                      float* out_normalized, uint64_t* out_codes, float* out_tau,
                      int32_t* out_query_status);

/* SM2 distance of query code rows a (npairs x 2W, reference layout) against
 * node ids of the index: out[i] = sm2(a_i, node ids[i]). */
qvg_status qvg_sm2_distance(qvg_index* index, const uint64_t* query_codes,
                            const uint32_t* ids, uint64_t npairs, uint32_t* out);

/* GPU graph construction (BQ-space Vamana, batched insertion).  data: n x dim
 * f32 (normalised on device exactly like stage0_preinstall).  passes: 1 or 2
 * (2 = alpha 1.0 then `alpha`).  batch: insertion batch size (0 = default). */
typedef struct qvg_build_params {
    uint32_t m;        /* max degree R = 2m */
    uint32_t ef_c;     /* construction beam width L */
    float alpha;       /* final-pass alpha */
    uint32_t passes;   /* 1 or 2 */
    uint32_t batch;    /* max insertion batch (0 = 65536) */
    uint64_t seed;     /* insertion-order shuffle */
    uint32_t prune_candidates; /* RobustPrune candidates besides the L-best pool
                                  (+ the node's row on the 2nd pass): bit 0 / bit 1
                                  = also Vamana's visited set V (the search's
                                  expanded nodes) on the first / the final alpha
                                  pass; 0 = default (3: both passes) */
    uint32_t reserved[3];
} qvg_build_params;

typedef struct qvg_build_stats {
    double seconds;
    uint64_t reprunes;
    uint64_t batches;
    double mean_degree;
    uint32_t min_degree, max_degree;
} qvg_build_stats;

qvg_status qvg_build(const float* data, uint64_t n, uint32_t dim, const qvg_build_params* p,
                     int device, qvg_index** out, qvg_build_stats* stats);

/* qivr::robust_prune (graph.hpp:162-183), batched, with dist_fn = the SM2
 * distance of the index's codes (SignatureStore::distance, as link_node /
 * insert_bidirectional bind it, builder.cpp:130-131).  Task t prunes the
 * candidates cand_ids/cand_dists[offsets[t], offsets[t+1]) (cand_dists =
 * dist(c, target), the Candidate::dist the caller computed): ascending (dist,
 * id), c kept iff float(c.dist) <= alpha * float(dist(c, s)) for every kept s,
 * at most max_degree kept.  Output: out_ids[t * max_degree ...] (unused slots
 * UINT32_MAX), out_count[t].  The builder's own prune kernel (qvg_build) runs
 * it.  Candidate ids must be distinct within a task (they are at every
 * reference call site); at most 480 per task; 1 <= max_degree <= 128.  All
 * pointers host or device. */
qvg_status qvg_robust_prune(qvg_index* index, uint64_t ntasks, const uint64_t* offsets,
                            const uint32_t* cand_ids, const uint32_t* cand_dists,
                            uint32_t max_degree, float alpha, uint32_t* out_ids,
                            uint32_t* out_count);

/* ---- evaluation support ------------------------ */

/* Scorers of qivr::Scorer (eval.hpp:13). */
#define QVG_SCORER_FLOAT_COSINE 0
#define QVG_SCORER_SM2 1
#define QVG_SCORER_SIGN1 2
#define QVG_SCORER_SQ2 3

/* qivr::brute_force_topk (eval.hpp:19-21, eval.cpp:81-168): exact top-k of
 * every base row per query.  float_cosine ranks dot_f32 (the 4-chain double
 * dot) descending; sm2 / sign1 / sq2 rank the raw codes' distances ascending; ties
 * by ascending id; exclude_identity skips row j == query index.  base n x dim,
 * queries nq x dim (host or device).  out_ids nq x k (rows shorter than k
 * padded with UINT32_MAX); out_scores (float_cosine) / out_dists (code
 * scorers) / out_count nullable.  k <= 256. */
qvg_status qvg_brute_force_topk(int device, const float* base, uint64_t n, const float* queries,
                                uint64_t nq, uint32_t dim, uint32_t k, int scorer,
                                int exclude_identity, uint32_t* out_ids, float* out_scores,
                                uint32_t* out_dists, uint32_t* out_count);

/* Raw (unnormalised) row encoders of the code scorers: sm2 = encode_sm2
 * (encoding.cpp:32-58; out n x 2W u64, reference layout, out_tau n x f32
 * nullable), sign1 = encode_sign1 (encoding.cpp:60-72; n x W u64), sq2 =
 * encode_sq2 (encoding.cpp:74-106; n x dim u8).  Non-finite input ->
 * QVG_INVALID_ARGUMENT "encode: non-finite coordinate". */
qvg_status qvg_encode_rows(int device, const float* x, uint64_t n, uint32_t dim, int scorer,
                           void* out_codes, float* out_tau);

/* qivr::ProbeReport (eval.hpp:28-33) */
typedef struct qvg_probe_report {
    double overlap_at_k;
    uint64_t sample_size;
    uint32_t k;
    uint32_t go; /* overlap_at_k > 0.5 */
} qvg_probe_report;

/* qivr::compatibility_probe (eval.hpp:35-37, eval.cpp:196-222): the first
 * min(sample_size, n) rows; the first min(1000, sample) of them as queries
 * against the sample with exclude_identity; overlap = recall_at_k(code
 * ranking, float ranking, k).  Errors as the reference (sample < 100,
 * all-identical sample). */
qvg_status qvg_compatibility_probe(int device, const float* data, uint64_t n, uint32_t dim,
                                   uint64_t sample_size, uint32_t k, int scorer,
                                   qvg_probe_report* out);

/* qivr::EncodingDiagnostics (encoding.hpp) */
typedef struct qvg_encoding_diagnostics {
    uint64_t sample_size;
    double p_s; /* strong bits / (rows * dim) */
    double nu2; /* (1 + 3 p_s)^2 */
} qvg_encoding_diagnostics;

/* qivr::strong_bit_rate: index != NULL -> the index's signatures
 * (encoding.cpp:150-167, data ignored); else raw-encoded data rows
 * (encoding.cpp:132-148) on `device`. */
qvg_status qvg_strong_bit_rate(qvg_index* index, const float* data, uint64_t count, uint32_t dim,
                               int device, qvg_encoding_diagnostics* out);

#ifdef __cplusplus
}
#endif

#endif /* QVG_H_ */

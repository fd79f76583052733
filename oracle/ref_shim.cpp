// TEST INFRASTRUCTURE ONLY — never linked into the product (paper_2605_02171_b200/).
//
// A thin extern "C" shim over the UNMODIFIED reference library `qivr`
// (/root/reference/proj/core/src/*.cpp), compiled together with it by
// oracle/Makefile into oracle/_ref/libqivr_ref.so.  Only tests/, the smoke
// check and bench.py's CPU-baseline / reference leg load it.  Every entry point
// forwards to the reference's own public API; nothing here re-implements the
// algorithm:
//   build      -> qivr::build_index            (builder.cpp:137-155)
//   save/load  -> qivr::save_index/load_index  (store_io.cpp:99-169)
//   batch      -> qivr::run_query_batch        (eval.cpp:225-247)
//   pool       -> qivr::beam_search_words      (search.cpp:27-81)
//   encode     -> qivr::normalize_l2 + encode_sm2_into (vec_math.hpp:37-44, encoding.cpp:32-45)
//   gt         -> qivr::brute_force_topk       (eval.cpp:81-169)
//   prune      -> qivr::robust_prune           (graph.hpp:162-183)
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "qivr/builder.hpp"
#include "qivr/encoding.hpp"
#include "qivr/eval.hpp"
#include "qivr/graph.hpp"
#include "qivr/index.hpp"
#include "qivr/search.hpp"
#include "qivr/store_io.hpp"
#include "qivr/vec_math.hpp"

namespace {

thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 runtime_error, 3 other
template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

qivr::Index* as_index(void* h) { return static_cast<qivr::Index*>(h); }

}  // namespace

extern "C" {

const char* qref_last_error(void) { return g_err.c_str(); }

int qref_build(const float* data, uint64_t n, uint32_t dim, uint32_t m, uint32_t ef_c,
               float alpha, uint32_t threads, uint64_t seed, void** out) {
    *out = nullptr;
    return guarded([&] {
        qivr::BuildParams p;
        p.m = m;
        p.ef_c = ef_c;
        p.alpha = alpha;
        p.threads = threads;
        p.seed = seed;
        *out = new qivr::Index(qivr::build_index(data, n, dim, p));
    });
}

int qref_load(const char* path, int mapped, void** out) {
    *out = nullptr;
    return guarded([&] {
        *out = new qivr::Index(qivr::load_index(
            path, mapped ? qivr::ColdMode::mapped : qivr::ColdMode::eager));
    });
}

int qref_save(void* h, const char* path) {
    return guarded([&] { qivr::save_index(*as_index(h), path); });
}

void qref_free(void* h) { delete as_index(h); }

void qref_info(void* h, uint64_t* n, uint32_t* dim, uint32_t* m, uint32_t* entry,
               float* alpha) {
    const qivr::Index& ix = *as_index(h);
    *n = ix.size();
    *dim = ix.dim;
    *m = ix.params.m;
    *entry = ix.entry_point;
    *alpha = ix.params.alpha;
}

const uint64_t* qref_codes(void* h) { return as_index(h)->signatures.raw(); }
const uint32_t* qref_adj(void* h) { return as_index(h)->adjacency.raw(); }
const float* qref_cold(void* h) { return as_index(h)->cold.raw(); }
uint64_t qref_cold_access_count(void* h) { return as_index(h)->cold.access_count(); }
void qref_reset_cold_access_count(void* h) { as_index(h)->cold.reset_access_count(); }

// Batch search through the reference's own batch entry point.  Result rows are
// padded with id UINT32_MAX / score NaN past out_count[i].
int qref_run_query_batch(void* h, const float* queries, uint64_t nq, uint32_t ef, uint32_t k,
                         uint32_t threads, uint32_t* out_ids, float* out_scores,
                         uint32_t* out_count) {
    return guarded([&] {
        qivr::SearchParams sp{ef, k};
        sp.validate();
        auto res = qivr::run_query_batch(*as_index(h), queries, nq, sp, threads);
        for (uint64_t i = 0; i < nq; ++i) {
            const auto& r = res[i];
            out_count[i] = static_cast<uint32_t>(r.ids.size());
            for (uint32_t j = 0; j < k; ++j) {
                out_ids[i * k + j] = j < r.ids.size() ? r.ids[j] : UINT32_MAX;
                out_scores[i * k + j] = j < r.ids.size() ? r.scores[j] : NAN;
            }
        }
    });
}

// Single query through qivr::query (throws exactly like the reference).
int qref_query(void* h, const float* q, uint32_t qdim, uint32_t ef, uint32_t k,
               uint32_t* out_ids, float* out_scores, uint32_t* out_count) {
    return guarded([&] {
        auto r = qivr::query(*as_index(h), {q, qdim}, qivr::SearchParams{ef, k});
        *out_count = static_cast<uint32_t>(r.ids.size());
        for (size_t j = 0; j < r.ids.size(); ++j) {
            out_ids[j] = r.ids[j];
            out_scores[j] = r.scores[j];
        }
    });
}

// Query-path encode: finite check, normalize_l2, encode_sm2_into — the exact
// sequence of qivr::query (search.cpp:128-136).  Codes in the reference layout
// (W pos words then W strong words).
int qref_encode_query(const float* x, uint32_t dim, float* out_norm, uint64_t* out_code,
                      float* out_tau) {
    return guarded([&] {
        std::vector<float> v(x, x + dim);
        for (float f : v)
            if (!std::isfinite(f)) throw std::invalid_argument("query: non-finite coordinate");
        qivr::normalize_l2(v.data(), v.size());
        const size_t w = qivr::words_for_dim(dim);
        *out_tau = qivr::encode_sm2_into(v, out_code, out_code + w);
        std::memcpy(out_norm, v.data(), dim * sizeof(float));
    });
}

// Raw encode (no normalisation): encode_sm2 on the vector as given.
int qref_encode_raw(const float* x, uint32_t dim, uint64_t* out_code, float* out_tau) {
    return guarded([&] {
        auto sig = qivr::encode_sm2({x, dim});
        const size_t w = qivr::words_for_dim(dim);
        std::memcpy(out_code, sig.pos_bits.data(), w * 8);
        std::memcpy(out_code + w, sig.strong_bits.data(), w * 8);
        *out_tau = sig.tau;
    });
}

uint32_t qref_sm2_distance_words(const uint64_t* a, const uint64_t* b, uint64_t words) {
    return qivr::sm2_distance_words(a, a + words, b, b + words, words);
}

float qref_dot_f32(const float* a, const float* b, uint64_t n) { return qivr::dot_f32(a, b, n); }

// Pool (ids + dists, ascending (dist,id)) of beam_search_words for given
// query code words (reference layout), from `entry` (UINT32_MAX = index entry).
int qref_beam_search(void* h, const uint64_t* qcode, uint32_t ef, uint32_t entry,
                     uint32_t* out_ids, uint32_t* out_dists, uint32_t* out_n) {
    return guarded([&] {
        const qivr::Index& ix = *as_index(h);
        if (entry == UINT32_MAX) entry = ix.entry_point;
        if (entry >= ix.size()) throw std::invalid_argument("beam_search: invalid entry point");
        thread_local qivr::VisitedSet visited;
        thread_local std::vector<uint32_t> row;
        const size_t w = ix.signatures.words();
        auto pool = qivr::beam_search_words(ix, qcode, qcode + w, ef, entry, visited, row,
                                            /*lock_adjacency=*/false);
        *out_n = static_cast<uint32_t>(pool.size());
        for (size_t i = 0; i < pool.size(); ++i) {
            out_ids[i] = pool[i].id;
            out_dists[i] = pool[i].dist;
        }
    });
}

// Exact top-k by brute force. scorer: 0 float_cosine, 1 sm2.
// qivr::encode_sq2 (encoding.cpp:74-106): dim bytes
int qref_encode_sq2(const float* x, uint32_t dim, uint8_t* out) {
    return guarded([&] {
        const auto c = qivr::encode_sq2({x, dim});
        std::memcpy(out, c.codes.data(), dim);
    });
}

// qivr::encode_sign1 (encoding.cpp:60-72): ceil(dim/64) words
int qref_encode_sign1(const float* x, uint32_t dim, uint64_t* out) {
    return guarded([&] {
        const auto c = qivr::encode_sign1({x, dim});
        std::memcpy(out, c.bits.data(), c.bits.size() * 8);
    });
}

// scorer 0..3 = float_cosine, sm2, sign1, sq2; rows shorter than k padded
// with UINT32_MAX
int qref_brute_force_topk_ex(const float* base, uint64_t n, const float* queries, uint64_t nq,
                             uint32_t dim, uint32_t k, uint32_t threads, int scorer,
                             int exclude_identity, uint32_t* out) {
    return guarded([&] {
        static const qivr::Scorer sc[4] = {qivr::Scorer::float_cosine, qivr::Scorer::sm2,
                                           qivr::Scorer::sign1, qivr::Scorer::sq2};
        auto res = qivr::brute_force_topk(base, n, queries, nq, dim, k, sc[scorer & 3], threads,
                                          exclude_identity != 0);
        for (uint64_t i = 0; i < nq; ++i)
            for (uint32_t j = 0; j < k; ++j)
                out[i * k + j] = j < res[i].size() ? res[i][j] : UINT32_MAX;
    });
}

int qref_compatibility_probe(const float* data, uint64_t n, uint32_t dim, uint64_t sample_size,
                             uint32_t k, int scorer, double* overlap, uint64_t* sample_n,
                             int* go) {
    return guarded([&] {
        static const qivr::Scorer sc[4] = {qivr::Scorer::float_cosine, qivr::Scorer::sm2,
                                           qivr::Scorer::sign1, qivr::Scorer::sq2};
        const auto r = qivr::compatibility_probe(data, n, dim, sample_size, k, sc[scorer & 3]);
        *overlap = r.overlap_at_k;
        *sample_n = r.sample_size;
        *go = r.go ? 1 : 0;
    });
}

// strong_bit_rate(data) (encoding.cpp:132-148) and (store) (encoding.cpp:150-167)
int qref_strong_bit_rate_data(const float* data, uint64_t count, uint32_t dim, double* p_s,
                              double* nu2) {
    return guarded([&] {
        const auto d = qivr::strong_bit_rate(data, count, dim);
        *p_s = d.p_s;
        *nu2 = d.nu2;
    });
}

int qref_strong_bit_rate_index(void* h, double* p_s, double* nu2, uint64_t* sample) {
    return guarded([&] {
        const auto d = qivr::strong_bit_rate(as_index(h)->signatures);
        *p_s = d.p_s;
        *nu2 = d.nu2;
        *sample = d.sample_size;
    });
}

int qref_brute_force_topk(const float* base, uint64_t n, const float* queries, uint64_t nq,
                          uint32_t dim, uint32_t k, uint32_t threads, int scorer,
                          uint32_t* out) {
    return guarded([&] {
        auto res = qivr::brute_force_topk(base, n, queries, nq, dim, k,
                                          scorer == 0 ? qivr::Scorer::float_cosine
                                                      : qivr::Scorer::sm2,
                                          threads, false);
        for (uint64_t i = 0; i < nq; ++i)
            for (uint32_t j = 0; j < k; ++j)
                out[i * k + j] = j < res[i].size() ? res[i][j] : UINT32_MAX;
    });
}

// robust_prune over the index's signature store (BQ distances).  Candidates as
// parallel (id, dist) arrays; returns kept ids in selection order.
int qref_robust_prune(void* h, const uint32_t* ids, const uint32_t* dists, uint32_t n,
                      uint32_t max_degree, float alpha, uint32_t* out, uint32_t* out_n) {
    return guarded([&] {
        const qivr::SignatureStore& s = as_index(h)->signatures;
        std::vector<qivr::Candidate> c(n);
        for (uint32_t i = 0; i < n; ++i) c[i] = {ids[i], dists[i]};
        auto kept = qivr::robust_prune(
            std::move(c), [&s](uint32_t a, uint32_t b) { return s.distance(a, b); },
            max_degree, alpha);
        *out_n = static_cast<uint32_t>(kept.size());
        std::memcpy(out, kept.data(), kept.size() * sizeof(uint32_t));
    });
}

// Index assembled from raw parts in the reference layouts (used to hand a
// GPU-built or hand-made graph to the reference search).  `cold` must already
// be unit-normalised; codes in SignatureStore layout; adj in slot layout.
int qref_from_parts(const uint64_t* codes, const uint32_t* adj, const float* cold, uint64_t n,
                    uint32_t dim, uint32_t m, uint32_t entry, float alpha, void** out) {
    *out = nullptr;
    return guarded([&] {
        auto ix = std::make_unique<qivr::Index>();
        ix->params.m = m;
        ix->params.alpha = alpha;
        ix->dim = dim;
        ix->entry_point = entry;
        ix->signatures = qivr::SignatureStore(n, dim);
        std::memcpy(ix->signatures.raw(), codes, ix->signatures.size_bytes());
        ix->adjacency = qivr::AdjacencyTable(static_cast<uint32_t>(n), 2 * m);
        std::memcpy(ix->adjacency.raw(), adj, ix->adjacency.size_bytes());
        ix->cold = qivr::ColdStore::owned(std::vector<float>(cold, cold + n * dim), n, dim);
        *out = ix.release();
    });
}

// Reference Index over raw (unnormalised) vectors and a given graph: the
// reference's own stage0_preinstall (builder.cpp:59-88: normalize_l2 +
// SignatureStore::encode per row, bulk adjacency, medoid entry) followed by
// installing the given adjacency slots and entry point.  Used to run the
// reference search on a cached graph without repeating the build.
int qref_index_from_graph(const float* data, uint64_t n, uint32_t dim, const uint32_t* adj,
                          uint32_t m, uint32_t entry, float alpha, uint32_t threads,
                          void** out) {
    *out = nullptr;
    return guarded([&] {
        qivr::BuildParams p;
        p.m = m;
        p.alpha = alpha;
        p.threads = threads;
        auto ix = std::make_unique<qivr::Index>(qivr::stage0_preinstall(data, n, dim, p));
        std::memcpy(ix->adjacency.raw(), adj, ix->adjacency.size_bytes());
        ix->entry_point = entry;
        *out = ix.release();
    });
}

}  // extern "C"

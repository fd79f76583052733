// qvg.hpp — header-only C++ drop-in over the qvg C-ABI (qvg.h).
//
// Mirrors the reference's query surface (paths under /root/reference/proj/core):
//   qivr::run_query_batch(const Index&, const float*, size_t, const SearchParams&,
//                         uint32_t threads)            eval.hpp:42-44, eval.cpp:225-247
//   qivr::query(const Index&, span<const float>, const SearchParams&)
//                                                      search.hpp:95-98, search.cpp:122-143
//   qivr::load_index(path, ColdMode)                   store_io.hpp:40
// with the same error classes: std::invalid_argument for bad params / queries
// (search.hpp:16-19, search.cpp:124-131, vec_math.hpp:39-41), std::runtime_error
// for file / format problems (store_io.cpp:48-95).
//
// When the reference headers are on the include path, qvg::GpuIndex is built
// straight from a qivr::Index through its public raw() accessors and
// qvg::run_query_batch returns std::vector<qivr::SearchResult>:
//
//     qivr::Index index = qivr::load_index(path, qivr::ColdMode::eager);
//     qvg::GpuIndex gpu(index);                          // one-time upload to HBM
//     auto results = qvg::run_query_batch(gpu, queries, nq, qivr::SearchParams{64, 10});
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "qvg.h"

#if defined(__has_include)
#if __has_include("qivr/search.hpp") && __has_include("qivr/index.hpp")
#include "qivr/index.hpp"
#include "qivr/search.hpp"
#define QVG_HAVE_QIVR 1
#endif
#endif

namespace qvg {

class CudaError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

class CapacityOverflow : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

inline void check(qvg_status st) {
    switch (st) {
        case QVG_OK: return;
        case QVG_INVALID_ARGUMENT: throw std::invalid_argument(qvg_last_error());
        case QVG_RUNTIME_ERROR: throw std::runtime_error(qvg_last_error());
        case QVG_CAPACITY_OVERFLOW: throw CapacityOverflow(qvg_last_error());
        case QVG_OUT_OF_MEMORY: throw std::bad_alloc();
        default: throw CudaError(qvg_last_error());
    }
}

/// Results of a batch: row-major nq x k, rows padded past count[i].
struct BatchResults {
    std::vector<uint32_t> ids;
    std::vector<float> scores;
    std::vector<uint32_t> count;
    uint32_t k = 0;
};

/// One HBM-resident index (move-only handle).
class GpuIndex {
public:
    GpuIndex(const uint64_t* codes, uint64_t n, uint32_t dim, const uint32_t* adj_slots,
             uint32_t max_degree, const float* cold, uint32_t entry_point, int device = 0) {
        check(qvg_index_create(codes, n, dim, adj_slots, max_degree, cold, entry_point, device,
                               &h_));
    }

#ifdef QVG_HAVE_QIVR
    /// Upload a reference index through its public raw() layouts
    /// (encoding.hpp:247-248, graph.hpp:135-136, cold_store.hpp:58).
    explicit GpuIndex(const qivr::Index& ix, int device = 0)
        : GpuIndex(ix.signatures.raw(), ix.size(), ix.dim, ix.adjacency.raw(),
                   ix.adjacency.max_degree(), ix.cold.raw(), ix.entry_point, device) {}
#endif

    /// qivr::load_index equivalent: .qivr v1 straight into HBM.
    static GpuIndex load(const std::string& path, int device = 0) {
        qvg_index* h = nullptr;
        check(qvg_index_load(path.c_str(), device, &h));
        return GpuIndex(h);
    }

    GpuIndex(GpuIndex&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    GpuIndex& operator=(GpuIndex&& o) noexcept {
        if (this != &o) {
            if (h_) qvg_index_destroy(h_);
            h_ = std::exchange(o.h_, nullptr);
        }
        return *this;
    }
    GpuIndex(const GpuIndex&) = delete;
    GpuIndex& operator=(const GpuIndex&) = delete;
    ~GpuIndex() {
        if (h_) qvg_index_destroy(h_);
    }

    void save(const std::string& path) const { check(qvg_index_save(h_, path.c_str())); }

    uint32_t dim() const {
        uint32_t d = 0;
        check(qvg_index_info(h_, nullptr, &d, nullptr, nullptr));
        return d;
    }

    /// Batched search; throws std::invalid_argument like the reference.
    BatchResults search(const float* queries, size_t nq, uint32_t k, uint32_t ef) const {
        BatchResults r;
        r.k = k;
        r.ids.resize(nq * k);
        r.scores.resize(nq * k);
        r.count.resize(nq);
        check(qvg_search(h_, queries, nq, k, ef, r.ids.data(), r.scores.data(), r.count.data(),
                         nullptr, nullptr));
        return r;
    }

    qvg_index* handle() const { return h_; }

private:
    explicit GpuIndex(qvg_index* h) : h_(h) {}
    qvg_index* h_ = nullptr;
};

#ifdef QVG_HAVE_QIVR
/// Drop-in for qivr::run_query_batch (eval.cpp:225-247).  `threads` is
/// accepted for source compatibility and ignored: one launch serves the batch.
inline std::vector<qivr::SearchResult> run_query_batch(const GpuIndex& index, const float* queries,
                                                       size_t nq, const qivr::SearchParams& params,
                                                       uint32_t threads = 0) {
    (void)threads;
    params.validate();  // same exceptions, same order as the reference
    const BatchResults r = index.search(queries, nq, params.k, params.ef);
    std::vector<qivr::SearchResult> out(nq);
    for (size_t i = 0; i < nq; ++i) {
        out[i].ids.assign(r.ids.begin() + i * params.k, r.ids.begin() + i * params.k + r.count[i]);
        out[i].scores.assign(r.scores.begin() + i * params.k,
                             r.scores.begin() + i * params.k + r.count[i]);
    }
    return out;
}

/// Drop-in for qivr::query (search.cpp:122-143) — single query.
inline qivr::SearchResult query(const GpuIndex& index, std::span<const float> q,
                                const qivr::SearchParams& params) {
    params.validate();
    if (q.size() != index.dim()) throw std::invalid_argument("query: dimension mismatch");
    return run_query_batch(index, q.data(), 1, params)[0];
}
#endif

}  // namespace qvg

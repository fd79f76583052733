// Drop-in check, written the way a maintainer of the reference would: build a
// qivr::Index with the reference's own builder, upload it with
// qvg::GpuIndex(const qivr::Index&), and compare qivr::run_query_batch with
// qvg::run_query_batch (ids equal, score bit patterns equal), plus the
// reference's error classes.  Built by oracle/Makefile (dropin target) against
// the reference headers and oracle/_ref/libqivr_ref.so; run by
// tests/test_gpu_parity.py::test_cpp_dropin on the GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <vector>

#include "qivr/builder.hpp"
#include "qivr/eval.hpp"
#include "qivr/search.hpp"
#include "qvg.hpp"

int main() {
    const size_t n = 5000, nq = 300;
    const uint32_t dim = 96;
    std::mt19937_64 rng(17);
    std::normal_distribution<float> g(0.0f, 1.0f);
    std::vector<float> data(n * dim), queries(nq * dim);
    for (auto& v : data) v = g(rng);
    for (auto& v : queries) v = g(rng);

    qivr::BuildParams bp;
    bp.m = 8;
    bp.ef_c = 48;
    bp.threads = 4;
    qivr::Index index = qivr::build_index(data.data(), n, dim, bp);
    qvg::GpuIndex gpu(index);

    int failures = 0;
    for (uint32_t ef : {10u, 32u, 64u, 200u}) {
        qivr::SearchParams sp{ef, 10};
        auto want = qivr::run_query_batch(index, queries.data(), nq, sp, 4);
        auto got = qvg::run_query_batch(gpu, queries.data(), nq, sp);
        for (size_t i = 0; i < nq; ++i) {
            bool same = want[i].ids == got[i].ids && want[i].scores.size() == got[i].scores.size();
            for (size_t j = 0; same && j < want[i].scores.size(); ++j)
                same = std::memcmp(&want[i].scores[j], &got[i].scores[j], 4) == 0;
            if (!same) {
                ++failures;
                std::printf("mismatch ef=%u query=%zu\n", ef, i);
                break;
            }
        }
    }
    // error classes match the reference
    auto expect_invalid = [&](auto fn, const char* what) {
        try {
            fn();
            std::printf("no exception: %s\n", what);
            ++failures;
        } catch (const std::invalid_argument&) {
        }
    };
    expect_invalid([&] { qvg::run_query_batch(gpu, queries.data(), 1, qivr::SearchParams{4, 5}); },
                   "ef < k");
    std::vector<float> zero(dim, 0.0f);
    expect_invalid([&] { qvg::run_query_batch(gpu, zero.data(), 1, qivr::SearchParams{16, 5}); },
                   "zero query");
    std::vector<float> bad(dim, 1.0f);
    bad[3] = NAN;
    expect_invalid([&] { qvg::run_query_batch(gpu, bad.data(), 1, qivr::SearchParams{16, 5}); },
                   "NaN query");
    expect_invalid([&] { qvg::query(gpu, std::span<const float>(bad.data(), 3), qivr::SearchParams{16, 5}); },
                   "dim mismatch");
    std::printf("dropin: %s\n", failures ? "FAIL" : "OK");
    return failures ? 1 : 0;
}

// K5 — GPU batched BQ-space Vamana construction (secondary path).
// Reference: build_index / stage0_preinstall / select_entry_point / link_node
// (builder.cpp:59-155), robust_prune + insert_bidirectional (graph.hpp:162-227).
#include "qvg_internal.cuh"

using namespace qvg;

extern "C" qvg_status qvg_build(const float* data, uint64_t n, uint32_t dim,
                                const qvg_build_params* p, int device, qvg_index** out,
                                qvg_build_stats* stats) {
    (void)data; (void)n; (void)dim; (void)p; (void)device; (void)stats;
    if (out) *out = nullptr;
    set_error("qvg_build: not implemented yet");
    return QVG_NOT_IMPLEMENTED;
}

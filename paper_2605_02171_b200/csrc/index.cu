// HBM-resident index: creation from the reference's raw layouts, .qivr v1
// load/save, export back to the reference layouts.
//
// Reference layouts consumed (paths under /root/reference/proj/core):
//   SignatureStore::raw  encoding.hpp:217-232, 247-248  node-major, W pos words
//                        then W strong words per node
//   AdjacencyTable::raw  graph.hpp:65-67, 118-126, 135-136  [deg, id_0..id_{R-1}],
//                        unused slots zero (zero is a valid id: honour deg)
//   ColdStore::raw       cold_store.hpp:58  n x dim f32, unit rows
//   .qivr v1             store_io.hpp:12-30, store_io.cpp:34-126 (64-B LE header,
//                        sig | adj | cold segments), validate_header
//                        store_io.cpp:77-95 (fail closed)
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "qvg_internal.cuh"

namespace qvg {

namespace {

// Relayout one adjacency slot: validate, drop repeated ids (keep the first —
// the reference's visited test makes a repeat a no-op, search.cpp:62-63),
// keep row order, fill the tail with kSentinel.
__global__ void adj_relayout_kernel(const uint32_t* __restrict__ slots, uint64_t n, uint32_t R,
                                    uint32_t RS, uint32_t* __restrict__ out,
                                    uint32_t* __restrict__ err) {
    const uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (u >= n) return;
    const uint32_t* s = slots + u * (uint64_t)(R + 1);
    uint32_t* o = out + u * (uint64_t)RS;
    uint32_t deg = s[0];
    if (deg > R) {
        atomicOr(err, 1u);
        deg = 0;
    }
    uint32_t m = 0;
    for (uint32_t i = 0; i < deg; ++i) {
        const uint32_t v = s[1 + i];
        if (v >= n) {
            atomicOr(err, 2u);
            continue;
        }
        bool dup = false;
        for (uint32_t j = 0; j < m; ++j) dup |= o[j] == v;
        if (!dup) o[m++] = v;
    }
    for (uint32_t i = m; i < RS; ++i) o[i] = kSentinel;
}

// back to the reference slot layout (degree + ids, zero-filled tail)
__global__ void adj_export_kernel(const uint32_t* __restrict__ rows, uint64_t n, uint32_t R,
                                  uint32_t RS, uint32_t* __restrict__ slots) {
    const uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (u >= n) return;
    const uint32_t* r = rows + u * (uint64_t)RS;
    uint32_t* s = slots + u * (uint64_t)(R + 1);
    uint32_t d = 0;
    for (uint32_t i = 0; i < R; ++i) {
        const uint32_t v = r[i];
        if (v != kSentinel) s[1 + d++] = v;
    }
    for (uint32_t i = d; i < R; ++i) s[1 + i] = 0;
    s[0] = d;
}

uint32_t words_for_dim(uint32_t d) { return (d + 63) / 64; }

void free_index(qvg_index* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    cudaFree(h->d_codes);
    cudaFree(h->d_adj);
    cudaFree(h->d_cold);
    Buffer* bufs[] = {&h->s_in,   &h->s_qn,     &h->s_qc,     &h->s_qst,    &h->s_ids,
                      &h->s_sc,   &h->s_cnt,    &h->s_pool_i, &h->s_pool_d, &h->s_pool_n,
                      &h->s_qctr, &h->s_counter, &h->s_exact, &h->s_pair_ids, &h->s_pair_out, &h->s_st,
                      &h->s_susp};
    for (Buffer* b : bufs) cudaFree(b->p);
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
    if (h->ev_copy) cudaEventDestroy(h->ev_copy);
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    if (h->ready_host) cudaFreeHost(h->ready_host);
    if (h->host_flags) cudaFreeHost(h->host_flags);
    if (h->own_stream) cudaStreamDestroy(h->own_stream);
    delete h;
}

qvg_status alloc_handle(int device, uint64_t n, uint32_t dim, uint32_t R, uint32_t entry,
                        qvg_index** out) {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
    auto* h = new qvg_index();
    h->device = device;
    e = cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        free_index(h);
        return cuda_status(e, "cudaStreamCreate");
    }
    h->stream = h->own_stream;
    for (auto& ev : h->ev) cudaEventCreate(&ev);
    DevIndex& ix = h->ix;
    ix.n = n;
    ix.dim = dim;
    ix.W = words_for_dim(dim);
    ix.R = R;
    ix.RS = (R + 3) & ~3u;
    ix.Dp = (dim + 3) & ~3u;
    ix.entry = entry;
    e = cudaMalloc(&h->d_codes, n * ix.W * sizeof(uint4));
    if (e == cudaSuccess) e = cudaMalloc(&h->d_adj, n * ix.RS * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMalloc(&h->d_cold, n * ix.Dp * sizeof(float));
    if (e != cudaSuccess) {
        free_index(h);
        return cuda_status(e, "cudaMalloc(index)");
    }
    ix.codes = static_cast<const uint4*>(h->d_codes);
    ix.adj = static_cast<const uint32_t*>(h->d_adj);
    ix.cold = static_cast<const float*>(h->d_cold);
    h->has_tmap = make_code_tmap(&h->tmap, h->d_codes, n, ix.W);
    *out = h;
    return QVG_OK;
}

qvg_status check_geometry(uint64_t n, uint32_t dim, uint32_t R, uint32_t entry) {
    if (n == 0) {
        set_error("index: no nodes");
        return QVG_INVALID_ARGUMENT;
    }
    if (n >= 0xFFFFFFFFull) {
        set_error("index: too many nodes for 32-bit ids");
        return QVG_INVALID_ARGUMENT;
    }
    if (dim == 0) {
        set_error("index: zero dimension");
        return QVG_INVALID_ARGUMENT;
    }
    if (R == 0 || R > kMaxDegree) {
        set_error("index: max_degree must be in [1, " + std::to_string(kMaxDegree) + "]");
        return QVG_INVALID_ARGUMENT;
    }
    if (entry >= n) {
        set_error("index: invalid entry point");
        return QVG_INVALID_ARGUMENT;
    }
    return QVG_OK;
}

// codes/adj may be host or device pointers (cudaMemcpyDefault, UVA)
qvg_status upload_hot(qvg_index* h, const uint64_t* codes, const uint32_t* adj) {
    const DevIndex& ix = h->ix;
    cudaStream_t s = h->stream;
    void* tmp = nullptr;
    const size_t code_bytes = ix.n * 2 * ix.W * sizeof(uint64_t);
    const size_t adj_bytes = ix.n * (size_t)(ix.R + 1) * sizeof(uint32_t);
    cudaError_t e = cudaMalloc(&tmp, code_bytes > adj_bytes ? code_bytes : adj_bytes);
    if (e != cudaSuccess) return cuda_status(e, "cudaMalloc(staging)");
    uint32_t* d_err = nullptr;
    e = cudaMalloc(&d_err, sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemsetAsync(d_err, 0, sizeof(uint32_t), s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(tmp, codes, code_bytes, cudaMemcpyDefault, s);
    if (e == cudaSuccess) {
        launch_codes_to_chunks(static_cast<const uint64_t*>(tmp), ix.n, ix.W,
                               static_cast<uint4*>(h->d_codes), s);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(tmp, adj, adj_bytes, cudaMemcpyDefault, s);
    if (e == cudaSuccess) {
        adj_relayout_kernel<<<(unsigned)((ix.n + 127) / 128), 128, 0, s>>>(
            static_cast<const uint32_t*>(tmp), ix.n, ix.R, ix.RS,
            static_cast<uint32_t*>(h->d_adj), d_err);
        e = cudaGetLastError();
    }
    uint32_t err = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&err, d_err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(tmp);
    cudaFree(d_err);
    if (e != cudaSuccess) return cuda_status(e, "upload(hot segments)");
    if (err & 1u) {
        set_error("AdjacencyTable: degree cap exceeded");
        return QVG_INVALID_ARGUMENT;
    }
    if (err & 2u) {
        set_error("adjacency: neighbor id out of range");
        return QVG_INVALID_ARGUMENT;
    }
    return QVG_OK;
}

qvg_status upload_cold(qvg_index* h, const float* cold) {
    const DevIndex& ix = h->ix;
    cudaError_t e;
    if (ix.Dp == ix.dim) {
        e = cudaMemcpyAsync(h->d_cold, cold, ix.n * (size_t)ix.dim * sizeof(float),
                            cudaMemcpyDefault, h->stream);
    } else {
        e = cudaMemsetAsync(h->d_cold, 0, ix.n * (size_t)ix.Dp * sizeof(float), h->stream);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(h->d_cold, ix.Dp * sizeof(float), cold, ix.dim * sizeof(float),
                                  ix.dim * sizeof(float), ix.n, cudaMemcpyDefault, h->stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    return e == cudaSuccess ? QVG_OK : cuda_status(e, "upload(cold)");
}

// ---- .qivr v1 header (store_io.cpp:34-67) ------------------------------------
constexpr size_t kHeaderBytes = 64;

uint32_t get_u32(const uint8_t* p) {
    return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24;
}
uint64_t get_u64(const uint8_t* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}
void put_u32(uint8_t* p, uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
void put_u64(uint8_t* p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

struct Header {
    uint32_t version;
    uint64_t n;
    uint32_t dim, m, alpha_milli;
    uint64_t entry, sig_off, adj_off, cold_off;
};

struct FileCloser {
    void operator()(FILE* f) const {
        if (f) fclose(f);
    }
};

bool read_at(FILE* f, uint64_t off, void* dst, size_t bytes) {
    if (fseeko(f, (off_t)off, SEEK_SET) != 0) return false;
    return fread(dst, 1, bytes, f) == bytes;
}

}  // namespace

}  // namespace qvg

using namespace qvg;

extern "C" {

qvg_status qvg_index_create(const uint64_t* codes, uint64_t n, uint32_t dim,
                            const uint32_t* adj_slots, uint32_t max_degree, const float* cold,
                            uint32_t entry_point, int device, qvg_index** out) {
    if (!out || !codes || !adj_slots || !cold) {
        set_error("qvg_index_create: null argument");
        return QVG_INVALID_ARGUMENT;
    }
    *out = nullptr;
    qvg_status st = check_geometry(n, dim, max_degree, entry_point);
    if (st != QVG_OK) return st;
    qvg_index* h = nullptr;
    st = alloc_handle(device, n, dim, max_degree, entry_point, &h);
    if (st != QVG_OK) return st;
    h->m = max_degree / 2;
    st = upload_hot(h, codes, adj_slots);
    if (st == QVG_OK) st = upload_cold(h, cold);
    if (st != QVG_OK) {
        free_index(h);
        return st;
    }
    *out = h;
    return QVG_OK;
}

qvg_status qvg_index_load(const char* path, int device, qvg_index** out) {
    if (!out || !path) {
        set_error("qvg_index_load: null argument");
        return QVG_INVALID_ARGUMENT;
    }
    *out = nullptr;
    std::unique_ptr<FILE, FileCloser> f(fopen(path, "rb"));
    if (!f) {
        set_error(std::string("load_index: cannot open ") + path);
        return QVG_RUNTIME_ERROR;
    }
    fseeko(f.get(), 0, SEEK_END);
    const uint64_t file_size = (uint64_t)ftello(f.get());
    if (file_size < kHeaderBytes) {
        set_error("load_index: truncated file");
        return QVG_RUNTIME_ERROR;
    }
    uint8_t hb[kHeaderBytes];
    if (!read_at(f.get(), 0, hb, kHeaderBytes)) {
        set_error("load_index: header read failed");
        return QVG_RUNTIME_ERROR;
    }
    if (std::memcmp(hb, "QIVR", 4) != 0) {
        set_error("load_index: bad magic");
        return QVG_RUNTIME_ERROR;
    }
    Header H;
    H.version = get_u32(hb + 4);
    if (H.version != 1) {
        set_error("load_index: unsupported version " + std::to_string(H.version));
        return QVG_RUNTIME_ERROR;
    }
    H.n = get_u64(hb + 8);
    H.dim = get_u32(hb + 16);
    H.m = get_u32(hb + 20);
    H.alpha_milli = get_u32(hb + 24);
    H.entry = get_u64(hb + 28);
    H.sig_off = get_u64(hb + 36);
    H.adj_off = get_u64(hb + 44);
    H.cold_off = get_u64(hb + 52);
    // validate_header (store_io.cpp:77-95)
    if (H.n == 0 || H.dim == 0 || H.m == 0) {
        set_error("load_index: degenerate header fields");
        return QVG_RUNTIME_ERROR;
    }
    const uint64_t W = words_for_dim(H.dim);
    const uint64_t sig_sz = H.n * 2 * W * 8, adj_sz = H.n * (2ull * H.m + 1) * 4,
                   cold_sz = H.n * (uint64_t)H.dim * 4;
    if (H.sig_off < kHeaderBytes || H.adj_off <= H.sig_off || H.cold_off <= H.adj_off) {
        set_error("load_index: offsets not strictly increasing");
        return QVG_RUNTIME_ERROR;
    }
    if (H.adj_off - H.sig_off != sig_sz || H.cold_off - H.adj_off != adj_sz) {
        set_error("load_index: segment lengths inconsistent with header");
        return QVG_RUNTIME_ERROR;
    }
    if (file_size != H.cold_off + cold_sz) {
        set_error("load_index: truncated or oversized file");
        return QVG_RUNTIME_ERROR;
    }
    if (H.entry >= H.n) {
        set_error("load_index: entry point out of range");
        return QVG_RUNTIME_ERROR;
    }
    qvg_status st = check_geometry(H.n, H.dim, 2 * H.m, (uint32_t)H.entry);
    if (st != QVG_OK) return st;
    std::vector<uint64_t> codes(H.n * 2 * W);
    std::vector<uint32_t> adj(H.n * (2ull * H.m + 1));
    if (!read_at(f.get(), H.sig_off, codes.data(), sig_sz) ||
        !read_at(f.get(), H.adj_off, adj.data(), adj_sz)) {
        set_error("load_index: hot segment read failed");
        return QVG_RUNTIME_ERROR;
    }
    qvg_index* h = nullptr;
    st = alloc_handle(device, H.n, H.dim, 2 * H.m, (uint32_t)H.entry, &h);
    if (st != QVG_OK) return st;
    h->m = H.m;
    h->alpha = (float)H.alpha_milli / 1000.0f;
    st = upload_hot(h, codes.data(), adj.data());
    if (st != QVG_OK) {
        free_index(h);
        return st;
    }
    codes = {};
    adj = {};
    // cold segment: stream through a pinned staging buffer straight into HBM
    const size_t chunk_rows = std::max<size_t>(1, (64u << 20) / (H.dim * 4ull));
    float* pinned[2] = {nullptr, nullptr};
    cudaError_t e = cudaMallocHost(&pinned[0], chunk_rows * H.dim * 4);
    if (e == cudaSuccess) e = cudaMallocHost(&pinned[1], chunk_rows * H.dim * 4);
    if (e == cudaSuccess && h->ix.Dp != h->ix.dim)
        e = cudaMemsetAsync(h->d_cold, 0, H.n * (size_t)h->ix.Dp * 4, h->stream);
    if (fseeko(f.get(), (off_t)H.cold_off, SEEK_SET) != 0) {
        st = QVG_RUNTIME_ERROR;
        set_error("load_index: cold segment read failed");
    }
    // one event per staging buffer: reading chunk i+1 from the file overlaps the
    // H2D copy of chunk i (waiting on the stream would also wait for the other
    // buffer's copy and serialise file read and upload)
    cudaEvent_t freed[2] = {nullptr, nullptr};
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&freed[0], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&freed[1], cudaEventDisableTiming);
    bool used[2] = {false, false};
    int buf = 0;
    for (uint64_t r0 = 0; e == cudaSuccess && st == QVG_OK && r0 < H.n; r0 += chunk_rows) {
        const uint64_t rows = std::min<uint64_t>(chunk_rows, H.n - r0);
        if (used[buf]) e = cudaEventSynchronize(freed[buf]);  // this buffer's last copy is done
        if (e != cudaSuccess) break;
        if (fread(pinned[buf], 4ull * H.dim, rows, f.get()) != rows) {
            st = QVG_RUNTIME_ERROR;
            set_error("load_index: cold segment read failed");
            break;
        }
        float* dst = static_cast<float*>(h->d_cold) + r0 * h->ix.Dp;
        if (h->ix.Dp == h->ix.dim)
            e = cudaMemcpyAsync(dst, pinned[buf], rows * H.dim * 4, cudaMemcpyHostToDevice,
                                h->stream);
        else
            e = cudaMemcpy2DAsync(dst, h->ix.Dp * 4, pinned[buf], H.dim * 4, H.dim * 4, rows,
                                  cudaMemcpyHostToDevice, h->stream);
        if (e == cudaSuccess) e = cudaEventRecord(freed[buf], h->stream);
        used[buf] = true;
        buf ^= 1;
    }
    const cudaError_t es = cudaStreamSynchronize(h->stream);  // never free a buffer in use
    if (e == cudaSuccess) e = es;
    for (cudaEvent_t ev : freed)
        if (ev) cudaEventDestroy(ev);
    cudaFreeHost(pinned[0]);
    cudaFreeHost(pinned[1]);
    if (e != cudaSuccess) st = cuda_status(e, "load_index: cold upload");
    if (st != QVG_OK) {
        free_index(h);
        return st;
    }
    *out = h;
    return QVG_OK;
}

qvg_status qvg_index_export(const qvg_index* h, uint64_t* codes, uint32_t* adj, float* cold) {
    if (!h) {
        set_error("qvg_index_export: null index");
        return QVG_INVALID_ARGUMENT;
    }
    cudaSetDevice(h->device);
    const DevIndex& ix = h->ix;
    cudaStream_t s = h->stream;
    cudaError_t e = cudaSuccess;
    void* tmp = nullptr;
    const size_t code_bytes = ix.n * 2 * ix.W * 8, adj_bytes = ix.n * (ix.R + 1ull) * 4;
    if (codes || adj) e = cudaMalloc(&tmp, std::max(code_bytes, adj_bytes));
    if (e == cudaSuccess && codes) {
        launch_chunks_to_codes(ix.codes, ix.n, ix.W, static_cast<uint64_t*>(tmp), s);
        e = cudaMemcpyAsync(codes, tmp, code_bytes, cudaMemcpyDefault, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    }
    if (e == cudaSuccess && adj) {
        adj_export_kernel<<<(unsigned)((ix.n + 127) / 128), 128, 0, s>>>(
            ix.adj, ix.n, ix.R, ix.RS, static_cast<uint32_t*>(tmp));
        e = cudaMemcpyAsync(adj, tmp, adj_bytes, cudaMemcpyDefault, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    }
    if (e == cudaSuccess && cold) {
        if (ix.Dp == ix.dim)
            e = cudaMemcpyAsync(cold, ix.cold, ix.n * ix.dim * 4ull, cudaMemcpyDefault, s);
        else
            e = cudaMemcpy2DAsync(cold, ix.dim * 4, ix.cold, ix.Dp * 4, ix.dim * 4, ix.n,
                                  cudaMemcpyDefault, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    }
    cudaFree(tmp);
    return e == cudaSuccess ? QVG_OK : cuda_status(e, "qvg_index_export");
}

qvg_status qvg_index_save(const qvg_index* h, const char* path) {
    if (!h || !path) {
        set_error("qvg_index_save: null argument");
        return QVG_INVALID_ARGUMENT;
    }
    const DevIndex& ix = h->ix;
    if (ix.R % 2 != 0) {
        set_error("save_index: max_degree must be even (2m) for the .qivr format");
        return QVG_INVALID_ARGUMENT;
    }
    const uint64_t W = ix.W;
    std::vector<uint64_t> codes(ix.n * 2 * W);
    std::vector<uint32_t> adj(ix.n * (ix.R + 1ull));
    std::vector<float> cold(ix.n * (uint64_t)ix.dim);
    qvg_status st = qvg_index_export(h, codes.data(), adj.data(), cold.data());
    if (st != QVG_OK) return st;
    uint8_t hb[kHeaderBytes];
    std::memset(hb, 0, sizeof(hb));
    std::memcpy(hb, "QIVR", 4);
    const uint64_t sig_sz = codes.size() * 8, adj_sz = adj.size() * 4;
    put_u32(hb + 4, 1);
    put_u64(hb + 8, ix.n);
    put_u32(hb + 16, ix.dim);
    put_u32(hb + 20, ix.R / 2);
    put_u32(hb + 24, (uint32_t)std::lround(h->alpha * 1000.0f));
    put_u64(hb + 28, ix.entry);
    put_u64(hb + 36, kHeaderBytes);
    put_u64(hb + 44, kHeaderBytes + sig_sz);
    put_u64(hb + 52, kHeaderBytes + sig_sz + adj_sz);
    std::unique_ptr<FILE, FileCloser> f(fopen(path, "wb"));
    if (!f) {
        set_error(std::string("save_index: cannot open ") + path);
        return QVG_RUNTIME_ERROR;
    }
    bool ok = fwrite(hb, 1, kHeaderBytes, f.get()) == kHeaderBytes &&
              fwrite(codes.data(), 1, sig_sz, f.get()) == sig_sz &&
              fwrite(adj.data(), 1, adj_sz, f.get()) == adj_sz &&
              fwrite(cold.data(), 4, cold.size(), f.get()) == cold.size();
    if (!ok) {
        set_error(std::string("save_index: write failed for ") + path);
        return QVG_RUNTIME_ERROR;
    }
    return QVG_OK;
}

void qvg_index_destroy(qvg_index* h) { free_index(h); }

qvg_status qvg_index_info(const qvg_index* h, uint64_t* n, uint32_t* dim, uint32_t* max_degree,
                          uint32_t* entry_point) {
    if (!h) {
        set_error("qvg_index_info: null index");
        return QVG_INVALID_ARGUMENT;
    }
    if (n) *n = h->ix.n;
    if (dim) *dim = h->ix.dim;
    if (max_degree) *max_degree = h->ix.R;
    if (entry_point) *entry_point = h->ix.entry;
    return QVG_OK;
}

qvg_status qvg_index_set_stream(qvg_index* h, void* stream) {
    if (!h) {
        set_error("qvg_index_set_stream: null index");
        return QVG_INVALID_ARGUMENT;
    }
    h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own_stream;
    return QVG_OK;
}

}  // extern "C"

namespace qvg {
// used by the builder to wrap device-resident stores into a handle
qvg_status make_handle_from_device(int device, uint64_t n, uint32_t dim, uint32_t R,
                                   uint32_t entry, qvg_index** out) {
    return alloc_handle(device, n, dim, R, entry, out);
}
void destroy_handle(qvg_index* h) { free_index(h); }
}  // namespace qvg

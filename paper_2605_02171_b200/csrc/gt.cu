// Exact brute-force top-k, encoding diagnostics and the compatibility probe
// (SURVEY §8(f) rows 2 and 4).
//
// Reference behaviour reproduced (paths under /root/reference/proj/core):
//   brute_force_topk      eval.cpp:81-168   per query, every base row scored;
//                                           float scores rank descending, code
//                                           distances ascending, ties by id asc;
//                                           exclude_identity skips row j == qi
//   dot_f32               vec_math.hpp:13-26 4 double chains (i mod 4) over
//                                           4*floor(D/4), tail into chain 0,
//                                           (s0+s1)+(s2+s3) rounded to float
//   encode_sm2_into       encoding.cpp:32-45 raw (unnormalised) 2-bit code,
//                                           tau = float(sum|x| / D) (:23-30)
//   encode_sign1          encoding.cpp:60-72 sign bit == the sm2 pos bit
//   encode_sq2            encoding.cpp:74-106, sq2_distance_bytes encoding.hpp:203-210
//   compatibility_probe   eval.cpp:196-222
//   strong_bit_rate       encoding.cpp:132-167
//
// B200 design.  float_cosine: the reference's own arithmetic on every pair —
// B200 runs FP64 FMA at half the FP32 rate, so the exact 4-chain double dot
// over all N x nq pairs costs less than a screen-then-rescore scheme and
// leaves nothing to a margin argument.  A block owns 8 queries (one warp each
// for selection) and a range of base rows; each thread scores one row of a
// 256-row tile against the 8 queries from a K-chunk staged in shared memory
// as doubles (rows transposed so a warp's loads are contiguous, query values
// read as broadcasts).  Each warp keeps its query's best k keys (sorted, in
// shared memory); a tile's keys that beat the current k-th are appended and
// the list re-sorted (warp bitonic sort), which is rare after the first
// tiles.  Row ranges are split over gridDim.y and the per-split lists merged.
// sm2 / sign1 / sq2: the same selection over integer distances of raw codes.
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "bq_device.cuh"
#include "qvg_internal.cuh"

namespace qvg {

namespace {

constexpr uint64_t kNoKey = ~0ull;
constexpr unsigned kAll = 0xFFFFFFFFu;
constexpr int kQ = 8;          // queries per block (one warp each)
constexpr int kRowsT = 256;    // rows per tile (one per thread)
constexpr int kKC = 16;        // elements per K chunk
constexpr uint32_t kMaxK = 256;

// ascending key == (score desc, id asc); -0.0 folds onto +0.0 (the reference
// compares with `>`, under which they tie)
__device__ __forceinline__ uint64_t score_key(float s, uint32_t id) {
    uint32_t u = __float_as_uint(s);
    if ((u & 0x7fffffffu) == 0) u = 0;
    const uint32_t ord = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((uint64_t)(~ord) << 32) | id;
}
__device__ __forceinline__ float key_score(uint64_t key) {
    const uint32_t ord = ~(uint32_t)(key >> 32);
    const uint32_t u = (ord & 0x80000000u) ? (ord & 0x7fffffffu) : ~ord;
    return __uint_as_float(u);
}

// warp bitonic sort (ascending) of a[0, N), N a power of two <= 512
__device__ void warp_sort(uint64_t* a, uint32_t N, uint32_t lane) {
    for (uint32_t size = 2; size <= N; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = lane; t < N / 2; t += 32) {
                const uint32_t i = 2 * t - (t & (stride - 1));
                const uint32_t j = i + stride;
                const bool asc = (i & size) == 0;
                const uint64_t x = a[i], y = a[j];
                if ((x > y) == asc) {
                    a[i] = y;
                    a[j] = x;
                }
            }
            __syncwarp();
        }
    }
}

__device__ __forceinline__ uint32_t pow2_at_least(uint32_t x) {
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

// merge the keys of one tile (tile[0, cnt)) into the sorted best-k list L
// (length ln, room for k + cnt): append the ones below the current k-th, sort
__device__ void offer_tile(uint64_t* L, uint32_t& ln, uint32_t k, const uint64_t* tile,
                           uint32_t cnt, uint32_t lane) {
    const uint64_t thr = ln == k ? L[k - 1] : kNoKey;
    uint32_t m = 0;
    for (uint32_t c = 0; c < cnt; c += 32) {
        const uint64_t key = c + lane < cnt ? tile[c + lane] : kNoKey;
        const bool pass = key < thr;
        const unsigned b = __ballot_sync(kAll, pass);
        if (pass) L[ln + m + __popc(b & ((1u << lane) - 1u))] = key;
        m += __popc(b);
    }
    if (m == 0) return;
    __syncwarp();
    const uint32_t tot = ln + m;
    const uint32_t N = pow2_at_least(tot);
    for (uint32_t i = tot + lane; i < N; i += 32) L[i] = kNoKey;
    __syncwarp();
    warp_sort(L, N, lane);
    ln = tot < k ? tot : k;
}

struct TopkArgs {
    const float* base;     // float scorer: n x dim
    const float* queries;  // float scorer: nq x dim
    const uint4* bcodes;   // code scorers: n x W chunks
    const uint4* qcodes;   // code scorers: nq x W chunks
    const uint4* bsq;      // sq2: n x Dq bytes (zero padded)
    const uint4* qsq;      // sq2: nq x Dq bytes
    uint64_t n, nq, rows_per_split;
    uint32_t dim, W, Dq, k, S;
    int exclude_identity;
    int scorer;            // 0 float_cosine, 1 sm2, 2 sign1, 3 sq2
    uint64_t* part;        // nq x S x k keys
};

// shared memory: lists [kQ][2 * kMaxK] keys, tile keys [kQ][kRowsT], then the
// scorer's staging (float: rows [kKC][kRowsT] + queries [kKC][kQ] doubles;
// codes: query chunks [kQ][W])
constexpr size_t kListBytes = (size_t)kQ * 2 * kMaxK * 8;
constexpr size_t kTileBytes = (size_t)kQ * kRowsT * 8;

__global__ void __launch_bounds__(256) topk_kernel(const TopkArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint64_t* lists = reinterpret_cast<uint64_t*>(sm);
    uint64_t* tkeys = reinterpret_cast<uint64_t*>(sm + kListBytes);
    unsigned char* stage = sm + kListBytes + kTileBytes;
    const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint64_t q0 = (uint64_t)blockIdx.x * kQ;
    const uint32_t split = blockIdx.y;
    const uint64_t r_beg = (uint64_t)split * a.rows_per_split;
    const uint64_t r_end = min(a.n, r_beg + a.rows_per_split);
    uint64_t* L = lists + (size_t)w * 2 * kMaxK;
    uint32_t ln = 0;

    if (a.scorer == 1 || a.scorer == 2) {  // stage the block's query codes once
        uint4* qc = reinterpret_cast<uint4*>(stage);
        for (uint32_t i = tid; i < kQ * a.W; i += blockDim.x) {
            const uint32_t q = i / a.W, c = i % a.W;
            qc[i] = q0 + q < a.nq ? a.qcodes[(q0 + q) * a.W + c] : make_uint4(0, 0, 0, 0);
        }
        __syncthreads();
    } else if (a.scorer == 3) {
        uint4* qs = reinterpret_cast<uint4*>(stage);
        const uint32_t V = a.Dq / 16;
        for (uint32_t i = tid; i < kQ * V; i += blockDim.x) {
            const uint32_t q = i / V, c = i % V;
            qs[i] = q0 + q < a.nq ? a.qsq[(q0 + q) * V + c] : make_uint4(0, 0, 0, 0);
        }
        __syncthreads();
    }

    for (uint64_t t0 = r_beg; t0 < r_end; t0 += kRowsT) {
        const uint64_t row = t0 + tid;
        const bool rv = row < r_end;
        uint64_t key[kQ];
        if (a.scorer == 0) {
            double* rowt = reinterpret_cast<double*>(stage);       // [kKC][kRowsT]
            double* qt = rowt + kKC * kRowsT;                       // [kKC][kQ]
            double acc[kQ][4];
#pragma unroll
            for (int q = 0; q < kQ; ++q)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[q][c] = 0.0;
            const uint32_t main4 = a.dim & ~3u;
            // the next K chunk of this thread's row is loaded into registers
            // while the current one is being consumed (vector loads when rows
            // are 16-B aligned)
            const bool vec = (a.dim & 3u) == 0 && ((uintptr_t)a.base & 15u) == 0;
            float nx[kKC];
            auto load_chunk = [&](uint32_t kc) {
                const float* src = a.base + row * a.dim + kc;
                if (vec && rv && kc + kKC <= a.dim) {
#pragma unroll
                    for (int v = 0; v < kKC / 4; ++v) {
                        const float4 f = __ldg(reinterpret_cast<const float4*>(src) + v);
                        nx[4 * v] = f.x;
                        nx[4 * v + 1] = f.y;
                        nx[4 * v + 2] = f.z;
                        nx[4 * v + 3] = f.w;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < kKC; ++e)
                        nx[e] = (rv && kc + e < a.dim) ? __ldg(src + e) : 0.0f;
                }
            };
            load_chunk(0);
            for (uint32_t kc = 0; kc < a.dim; kc += kKC) {
                __syncthreads();
#pragma unroll
                for (int e = 0; e < kKC; ++e) rowt[e * kRowsT + tid] = (double)nx[e];
                if (tid < kQ * kKC) {
                    const uint32_t q = tid / kKC, e = tid % kKC;
                    qt[e * kQ + q] = (q0 + q < a.nq && kc + e < a.dim)
                                         ? (double)__ldg(a.queries + (q0 + q) * a.dim + kc + e)
                                         : 0.0;
                }
                __syncthreads();
                if (kc + kKC < a.dim) load_chunk(kc + kKC);
                const uint32_t lim = min((uint32_t)kKC, a.dim - kc);
                for (uint32_t e4 = 0; e4 < lim; e4 += 4) {
                    const uint32_t i = kc + e4;
                    if (i + 4 <= main4) {
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const double x = rowt[(e4 + c) * kRowsT + tid];
                            const double2* qq = reinterpret_cast<const double2*>(qt + (e4 + c) * kQ);
#pragma unroll
                            for (int h = 0; h < kQ / 2; ++h) {
                                const double2 v = qq[h];
                                acc[2 * h][c] = __fma_rn(v.x, x, acc[2 * h][c]);
                                acc[2 * h + 1][c] = __fma_rn(v.y, x, acc[2 * h + 1][c]);
                            }
                        }
                    } else {  // tail elements >= 4*floor(D/4) all go to chain 0
                        for (uint32_t c = 0; c < 4 && i + c < a.dim; ++c) {
                            const double x = rowt[(e4 + c) * kRowsT + tid];
#pragma unroll
                            for (int q = 0; q < kQ; ++q)
                                acc[q][0] = __fma_rn(qt[(e4 + c) * kQ + q], x, acc[q][0]);
                        }
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                const float s = __double2float_rn(
                    __dadd_rn(__dadd_rn(acc[q][0], acc[q][1]), __dadd_rn(acc[q][2], acc[q][3])));
                key[q] = score_key(s, (uint32_t)row);
            }
        } else if (a.scorer == 3) {  // sq2_distance_bytes: sum |a_i - b_i|
            const uint4* qs = reinterpret_cast<const uint4*>(stage);
            const uint32_t V = a.Dq / 16;
            uint32_t d[kQ];
#pragma unroll
            for (int q = 0; q < kQ; ++q) d[q] = 0;
            if (rv) {
                const uint4* rc = a.bsq + row * V;
                for (uint32_t c = 0; c < V; ++c) {
                    const uint4 v = __ldg(rc + c);
#pragma unroll
                    for (int q = 0; q < kQ; ++q) {
                        const uint4 u = qs[q * V + c];
                        uint32_t s = d[q];
                        s = __dp4a(__vabsdiffu4(u.x, v.x), 0x01010101u, s);
                        s = __dp4a(__vabsdiffu4(u.y, v.y), 0x01010101u, s);
                        s = __dp4a(__vabsdiffu4(u.z, v.z), 0x01010101u, s);
                        d[q] = __dp4a(__vabsdiffu4(u.w, v.w), 0x01010101u, s);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < kQ; ++q) key[q] = ((uint64_t)d[q] << 32) | (uint32_t)row;
        } else {
            const uint4* qc = reinterpret_cast<const uint4*>(stage);
            uint32_t d[kQ];
#pragma unroll
            for (int q = 0; q < kQ; ++q) d[q] = 0;
            if (rv) {
                const uint4* rc = a.bcodes + row * a.W;
                for (uint32_t c = 0; c < a.W; ++c) {
                    const uint4 v = __ldg(rc + c);
#pragma unroll
                    for (int q = 0; q < kQ; ++q) {
                        const uint4 u = qc[q * a.W + c];
                        d[q] += a.scorer == 1 ? dev::sm2_chunk(u, v)
                                              : (uint32_t)(__popc(u.x ^ v.x) + __popc(u.y ^ v.y));
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < kQ; ++q) key[q] = ((uint64_t)d[q] << 32) | (uint32_t)row;
        }
        __syncthreads();  // previous tile's keys consumed
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            const bool excl = a.exclude_identity && row == q0 + q;
            tkeys[q * kRowsT + tid] = (rv && !excl && q0 + q < a.nq) ? key[q] : kNoKey;
        }
        __syncthreads();
        offer_tile(L, ln, a.k, tkeys + w * kRowsT, kRowsT, lane);
    }
    const uint64_t q = q0 + w;
    if (q < a.nq) {
        uint64_t* out = a.part + (q * a.S + split) * a.k;
        for (uint32_t i = lane; i < a.k; i += 32) out[i] = i < ln ? L[i] : kNoKey;
    }
}

// one warp per query: merge the S per-split lists, emit ids / values
__global__ void merge_kernel(const uint64_t* __restrict__ part, uint64_t nq, uint32_t S,
                             uint32_t k, int scorer, uint32_t* __restrict__ out_ids,
                             float* __restrict__ out_scores, uint32_t* __restrict__ out_dists,
                             uint32_t* __restrict__ out_count) {
    extern __shared__ __align__(16) uint64_t L2[];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t q = (uint64_t)blockIdx.x * (blockDim.x / 32) + w;
    if (q >= nq) return;
    uint64_t* L = L2 + (size_t)w * 2 * kMaxK;
    uint32_t ln = 0;
    for (uint32_t s = 0; s < S; ++s) {
        const uint64_t* src = part + (q * S + s) * k;
        uint32_t cnt = 0;  // lists are sorted with kNoKey padding
        for (uint32_t i = lane; i < k; i += 32) L[ln + i] = src[i];
        __syncwarp();
        for (uint32_t c = 0; c < k; c += 32) {
            const bool v = c + lane < k && L[ln + c + lane] != kNoKey;
            cnt += __popc(__ballot_sync(kAll, v));
        }
        if (s == 0) {
            ln = cnt;
            continue;
        }
        const uint32_t tot = ln + cnt;
        const uint32_t N = pow2_at_least(tot);
        for (uint32_t i = tot + lane; i < N; i += 32) L[i] = kNoKey;
        __syncwarp();
        warp_sort(L, N, lane);
        ln = tot < k ? tot : k;
    }
    for (uint32_t i = lane; i < k; i += 32) {
        const bool v = i < ln;
        const uint64_t key = v ? L[i] : kNoKey;
        out_ids[q * k + i] = v ? (uint32_t)key : 0xFFFFFFFFu;
        if (out_scores) out_scores[q * k + i] = v && scorer == 0 ? key_score(key) : __int_as_float(0x7fc00000);
        if (out_dists) out_dists[q * k + i] = v && scorer != 0 ? (uint32_t)(key >> 32) : 0xFFFFFFFFu;
    }
    if (lane == 0 && out_count) out_count[q] = ln;
}

// raw code (encode_sm2_into, encoding.cpp:32-45): warp per row, lane 0 runs
// the index-ordered double sum of |x| (compute_threshold, encoding.cpp:23-30)
__global__ void __launch_bounds__(256) encode_raw_kernel(const float* __restrict__ x,
                                                         uint64_t rows, uint32_t dim,
                                                         uint4* __restrict__ codes,
                                                         uint32_t* __restrict__ bad,
                                                         float* __restrict__ tau_out) {
    extern __shared__ __align__(16) float rbuf[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t r = (uint64_t)blockIdx.x * 8 + wib;
    if (r >= rows) return;
    float* row = rbuf + (size_t)wib * dim;
    const float* src = x + r * dim;
    bool fin = true;
    for (uint32_t i = lane; i < dim; i += 32) {
        const float v = __ldg(src + i);
        fin &= isfinite(v);
        row[i] = v;
    }
    fin = __all_sync(kAll, fin);
    __syncwarp();
    float tau_l = 0.0f;
    if (lane == 0 && fin) {
        double s = 0.0;
        for (uint32_t i = 0; i < dim; ++i) s = __dadd_rn(s, fabs((double)row[i]));
        tau_l = __double2float_rn(__ddiv_rn(s, (double)dim));
    }
    const float tau = __shfl_sync(kAll, tau_l, 0);
    const uint32_t W = (dim + 63) / 64;
    for (uint32_t wd = lane; wd < W; wd += 32) {
        uint32_t p0 = 0, p1 = 0, s0 = 0, s1 = 0;
        const uint32_t b0 = wd * 64, lim = min(64u, dim - b0);
        for (uint32_t b = 0; b < lim; ++b) {
            const float y = row[b0 + b];
            const uint32_t pb = y > 0.0f, sb = fabsf(y) > tau;
            if (b < 32) {
                p0 |= pb << b;
                s0 |= sb << b;
            } else {
                p1 |= pb << (b - 32);
                s1 |= sb << (b - 32);
            }
        }
        codes[r * W + wd] = make_uint4(p0, p1, s0, s1);
    }
    if (lane == 0 && !fin) atomicOr(bad, 1u);
    if (lane == 0 && tau_out) tau_out[r] = tau;
}

// encode_sq2 (encoding.cpp:74-106): warp per row; lane 0 runs the two
// index-ordered double reductions.  The reference's C++ build (gnu++20, -O3,
// FMA-capable -march) contracts `var += (v - mean) * (v - mean)` into an FMA,
// so the chain is fma(d, d, var).  Bucket b = int((v - lo) / width) in float
// with x86 truncation semantics (out-of-range / NaN -> INT_MIN), clamped to
// [0, 3]; a zero-spread row is all zeros.
__global__ void __launch_bounds__(256) encode_sq2_kernel(const float* __restrict__ x,
                                                         uint64_t rows, uint32_t dim,
                                                         uint32_t Dq, uint8_t* __restrict__ codes,
                                                         uint32_t* __restrict__ bad) {
    extern __shared__ __align__(16) float sbuf[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t r = (uint64_t)blockIdx.x * 8 + wib;
    if (r >= rows) return;
    float* row = sbuf + (size_t)wib * dim;
    const float* src = x + r * dim;
    bool fin = true;
    for (uint32_t i = lane; i < dim; i += 32) {
        const float v = __ldg(src + i);
        fin &= isfinite(v);
        row[i] = v;
    }
    fin = __all_sync(kAll, fin);
    __syncwarp();
    float lo_l = 0.0f, width_l = 0.0f;
    int ok_l = 0;
    if (lane == 0 && fin) {
        double mean = 0.0;
        for (uint32_t i = 0; i < dim; ++i) mean = __dadd_rn(mean, (double)row[i]);
        mean = __ddiv_rn(mean, (double)dim);
        double var = 0.0;
        for (uint32_t i = 0; i < dim; ++i) {
            const double d = __dsub_rn((double)row[i], mean);
            var = __fma_rn(d, d, var);
        }
        const double sd = __dsqrt_rn(__ddiv_rn(var, (double)dim));
        if (sd > 0.0) {
            ok_l = 1;
            lo_l = __double2float_rn(__dsub_rn(mean, __dmul_rn(2.0, sd)));
            width_l = __double2float_rn(sd);
        }
    }
    const int ok = __shfl_sync(kAll, ok_l, 0);
    const float lo = __shfl_sync(kAll, lo_l, 0), width = __shfl_sync(kAll, width_l, 0);
    uint8_t* out = codes + r * Dq;
    for (uint32_t i = lane; i < Dq; i += 32) {
        int b = 0;
        if (ok && i < dim) {
            const float t = __fdiv_rn(__fsub_rn(row[i], lo), width);
            b = (t >= -2147483648.0f && t < 2147483648.0f) ? (int)t : INT_MIN;
            b = b < 0 ? 0 : (b > 3 ? 3 : b);
        }
        out[i] = (uint8_t)b;
    }
    if (lane == 0 && !fin) atomicOr(bad, 1u);
}

// sum of popcounts of the strong words (chunk .z/.w) of `rows` code rows
__global__ void strong_count_kernel(const uint4* __restrict__ codes, uint64_t total_chunks,
                                    unsigned long long* __restrict__ out) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total_chunks;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldg(codes + i);
        c += __popc(v.z) + __popc(v.w);
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kAll, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// any of rows 1..n-1 differs from row 0 (bitwise, memcmp semantics)
__global__ void rows_differ_kernel(const float* __restrict__ x, uint64_t n, uint32_t dim,
                                   uint32_t* __restrict__ flag) {
    const uint32_t* u = reinterpret_cast<const uint32_t*>(x);
    const uint64_t total = n * dim;
    for (uint64_t i = dim + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (u[i] != u[i % dim]) {
            *flag = 1u;
            return;
        }
}

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    bool alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 16) == cudaSuccess; }
};

// device view of a user buffer: device pointers are used in place, host
// buffers are copied in
qvg_status device_view(const float* src, size_t elems, DevBuf& buf, const float** out,
                       cudaStream_t s) {
    if (is_device_ptr(src)) {
        *out = src;
        return QVG_OK;
    }
    if (!buf.alloc(elems * 4)) return cuda_status(cudaErrorMemoryAllocation, "brute_force_topk");
    cudaError_t e = cudaMemcpyAsync(buf.p, src, elems * 4, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "H2D(brute_force_topk)");
    *out = static_cast<const float*>(buf.p);
    return QVG_OK;
}

qvg_status encode_raw(const float* x, uint64_t rows, uint32_t dim, uint4* codes, uint32_t* d_bad,
                      cudaStream_t s, float* tau = nullptr) {
    if (!rows) return QVG_OK;
    const size_t smem = 8ull * dim * 4;
    if (smem > 200 * 1024) {
        set_error("encode: dim too large for the row encoders");
        return QVG_NOT_IMPLEMENTED;
    }
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(encode_raw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    encode_raw_kernel<<<(unsigned)((rows + 7) / 8), 256, smem, s>>>(x, rows, dim, codes, d_bad,
                                                                      tau);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QVG_OK : cuda_status(e, "encode_raw");
}

qvg_status topk_device(int device, const float* d_base, uint64_t n, const float* d_q, uint64_t nq,
                       uint32_t dim, uint32_t k, int scorer, int exclude_identity,
                       uint32_t* d_ids, float* d_scores, uint32_t* d_dists, uint32_t* d_count,
                       cudaStream_t s) {
    qvg_status st;
    const uint32_t W = (dim + 63) / 64;
    DevBuf bcodes, qcodes, bad, part;
    TopkArgs a{};
    a.base = d_base;
    a.queries = d_q;
    a.n = n;
    a.nq = nq;
    a.dim = dim;
    a.W = W;
    a.k = k;
    a.exclude_identity = exclude_identity;
    a.scorer = scorer;
    a.Dq = (dim + 15) & ~15u;
    DevBuf bsq, qsq;
    if (scorer == 3) {
        const size_t esmem = 8ull * dim * 4;
        if (esmem > 200 * 1024 || (size_t)kQ * a.Dq > 96 * 1024) {
            set_error("brute_force_topk: dim too large for the sq2 scorer");
            return QVG_NOT_IMPLEMENTED;
        }
        if (!bsq.alloc(n * (size_t)a.Dq) || !qsq.alloc(nq * (size_t)a.Dq) || !bad.alloc(4))
            return cuda_status(cudaErrorMemoryAllocation, "brute_force_topk");
        cudaMemsetAsync(bad.p, 0, 4, s);
        if (esmem > 48 * 1024)
            cudaFuncSetAttribute(encode_sq2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)esmem);
        encode_sq2_kernel<<<(unsigned)((n + 7) / 8), 256, esmem, s>>>(
            d_base, n, dim, a.Dq, static_cast<uint8_t*>(bsq.p), static_cast<uint32_t*>(bad.p));
        encode_sq2_kernel<<<(unsigned)((nq + 7) / 8), 256, esmem, s>>>(
            d_q, nq, dim, a.Dq, static_cast<uint8_t*>(qsq.p), static_cast<uint32_t*>(bad.p));
        uint32_t hbad = 0;
        cudaError_t e = cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_status(e, "encode_sq2");
        if (hbad) {
            set_error("encode: non-finite coordinate");
            return QVG_INVALID_ARGUMENT;
        }
        a.bsq = static_cast<const uint4*>(bsq.p);
        a.qsq = static_cast<const uint4*>(qsq.p);
    } else if (scorer != 0) {
        if (!bcodes.alloc(n * W * 16ull) || !qcodes.alloc(nq * W * 16ull) || !bad.alloc(4))
            return cuda_status(cudaErrorMemoryAllocation, "brute_force_topk");
        cudaMemsetAsync(bad.p, 0, 4, s);
        if ((st = encode_raw(d_base, n, dim, static_cast<uint4*>(bcodes.p),
                             static_cast<uint32_t*>(bad.p), s)) != QVG_OK)
            return st;
        if ((st = encode_raw(d_q, nq, dim, static_cast<uint4*>(qcodes.p),
                             static_cast<uint32_t*>(bad.p), s)) != QVG_OK)
            return st;
        uint32_t hbad = 0;
        cudaError_t e = cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_status(e, "encode_raw");
        if (hbad) {
            set_error("encode: non-finite coordinate");
            return QVG_INVALID_ARGUMENT;
        }
        a.bcodes = static_cast<const uint4*>(bcodes.p);
        a.qcodes = static_cast<const uint4*>(qcodes.p);
    }
    // split the rows so that the grid fills the GPU about twice
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const uint64_t qblocks = (nq + kQ - 1) / kQ;
    uint64_t S = (2ull * sms + qblocks - 1) / qblocks;
    const uint64_t max_s = (n + kRowsT - 1) / kRowsT;
    if (S > max_s) S = max_s;
    if (S > 256) S = 256;
    if (S < 1) S = 1;
    a.S = (uint32_t)S;
    a.rows_per_split = ((n + S - 1) / S + kRowsT - 1) / kRowsT * kRowsT;
    if (!part.alloc(nq * S * k * 8ull)) return cuda_status(cudaErrorMemoryAllocation, "brute_force_topk");
    a.part = static_cast<uint64_t*>(part.p);
    const size_t stage = scorer == 0   ? (size_t)kKC * (kRowsT + kQ) * 8
                         : scorer == 3 ? (size_t)kQ * a.Dq
                                       : (size_t)kQ * W * 16;
    const size_t smem = kListBytes + kTileBytes + stage;
    cudaError_t e = cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "brute_force_topk: smem");
    topk_kernel<<<dim3((unsigned)qblocks, (unsigned)S), 256, smem, s>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_status(e, "launch(topk)");
    const size_t msmem = 8ull * 2 * kMaxK * 8;  // 8 warps per block
    cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msmem);
    merge_kernel<<<(unsigned)((nq + 7) / 8), 256, msmem, s>>>(a.part, nq, a.S, k, scorer, d_ids,
                                                              d_scores, d_dists, d_count);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_status(e, "launch(topk merge)");
    e = cudaStreamSynchronize(s);  // part / code buffers are freed on return
    return e == cudaSuccess ? QVG_OK : cuda_status(e, "brute_force_topk");
}

// device output buffer bound to a user pointer (device: in place; host: copied back)
struct OutBuf {
    void* user = nullptr;
    DevBuf own;
    void* dev = nullptr;
    size_t bytes = 0;
    qvg_status bind(void* u, size_t b) {
        user = u;
        bytes = b;
        if (!u) return QVG_OK;
        if (is_device_ptr(u)) {
            dev = u;
            return QVG_OK;
        }
        if (!own.alloc(b)) return cuda_status(cudaErrorMemoryAllocation, "brute_force_topk");
        dev = own.p;
        return QVG_OK;
    }
    qvg_status back() {
        if (!user || dev == user) return QVG_OK;
        cudaError_t e = cudaMemcpy(user, dev, bytes, cudaMemcpyDeviceToHost);
        return e == cudaSuccess ? QVG_OK : cuda_status(e, "D2H(brute_force_topk)");
    }
};

}  // namespace

}  // namespace qvg

using namespace qvg;

extern "C" {

qvg_status qvg_brute_force_topk(int device, const float* base, uint64_t n, const float* queries,
                                uint64_t nq, uint32_t dim, uint32_t k, int scorer,
                                int exclude_identity, uint32_t* out_ids, float* out_scores,
                                uint32_t* out_dists, uint32_t* out_count) {
    if (dim == 0 || k == 0) {
        set_error("brute_force_topk: dim and k must be >= 1");
        return QVG_INVALID_ARGUMENT;
    }
    if (scorer < 0 || scorer > 3) {
        set_error("brute_force_topk: unknown scorer");
        return QVG_INVALID_ARGUMENT;
    }
    if (k > kMaxK) {
        set_error("brute_force_topk: k > 256 is not supported");
        return QVG_NOT_IMPLEMENTED;
    }
    if (nq == 0) return QVG_OK;
    if (!out_ids || (n > 0 && (!base || !queries))) {
        set_error("brute_force_topk: null buffer");
        return QVG_INVALID_ARGUMENT;
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
    if (n == 0) {  // nothing to rank
        std::vector<uint32_t> ids(nq * k, 0xFFFFFFFFu);
        if (is_device_ptr(out_ids)) cudaMemcpy(out_ids, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice);
        else std::memcpy(out_ids, ids.data(), ids.size() * 4);
        if (out_count) {
            if (is_device_ptr(out_count)) cudaMemset(out_count, 0, nq * 4);
            else std::memset(out_count, 0, nq * 4);
        }
        return QVG_OK;
    }
    cudaStream_t s = nullptr;
    qvg_status st;
    DevBuf bb, qb;
    const float *d_base = nullptr, *d_q = nullptr;
    if ((st = device_view(base, n * (size_t)dim, bb, &d_base, s)) != QVG_OK) return st;
    if ((st = device_view(queries, nq * (size_t)dim, qb, &d_q, s)) != QVG_OK) return st;
    OutBuf oi, os, od, oc;
    if ((st = oi.bind(out_ids, nq * k * 4ull)) != QVG_OK) return st;
    if ((st = os.bind(scorer == 0 ? out_scores : nullptr, nq * k * 4ull)) != QVG_OK) return st;
    if ((st = od.bind(scorer != 0 ? out_dists : nullptr, nq * k * 4ull)) != QVG_OK) return st;
    if ((st = oc.bind(out_count, nq * 4ull)) != QVG_OK) return st;
    if ((st = topk_device(device, d_base, n, d_q, nq, dim, k, scorer, exclude_identity,
                          static_cast<uint32_t*>(oi.dev), static_cast<float*>(os.dev),
                          static_cast<uint32_t*>(od.dev), static_cast<uint32_t*>(oc.dev), s)) !=
        QVG_OK)
        return st;
    if ((st = oi.back()) != QVG_OK || (st = os.back()) != QVG_OK || (st = od.back()) != QVG_OK ||
        (st = oc.back()) != QVG_OK)
        return st;
    return QVG_OK;
}

qvg_status qvg_encode_rows(int device, const float* x, uint64_t n, uint32_t dim, int scorer,
                           void* out_codes, float* out_tau) {
    if (dim == 0) {
        set_error("encode: empty vector");
        return QVG_INVALID_ARGUMENT;
    }
    if (scorer < 1 || scorer > 3) {
        set_error("encode_rows: scorer must be sm2, sign1 or sq2");
        return QVG_INVALID_ARGUMENT;
    }
    if (n == 0) return QVG_OK;
    if (!x || !out_codes) {
        set_error("encode_rows: null buffer");
        return QVG_INVALID_ARGUMENT;
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
    qvg_status st;
    DevBuf xb, tmp, bad;
    const float* d = nullptr;
    if ((st = device_view(x, n * (size_t)dim, xb, &d, nullptr)) != QVG_OK) return st;
    if (!bad.alloc(4)) return cuda_status(cudaErrorMemoryAllocation, "encode_rows");
    cudaMemset(bad.p, 0, 4);
    const uint32_t W = (dim + 63) / 64;
    const size_t out_bytes = scorer == 3 ? n * (size_t)dim : n * (size_t)W * 8 * (scorer == 1 ? 2 : 1);
    OutBuf oc, ot;
    if ((st = oc.bind(out_codes, out_bytes)) != QVG_OK) return st;
    if ((st = ot.bind(scorer == 1 ? out_tau : nullptr, n * 4ull)) != QVG_OK) return st;
    if (scorer == 3) {
        const size_t esmem = 8ull * dim * 4;
        if (esmem > 200 * 1024) {
            set_error("encode: dim too large for the row encoders");
            return QVG_NOT_IMPLEMENTED;
        }
        if (esmem > 48 * 1024)
            cudaFuncSetAttribute(encode_sq2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)esmem);
        encode_sq2_kernel<<<(unsigned)((n + 7) / 8), 256, esmem>>>(
            d, n, dim, dim, static_cast<uint8_t*>(oc.dev), static_cast<uint32_t*>(bad.p));
    } else {
        DevBuf chunks, words;
        if (!chunks.alloc(n * W * 16ull) || !words.alloc(n * W * 16ull))
            return cuda_status(cudaErrorMemoryAllocation, "encode_rows");
        if ((st = encode_raw(d, n, dim, static_cast<uint4*>(chunks.p), static_cast<uint32_t*>(bad.p),
                             nullptr, static_cast<float*>(ot.dev))) != QVG_OK)
            return st;
        // reference layout per row: W pos words then W strong words; sign1
        // keeps the pos words (the sign bit is the sm2 pos bit)
        launch_chunks_to_codes(static_cast<const uint4*>(chunks.p), n, W,
                               static_cast<uint64_t*>(words.p), nullptr);
        if (scorer == 1)
            e = cudaMemcpy(oc.dev, words.p, n * W * 16ull, cudaMemcpyDeviceToDevice);
        else
            e = cudaMemcpy2D(oc.dev, W * 8, words.p, W * 16, W * 8, n, cudaMemcpyDeviceToDevice);
        if (e != cudaSuccess) return cuda_status(e, "encode_rows");
    }
    uint32_t hbad = 0;
    if ((e = cudaMemcpy(&hbad, bad.p, 4, cudaMemcpyDeviceToHost)) != cudaSuccess)
        return cuda_status(e, "encode_rows");
    if (hbad) {
        set_error("encode: non-finite coordinate");
        return QVG_INVALID_ARGUMENT;
    }
    if ((st = oc.back()) != QVG_OK || (st = ot.back()) != QVG_OK) return st;
    return QVG_OK;
}

qvg_status qvg_compatibility_probe(int device, const float* data, uint64_t n, uint32_t dim,
                                   uint64_t sample_size, uint32_t k, int scorer,
                                   qvg_probe_report* out) {
    if (!out || !data) {
        set_error("compatibility_probe: null buffer");
        return QVG_INVALID_ARGUMENT;
    }
    const uint64_t sample_n = sample_size < n ? sample_size : n;
    if (sample_n < 100) {
        set_error("compatibility_probe: sample too small (< 100)");
        return QVG_INVALID_ARGUMENT;
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
    qvg_status st;
    DevBuf db, flag;
    const float* d = nullptr;
    if ((st = device_view(data, sample_n * (size_t)dim, db, &d, nullptr)) != QVG_OK) return st;
    if (!flag.alloc(4)) return cuda_status(cudaErrorMemoryAllocation, "compatibility_probe");
    cudaMemset(flag.p, 0, 4);
    rows_differ_kernel<<<592, 256>>>(d, sample_n, dim, static_cast<uint32_t*>(flag.p));
    uint32_t differ = 0;
    if ((e = cudaMemcpy(&differ, flag.p, 4, cudaMemcpyDeviceToHost)) != cudaSuccess)
        return cuda_status(e, "compatibility_probe");
    if (!differ) {
        set_error("compatibility_probe: degenerate sample (all identical)");
        return QVG_INVALID_ARGUMENT;
    }
    const uint64_t nq = sample_n < 1000 ? sample_n : 1000;
    std::vector<uint32_t> f(nq * k), b(nq * k), fc(nq), bc(nq);
    if ((st = qvg_brute_force_topk(device, d, sample_n, d, nq, dim, k, 0, 1, f.data(), nullptr,
                                   nullptr, fc.data())) != QVG_OK)
        return st;
    if ((st = qvg_brute_force_topk(device, d, sample_n, d, nq, dim, k, scorer, 1, b.data(),
                                   nullptr, nullptr, bc.data())) != QVG_OK)
        return st;
    // recall_at_k(bq, float, k) (eval.cpp:170-194)
    double total = 0.0;
    for (uint64_t qi = 0; qi < nq; ++qi) {
        if (fc[qi] < k) {
            set_error("recall_at_k: ground-truth row shorter than k");
            return QVG_INVALID_ARGUMENT;
        }
        size_t hits = 0;
        for (uint32_t i = 0; i < bc[qi]; ++i)
            for (uint32_t j = 0; j < k; ++j)
                if (b[qi * k + i] == f[qi * k + j]) {
                    ++hits;
                    break;
                }
        total += (double)hits / k;
    }
    out->overlap_at_k = total / (double)nq;
    out->sample_size = sample_n;
    out->k = k;
    out->go = out->overlap_at_k > 0.5 ? 1u : 0u;
    return QVG_OK;
}

qvg_status qvg_strong_bit_rate(qvg_index* index, const float* data, uint64_t count, uint32_t dim,
                               int device, qvg_encoding_diagnostics* out) {
    if (!out) {
        set_error("strong_bit_rate: null output");
        return QVG_INVALID_ARGUMENT;
    }
    DevBuf codes, bad, ctr;
    const uint4* d_codes = nullptr;
    uint64_t rows;
    uint32_t D, W;
    if (index) {  // strong_bit_rate(const SignatureStore&)
        if (index->ix.n == 0) {
            set_error("strong_bit_rate: empty store");
            return QVG_INVALID_ARGUMENT;
        }
        device = index->device;
        rows = index->ix.n;
        D = index->ix.dim;
        W = index->ix.W;
        d_codes = index->ix.codes;
    } else {  // strong_bit_rate(data, count, dim)
        if (count == 0 || dim == 0 || !data) {
            set_error("strong_bit_rate: empty sample");
            return QVG_INVALID_ARGUMENT;
        }
        rows = count;
        D = dim;
        W = (dim + 63) / 64;
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
    qvg_status st;
    if (!index) {
        DevBuf db;
        const float* d = nullptr;
        if ((st = device_view(data, rows * (size_t)D, db, &d, nullptr)) != QVG_OK) return st;
        if (!codes.alloc(rows * W * 16ull) || !bad.alloc(4))
            return cuda_status(cudaErrorMemoryAllocation, "strong_bit_rate");
        cudaMemset(bad.p, 0, 4);
        if ((st = encode_raw(d, rows, D, static_cast<uint4*>(codes.p),
                             static_cast<uint32_t*>(bad.p), nullptr)) != QVG_OK)
            return st;
        uint32_t hbad = 0;
        if ((e = cudaMemcpy(&hbad, bad.p, 4, cudaMemcpyDeviceToHost)) != cudaSuccess)
            return cuda_status(e, "strong_bit_rate");
        if (hbad) {
            set_error("encode: non-finite coordinate");
            return QVG_INVALID_ARGUMENT;
        }
        d_codes = static_cast<const uint4*>(codes.p);
    }
    if (!ctr.alloc(8)) return cuda_status(cudaErrorMemoryAllocation, "strong_bit_rate");
    cudaMemset(ctr.p, 0, 8);
    strong_count_kernel<<<592, 256>>>(d_codes, rows * W, static_cast<unsigned long long*>(ctr.p));
    unsigned long long total = 0;
    if ((e = cudaMemcpy(&total, ctr.p, 8, cudaMemcpyDeviceToHost)) != cudaSuccess)
        return cuda_status(e, "strong_bit_rate");
    out->sample_size = rows;
    out->p_s = (double)total / ((double)rows * D);
    out->nu2 = (1.0 + 3.0 * out->p_s) * (1.0 + 3.0 * out->p_s);
    return QVG_OK;
}

}  // extern "C"

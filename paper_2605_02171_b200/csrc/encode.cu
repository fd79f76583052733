// K1 — batched query encode (normalise + 2-bit Sign-Magnitude code), bit-exact
// with the reference's query path:
//   finite check           search.cpp:128-131
//   l2_norm / normalize_l2 vec_math.hpp:28-44  (sequential double sum, sqrt,
//                          float(1/n), float multiply)
//   compute_threshold      encoding.cpp:23-30  (sequential double sum of |y|,
//                          float(acc / D))
//   encode_sm2_into        encoding.cpp:32-45  (pos = y > 0, strong = |y| > tau,
//                          strict, pad bits zero)
// The double reductions must run in index order to round identically, so one
// lane owns one query's chain and the batch supplies the parallelism.
// Kernels (all bit-exact, tests/test_gpu_parity.py):
//   encode_lpq_kernel   (default) lane per query, rows staged in shared memory
//   encode_tiled_kernel lane per query through 32x32 transposed tiles (rows too
//                       wide for the staging buffer)
//   encode_warp_kernel  warp per query, lane 0 runs the chains
// QVG_ENCODE=1 / 2 forces the tiled / warp kernel (test hook, not a tuning
// surface: the default is the measured-fastest for every BASELINE geometry).
// All arithmetic uses explicit _rn intrinsics so no contraction can change a
// rounding.
#include <algorithm>
#include <cstdlib>

#include "qvg_internal.cuh"

namespace qvg {

namespace {

__device__ __forceinline__ bool finitef(float v) { return isfinite(v); }

__global__ void __launch_bounds__(128) encode_tiled_kernel(
    const float* __restrict__ x, uint64_t nq, uint32_t dim, uint32_t Dp, float* __restrict__ qn,
    uint4* __restrict__ qcodes, float* __restrict__ tau_out, int32_t* __restrict__ status,
    uint32_t* __restrict__ flags) {
    __shared__ float tile_all[4][32][33];  // +1 column: conflict-free transposes
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t q0 = ((uint64_t)blockIdx.x * 4 + wib) * 32;
    if (q0 >= nq) return;
    float(*T)[33] = tile_all[wib];
    const uint64_t myq = q0 + lane;
    const bool mine = myq < nq;
    const uint32_t W = (dim + 63) / 64;
    // columns [c0, c0+32) of the warp's 32 rows (row stride ld) -> T.  x goes
    // through the read-only path; qn (written by this warp in pass 2) must use
    // coherent loads.
    auto load = [&](const float* src, uint64_t ld, uint32_t c0, bool readonly) {
        __syncwarp();
#pragma unroll 8
        for (uint32_t r = 0; r < 32; ++r) {
            const uint64_t q = q0 + r;
            const float* p = src + q * ld + c0 + lane;
            T[r][lane] = (q < nq && c0 + lane < dim) ? (readonly ? __ldg(p) : *p) : 0.0f;
        }
        __syncwarp();
    };

    // pass 1: finite check + sequential sum of squares (vec_math.hpp:28-34);
    // x*x is exact in double, so the FMA rounds exactly like acc + x*x
    bool finite = true;
    double acc = 0.0;
    for (uint32_t c0 = 0; c0 < dim; c0 += 32) {
        load(x, dim, c0, true);
        const uint32_t lim = min(32u, dim - c0);
        for (uint32_t j = 0; j < lim; ++j) {
            const float v = T[lane][j];
            finite &= finitef(v);
            acc = __fma_rn((double)v, (double)v, acc);
        }
    }
    int32_t st = QVG_Q_OK;
    if (!finite) st = QVG_Q_NONFINITE_COORD;
    const double norm = __dsqrt_rn(acc);
    if (st == QVG_Q_OK && (!(norm > 0.0) || isinf(norm))) st = QVG_Q_BAD_NORM;
    const float inv = st == QVG_Q_OK ? __double2float_rn(__ddiv_rn(1.0, norm)) : 0.0f;

    // pass 2: y = x * inv (f32), finite check, sequential sum of |y|; store y
    // (zero padding up to Dp)
    double s = 0.0;
    bool yfinite = true;
    for (uint32_t c0 = 0; c0 < Dp; c0 += 32) {
        load(x, dim, c0, true);
        const uint32_t lim = c0 < dim ? min(32u, dim - c0) : 0u;
        for (uint32_t j = 0; j < lim; ++j) {
            const float y = st == QVG_Q_OK ? __fmul_rn(T[lane][j], inv) : 0.0f;
            yfinite &= finitef(y);
            s = __dadd_rn(s, fabs((double)y));
            T[lane][j] = y;
        }
        __syncwarp();
#pragma unroll 8
        for (uint32_t r = 0; r < 32; ++r) {
            const uint64_t q = q0 + r;
            if (q < nq && c0 + lane < Dp)
                qn[q * Dp + c0 + lane] = c0 + lane < dim ? T[r][lane] : 0.0f;
        }
    }
    if (st == QVG_Q_OK && !yfinite) st = QVG_Q_NONFINITE_CODE;
    const float tau = st == QVG_Q_OK ? __double2float_rn(__ddiv_rn(s, (double)dim)) : 0.0f;

    // pass 3: bit planes from y (re-read coalesced); a 32-column chunk is one
    // half of a 64-bit word, little-endian; pad bits zero
    uint32_t p_lo = 0, s_lo = 0;
    for (uint32_t c0 = 0; c0 < W * 64; c0 += 32) {
        uint32_t pb = 0, sb = 0;
        if (c0 < dim) {
            load(qn, Dp, c0, false);
            const uint32_t lim = min(32u, dim - c0);
            for (uint32_t j = 0; j < lim; ++j) {
                const float y = T[lane][j];
                pb |= (uint32_t)(y > 0.0f) << j;
                sb |= (uint32_t)(fabsf(y) > tau) << j;
            }
        }
        if (st != QVG_Q_OK) pb = sb = 0;
        if ((c0 & 63) == 0) {
            p_lo = pb;
            s_lo = sb;
        } else if (mine) {
            qcodes[myq * W + c0 / 64] = make_uint4(p_lo, pb, s_lo, sb);
        }
    }
    if (mine) {
        status[myq] = st;
        if (st != QVG_Q_OK && flags) atomicOr(flags, 1u << st);
        if (tau_out) tau_out[myq] = tau;
    }
}

// Lane-per-query (default): a block of 512 threads owns QB <= 32 consecutive
// queries staged in shared memory with an odd row stride ld (at step i lane q
// reads word q*ld + i: 32 distinct banks).  Lane q of warp 0 runs query q's two
// index-ordered double reductions, so one FP64 warp-instruction advances 32
// chains: the FP64 pipe issues ~0.5 warp-instructions per clock per SM on the
// B200 whatever the active-lane count (tools/fp64_chain_bench.cu), so a lane-0
// chain per query leaves 31/32 of it idle and throughput-bound.  Staging,
// scaling, the qn stores and the bit packing (two ballots per 32 elements) are
// element-parallel over the block's 16 warps (staging is load-latency bound:
// more warps keep more row loads in flight).
constexpr uint32_t kLpqThreads = 512;  // 16 warps stage the rows (loads in flight); warp 0 chains

__device__ __forceinline__ uint32_t lpq_ld(uint32_t dim) { return dim | 1u; }

__global__ void __launch_bounds__(kLpqThreads) encode_lpq_kernel(
    const float* __restrict__ x, uint64_t nq, uint32_t dim, uint32_t Dp, uint32_t QB,
    float* __restrict__ qn, uint4* __restrict__ qcodes, float* __restrict__ tau_out,
    int32_t* __restrict__ status, uint32_t* __restrict__ flags) {
    extern __shared__ float rows[];  // QB x ld
    __shared__ float s_inv[32], s_tau[32];
    __shared__ int32_t s_st[32], s_bad[32], s_ybad[32];
    constexpr uint32_t kWarps = kLpqThreads / 32;
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint64_t q0 = (uint64_t)blockIdx.x * QB;
    const uint32_t nb = (uint32_t)min((uint64_t)QB, nq - q0);
    const uint32_t ld = lpq_ld(dim);
    const bool vec4 = (dim & 3u) == 0 && (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
    if (tid < 32) s_bad[tid] = s_ybad[tid] = 0;
    __syncthreads();
    // stage the rows (warp per row, coalesced) + finite check (search.cpp:128-131)
    for (uint32_t r = wid; r < nb; r += kWarps) {
        const float* src = x + (q0 + r) * dim;
        float* row = rows + (size_t)r * ld;
        bool bad = false;
        if (vec4) {
            const float4* src4 = reinterpret_cast<const float4*>(src);
#pragma unroll 6
            for (uint32_t i = lane; i < dim / 4; i += 32) {
                const float4 v = __ldg(src4 + i);
                bad |= !(isfinite(v.x) & isfinite(v.y) & isfinite(v.z) & isfinite(v.w));
                row[4 * i] = v.x;
                row[4 * i + 1] = v.y;
                row[4 * i + 2] = v.z;
                row[4 * i + 3] = v.w;
            }
        } else {
#pragma unroll 8
            for (uint32_t i = lane; i < dim; i += 32) {
                const float v = __ldg(src + i);
                bad |= !isfinite(v);
                row[i] = v;
            }
        }
        bad = __any_sync(0xFFFFFFFFu, bad);
        if (lane == 0 && bad) s_bad[r] = 1;
    }
    __syncthreads();
    // chain 1 (vec_math.hpp:28-44): sum of squares in index order; x*x is
    // exact in double, so the FMA rounds exactly like acc + x*x
    if (wid == 0 && lane < nb) {
        int32_t st = s_bad[lane] ? QVG_Q_NONFINITE_COORD : QVG_Q_OK;
        float inv = 0.0f;
        if (st == QVG_Q_OK) {
            const float* row = rows + (size_t)lane * ld;
            double acc = 0.0;
#pragma unroll 8
            for (uint32_t i = 0; i < dim; ++i) acc = __fma_rn((double)row[i], (double)row[i], acc);
            const double norm = __dsqrt_rn(acc);
            if (!(norm > 0.0) || isinf(norm)) st = QVG_Q_BAD_NORM;
            else inv = __double2float_rn(__ddiv_rn(1.0, norm));
        }
        s_st[lane] = st;
        s_inv[lane] = inv;
    }
    __syncthreads();
    // y = x * inv (f32), in place; qn row with zero padding to Dp
    for (uint32_t r = wid; r < nb; r += kWarps) {
        const bool ok = s_st[r] == QVG_Q_OK;
        const float inv = s_inv[r];
        float* row = rows + (size_t)r * ld;
        float* dst = qn + (q0 + r) * Dp;
        bool bad = false;
#pragma unroll 4
        for (uint32_t i = lane; i < Dp; i += 32) {
            float y = 0.0f;
            if (i < dim) {
                y = ok ? __fmul_rn(row[i], inv) : 0.0f;
                bad |= !isfinite(y);
                row[i] = y;
            }
            dst[i] = y;
        }
        bad = __any_sync(0xFFFFFFFFu, bad);
        if (lane == 0 && bad) s_ybad[r] = 1;
    }
    __syncthreads();
    // chain 2 (encoding.cpp:23-30): tau = float(sum |y| / D), index order
    if (wid == 0 && lane < nb) {
        int32_t st = s_st[lane];
        if (st == QVG_Q_OK && s_ybad[lane]) st = QVG_Q_NONFINITE_CODE;
        float tau = 0.0f;
        if (st == QVG_Q_OK) {
            const float* row = rows + (size_t)lane * ld;
            double s = 0.0;
#pragma unroll 8
            for (uint32_t i = 0; i < dim; ++i) s = __dadd_rn(s, fabs((double)row[i]));
            tau = __double2float_rn(__ddiv_rn(s, (double)dim));
        }
        s_st[lane] = st;
        s_tau[lane] = tau;
        const uint64_t q = q0 + lane;
        status[q] = st;
        if (st != QVG_Q_OK && flags) atomicOr(flags, 1u << st);
        if (tau_out) tau_out[q] = tau;
    }
    __syncthreads();
    // bit planes (encode_sm2_into, encoding.cpp:32-45): warp per (row, 64-bit
    // word), lane b of each half sets bit b; pad bits and failed rows zero
    const uint32_t W = (dim + 63) / 64;
    for (uint32_t t = wid; t < nb * W; t += kWarps) {
        const uint32_t r = t / W, w = t - r * W;
        const bool ok = s_st[r] == QVG_Q_OK;
        const float tau = s_tau[r];
        const float* row = rows + (size_t)r * ld;
        uint32_t pb[2], sb[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t i = w * 64 + h * 32 + lane;
            const float y = (ok && i < dim) ? row[i] : 0.0f;
            pb[h] = __ballot_sync(0xFFFFFFFFu, y > 0.0f);
            sb[h] = __ballot_sync(0xFFFFFFFFu, ok && i < dim && fabsf(y) > tau);
        }
        if (lane == 0) qcodes[(q0 + r) * W + w] = make_uint4(pb[0], pb[1], sb[0], sb[1]);
    }
}

// Warp-per-query variant: the row is loaded coalesced into shared memory, lane
// 0 runs the two order-sensitive double reductions from shared memory (the
// DFMA/DADD dependency chain is the cost, ~D steps), and all lanes do the
// elementwise scaling, stores and bit packing.  With one warp per query the
// batch provides thousands of warps to hide the chains' latency.
__global__ void __launch_bounds__(256) encode_warp_kernel(
    const float* __restrict__ x, uint64_t nq, uint32_t dim, uint32_t Dp, float* __restrict__ qn,
    uint4* __restrict__ qcodes, float* __restrict__ tau_out, int32_t* __restrict__ status,
    uint32_t* __restrict__ flags) {
    extern __shared__ __align__(16) float rows_all[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t q = (uint64_t)blockIdx.x * 8 + wib;
    if (q >= nq) return;
    float* row = rows_all + (size_t)wib * Dp;
    const float* src = x + q * dim;
    const uint32_t W = (dim + 63) / 64;

    bool finite = true;
    for (uint32_t i = lane; i < dim; i += 32) {
        const float v = __ldg(src + i);
        finite &= finitef(v);
        row[i] = v;
    }
    finite = __all_sync(0xFFFFFFFFu, finite);
    __syncwarp();
    // pass 1 (lane 0): sequential sum of squares (vec_math.hpp:28-34)
    double inv_d = 0.0;
    int32_t st = finite ? QVG_Q_OK : QVG_Q_NONFINITE_COORD;
    if (lane == 0 && st == QVG_Q_OK) {
        double acc = 0.0;
#pragma unroll 8
        for (uint32_t i = 0; i < dim; ++i) acc = __fma_rn((double)row[i], (double)row[i], acc);
        const double norm = __dsqrt_rn(acc);
        if (!(norm > 0.0) || isinf(norm)) st = QVG_Q_BAD_NORM;
        else inv_d = __ddiv_rn(1.0, norm);
    }
    st = __shfl_sync(0xFFFFFFFFu, st, 0);
    const float inv = __double2float_rn(__shfl_sync(0xFFFFFFFFu, inv_d, 0));
    // y = x * inv, stored to smem and (coalesced) to qn with zero padding
    bool yfinite = true;
    for (uint32_t i = lane; i < Dp; i += 32) {
        const float y = (i < dim && st == QVG_Q_OK) ? __fmul_rn(row[i], inv) : 0.0f;
        yfinite &= finitef(y);
        if (i < dim) row[i] = y;
        qn[q * Dp + i] = y;
    }
    yfinite = __all_sync(0xFFFFFFFFu, yfinite);
    if (st == QVG_Q_OK && !yfinite) st = QVG_Q_NONFINITE_CODE;
    __syncwarp();
    // pass 2 (lane 0): sequential sum of |y| -> tau (encoding.cpp:23-30)
    float tau_l = 0.0f;
    if (lane == 0 && st == QVG_Q_OK) {
        double s = 0.0;
#pragma unroll 8
        for (uint32_t i = 0; i < dim; ++i) s = __dadd_rn(s, fabs((double)row[i]));
        tau_l = __double2float_rn(__ddiv_rn(s, (double)dim));
    }
    const float tau = __shfl_sync(0xFFFFFFFFu, tau_l, 0);
    // bit planes: lane w packs 64-bit word w
    for (uint32_t w = lane; w < W; w += 32) {
        uint32_t p0 = 0, p1 = 0, s0 = 0, s1 = 0;
        if (st == QVG_Q_OK) {
            const uint32_t b0 = w * 64, lim = min(64u, dim - b0);
            for (uint32_t b = 0; b < lim; ++b) {
                const float y = row[b0 + b];
                const uint32_t pbit = y > 0.0f, sbit = fabsf(y) > tau;
                if (b < 32) {
                    p0 |= pbit << b;
                    s0 |= sbit << b;
                } else {
                    p1 |= pbit << (b - 32);
                    s1 |= sbit << (b - 32);
                }
            }
        }
        qcodes[q * W + w] = make_uint4(p0, p1, s0, s1);
    }
    if (lane == 0) {
        status[q] = st;
        if (st != QVG_Q_OK && flags) atomicOr(flags, 1u << st);
        if (tau_out) tau_out[q] = tau;
    }
}

// reference layout (W pos words, W strong words per row) -> 16-B chunks
__global__ void codes_to_chunks_kernel(const uint64_t* __restrict__ ref, uint64_t rows,
                                       uint32_t W, uint4* __restrict__ out) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= rows * W) return;
    const uint64_t r = t / W;
    const uint32_t w = (uint32_t)(t % W);
    const uint64_t p = ref[r * 2 * W + w];
    const uint64_t s = ref[r * 2 * W + W + w];
    out[t] = make_uint4((uint32_t)p, (uint32_t)(p >> 32), (uint32_t)s, (uint32_t)(s >> 32));
}

__global__ void chunks_to_codes_kernel(const uint4* __restrict__ in, uint64_t rows, uint32_t W,
                                       uint64_t* __restrict__ ref) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= rows * W) return;
    const uint64_t r = t / W;
    const uint32_t w = (uint32_t)(t % W);
    const uint4 c = in[t];
    ref[r * 2 * W + w] = (uint64_t)c.x | ((uint64_t)c.y << 32);
    ref[r * 2 * W + W + w] = (uint64_t)c.z | ((uint64_t)c.w << 32);
}

}  // namespace

void launch_encode(const float* x, uint64_t nq, uint32_t dim, uint32_t Dp, float* qn,
                   uint4* qcodes, float* tau, int32_t* status, uint32_t* flags,
                   cudaStream_t s) {
    if (nq == 0) return;
    const size_t smem = 8ull * Dp * sizeof(float);
    static int variant = [] {
        const char* v = getenv("QVG_ENCODE");
        return v ? atoi(v) : 0;
    }();
    if (variant == 0) {
        // largest QB (<= 32 queries per block) that still fits the batch in one
        // wave of resident blocks; QB = 32 when no QB does (large batches)
        static int sms = [] {
            int d = 0, v = 0;
            cudaGetDevice(&d);
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
            return v > 0 ? v : 1;
        }();
        const size_t row_bytes = (size_t)(dim | 1u) * 4;
        const size_t cap = 200u * 1024u;
        uint32_t qb = 0;
        for (uint32_t c = 32; c >= 4; --c) {
            const size_t sm = row_bytes * c;
            if (sm > cap) continue;
            const uint64_t per_sm = std::min<uint64_t>(227u * 1024u / (sm + 1024u), 2048u / kLpqThreads);
            if (!qb) qb = c;  // largest that fits in shared memory
            if ((nq + c - 1) / c <= per_sm * (uint64_t)sms) {
                qb = c;
                break;
            }
        }
        if (qb) {
            const size_t lsmem = row_bytes * qb;
            static size_t lpq_attr = 0;  // attribute calls cost host time on small batches
            if (lsmem > lpq_attr) {
                cudaFuncSetAttribute(encode_lpq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(200u * 1024u));
                lpq_attr = 200u * 1024u;
            }
            const unsigned blocks = (unsigned)((nq + qb - 1) / qb);
            encode_lpq_kernel<<<blocks, kLpqThreads, lsmem, s>>>(x, nq, dim, Dp, qb, qn, qcodes,
                                                                 tau, status, flags);
            return;
        }
    }
    if (variant == 1 || smem > 200 * 1024) {
        const unsigned blocks = (unsigned)((nq + 127) / 128);
        encode_tiled_kernel<<<blocks, 128, 0, s>>>(x, nq, dim, Dp, qn, qcodes, tau, status, flags);
        return;
    }
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(encode_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    const unsigned blocks = (unsigned)((nq + 7) / 8);
    encode_warp_kernel<<<blocks, 256, smem, s>>>(x, nq, dim, Dp, qn, qcodes, tau, status, flags);
}

void launch_codes_to_chunks(const uint64_t* ref_codes, uint64_t rows, uint32_t W, uint4* out,
                            cudaStream_t s) {
    const uint64_t t = rows * W;
    if (t == 0) return;
    codes_to_chunks_kernel<<<(unsigned)((t + 255) / 256), 256, 0, s>>>(ref_codes, rows, W, out);
}

void launch_chunks_to_codes(const uint4* chunks, uint64_t rows, uint32_t W, uint64_t* out,
                            cudaStream_t s) {
    const uint64_t t = rows * W;
    if (t == 0) return;
    chunks_to_codes_kernel<<<(unsigned)((t + 255) / 256), 256, 0, s>>>(chunks, rows, W, out);
}

}  // namespace qvg

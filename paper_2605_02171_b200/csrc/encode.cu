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
// thread owns one query; the batch supplies the parallelism (10k queries =
// 10k threads).  All arithmetic uses explicit _rn intrinsics so no contraction
// or fast-math can change a rounding.
#include "qvg_internal.cuh"

namespace qvg {

namespace {

__device__ __forceinline__ bool finitef(float v) { return isfinite(v); }

template <bool VEC4>
__global__ void __launch_bounds__(128) encode_kernel(const float* __restrict__ x, uint64_t nq,
                                                     uint32_t dim, uint32_t Dp,
                                                     float* __restrict__ qn,
                                                     uint4* __restrict__ qcodes,
                                                     float* __restrict__ tau_out,
                                                     int32_t* __restrict__ status,
                                                     uint32_t* __restrict__ flags) {
    const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint32_t W = (dim + 63) / 64;
    const float* row = x + q * dim;
    float* out = qn + q * Dp;
    uint4* code = qcodes + q * W;

    // pass 1: finite check + sum of squares (vec_math.hpp:28-34)
    bool finite = true;
    double acc = 0.0;
    if (VEC4) {
        const float4* r4 = reinterpret_cast<const float4*>(row);
        for (uint32_t i = 0; i < dim / 4; ++i) {
            const float4 v = __ldg(r4 + i);
            finite &= finitef(v.x) & finitef(v.y) & finitef(v.z) & finitef(v.w);
            acc = __fma_rn((double)v.x, (double)v.x, acc);  // product exact in double
            acc = __fma_rn((double)v.y, (double)v.y, acc);
            acc = __fma_rn((double)v.z, (double)v.z, acc);
            acc = __fma_rn((double)v.w, (double)v.w, acc);
        }
    } else {
        for (uint32_t i = 0; i < dim; ++i) {
            const float v = __ldg(row + i);
            finite &= finitef(v);
            acc = __fma_rn((double)v, (double)v, acc);
        }
    }
    int32_t st = QVG_Q_OK;
    if (!finite) st = QVG_Q_NONFINITE_COORD;
    const double norm = __dsqrt_rn(acc);
    if (st == QVG_Q_OK && (!(norm > 0.0) || isinf(norm))) st = QVG_Q_BAD_NORM;
    if (st != QVG_Q_OK) {
        status[q] = st;
        if (flags) atomicOr(flags, 1u << st);
        if (tau_out) tau_out[q] = 0.0f;
        for (uint32_t i = 0; i < Dp; ++i) out[i] = 0.0f;
        for (uint32_t w = 0; w < W; ++w) code[w] = make_uint4(0, 0, 0, 0);
        return;
    }
    const float inv = __double2float_rn(__ddiv_rn(1.0, norm));

    // pass 2: y = x * inv (f32), finite check of y, sequential sum of |y|
    double s = 0.0;
    bool yfinite = true;
    if (VEC4) {
        const float4* r4 = reinterpret_cast<const float4*>(row);
        float4* o4 = reinterpret_cast<float4*>(out);
        for (uint32_t i = 0; i < dim / 4; ++i) {
            const float4 v = __ldg(r4 + i);
            float4 y;
            y.x = __fmul_rn(v.x, inv);
            y.y = __fmul_rn(v.y, inv);
            y.z = __fmul_rn(v.z, inv);
            y.w = __fmul_rn(v.w, inv);
            yfinite &= finitef(y.x) & finitef(y.y) & finitef(y.z) & finitef(y.w);
            s = __dadd_rn(s, fabs((double)y.x));
            s = __dadd_rn(s, fabs((double)y.y));
            s = __dadd_rn(s, fabs((double)y.z));
            s = __dadd_rn(s, fabs((double)y.w));
            o4[i] = y;
        }
    } else {
        for (uint32_t i = 0; i < dim; ++i) {
            const float y = __fmul_rn(__ldg(row + i), inv);
            yfinite &= finitef(y);
            s = __dadd_rn(s, fabs((double)y));
            out[i] = y;
        }
    }
    for (uint32_t i = dim; i < Dp; ++i) out[i] = 0.0f;
    if (!yfinite) {
        status[q] = QVG_Q_NONFINITE_CODE;
        if (flags) atomicOr(flags, 1u << QVG_Q_NONFINITE_CODE);
        if (tau_out) tau_out[q] = 0.0f;
        for (uint32_t w = 0; w < W; ++w) code[w] = make_uint4(0, 0, 0, 0);
        return;
    }
    const float tau = __double2float_rn(__ddiv_rn(s, (double)dim));

    // pass 3: bit planes, little-endian within 64-bit words, pad bits zero
    for (uint32_t w = 0; w < W; ++w) {
        uint32_t p0 = 0, p1 = 0, s0 = 0, s1 = 0;
        const uint32_t base = w * 64;
        const uint32_t lim = min(64u, dim - base);
        for (uint32_t b = 0; b < lim; ++b) {
            const float y = out[base + b];
            const uint32_t pbit = y > 0.0f;
            const uint32_t sbit = fabsf(y) > tau;
            if (b < 32) {
                p0 |= pbit << b;
                s0 |= sbit << b;
            } else {
                p1 |= pbit << (b - 32);
                s1 |= sbit << (b - 32);
            }
        }
        code[w] = make_uint4(p0, p1, s0, s1);
    }
    status[q] = QVG_Q_OK;
    if (tau_out) tau_out[q] = tau;
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
    const unsigned blocks = (unsigned)((nq + 127) / 128);
    const bool vec4 = (dim % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    if (vec4)
        encode_kernel<true><<<blocks, 128, 0, s>>>(x, nq, dim, Dp, qn, qcodes, tau, status, flags);
    else
        encode_kernel<false><<<blocks, 128, 0, s>>>(x, nq, dim, Dp, qn, qcodes, tau, status, flags);
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

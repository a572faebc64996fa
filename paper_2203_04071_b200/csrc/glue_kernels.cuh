// glue_kernels.cuh -- model glue around the LUT layers (sm_100a): int8 max pooling, global
// average pooling (+ fused quantize) for the ResNet-50-shaped forward (BASELINE.json
// configs[3], A16/A17) and the LSTM cell with the pinned fp32 exp of DESIGN.md A18
// (BASELINE.json configs[4]).  All HBM-bound element-wise kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "epilogue.cuh"
#include "pinned_math.cuh"

namespace axq {

// ---- max pooling over int8 codes, NHWC, 4 channels per thread via byte-SIMD max ----
__global__ void maxpool_nhwc_i8_kernel(const int8_t* __restrict__ x, int64_t N, int H, int W,
                                       int C, int R, int S, int stride, int pad, int Ho, int Wo,
                                       int8_t* __restrict__ y) {
    const int C4 = C / 4;
    const int64_t total = N * Ho * Wo * (int64_t)C4;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += gs) {
        const int c4 = (int)(i % C4);
        int64_t t = i / C4;
        const int wo = (int)(t % Wo);
        t /= Wo;
        const int ho = (int)(t % Ho);
        const int64_t n = t / Ho;
        unsigned int m = 0x80808080u;  // -128 in every byte
        for (int r = 0; r < R; ++r) {
            const int hi = ho * stride - pad + r;
            if (hi < 0 || hi >= H) continue;
            for (int s = 0; s < S; ++s) {
                const int wi = wo * stride - pad + s;
                if (wi < 0 || wi >= W) continue;
                const unsigned int v = __ldg(reinterpret_cast<const unsigned int*>(
                    x + ((n * H + hi) * W + wi) * C) + c4);
                m = __vmaxs4(m, v);
            }
        }
        reinterpret_cast<unsigned int*>(y + ((n * Ho + ho) * Wo + wo) * C)[c4] = m;
    }
}

// 16 channels per thread (C % 16 == 0, 16-byte aligned), 32-bit indices (the caller checks the
// item count): the ResNet maxpool after the stem is HBM/L2 bound, not index-math bound
__global__ void maxpool_nhwc_i8x16_kernel(const int8_t* __restrict__ x, int N, int H, int W, int C, int R,
                                          int S, int stride, int pad, int Ho, int Wo,
                                          int8_t* __restrict__ y) {
    const int C16 = C >> 4;
    const int total = N * Ho * Wo * C16;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int c16 = i % C16;
        int t = i / C16;
        const int wo = t % Wo;
        t /= Wo;
        const int ho = t % Ho;
        const int n = t / Ho;
        uint4 m = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);   // -128
        for (int r = 0; r < R; ++r) {
            const int hi = ho * stride - pad + r;
            if (hi < 0 || hi >= H) continue;
            for (int s_ = 0; s_ < S; ++s_) {
                const int wi = wo * stride - pad + s_;
                if (wi < 0 || wi >= W) continue;
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + ((int64_t)(n * H + hi) * W + wi) * C) + c16);
                m.x = __vmaxs4(m.x, v.x); m.y = __vmaxs4(m.y, v.y);
                m.z = __vmaxs4(m.z, v.z); m.w = __vmaxs4(m.w, v.w);
            }
        }
        reinterpret_cast<uint4*>(y + ((int64_t)(n * Ho + ho) * Wo + wo) * C)[c16] = m;
    }
}

// fp32 NHWC max pooling (out-of-image taps ignored, A17): the calibration pass of the paper
// quantizer needs the pooled real values (a percentile does not commute with pooling as the
// max does)
__global__ void maxpool_nhwc_f32_kernel(const float* __restrict__ x, int64_t N, int H, int W, int C, int R,
                                        int S, int stride, int pad, int Ho, int Wo, float* __restrict__ y) {
    const int64_t total = N * Ho * Wo * (int64_t)C;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += gs) {
        const int c = (int)(i % C);
        int64_t t = i / C;
        const int wo = (int)(t % Wo);
        t /= Wo;
        const int ho = (int)(t % Ho);
        const int64_t n = t / Ho;
        float m = -INFINITY;
        for (int r = 0; r < R; ++r) {
            const int hi = ho * stride - pad + r;
            if (hi < 0 || hi >= H) continue;
            for (int s = 0; s < S; ++s) {
                const int wi = wo * stride - pad + s;
                if (wi < 0 || wi >= W) continue;
                m = fmaxf(m, __ldg(x + ((n * H + hi) * W + wi) * C + c));
            }
        }
        y[i] = m;
    }
}

__global__ void maxpool_nhwc_i8_bytes_kernel(const int8_t* __restrict__ x, int64_t N, int H, int W,
                                             int C, int R, int S, int stride, int pad, int Ho,
                                             int Wo, int8_t* __restrict__ y) {
    const int64_t total = N * Ho * Wo * (int64_t)C;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += gs) {
        const int c = (int)(i % C);
        int64_t t = i / C;
        const int wo = (int)(t % Wo);
        t /= Wo;
        const int ho = (int)(t % Ho);
        const int64_t n = t / Ho;
        int m = -128;
        for (int r = 0; r < R; ++r) {
            const int hi = ho * stride - pad + r;
            if (hi < 0 || hi >= H) continue;
            for (int s = 0; s < S; ++s) {
                const int wi = wo * stride - pad + s;
                if (wi < 0 || wi >= W) continue;
                m = max(m, (int)x[((n * H + hi) * W + wi) * C + c]);
            }
        }
        y[((n * Ho + ho) * Wo + wo) * C + c] = (int8_t)m;
    }
}

// ---- global average pool: sequential fp32 sum over hw, one IEEE division (A17) ----
__global__ void avgpool_nhwc_kernel(const float* __restrict__ x, int64_t N, int64_t HW,
                                    int64_t C, float* __restrict__ y, int8_t* __restrict__ q,
                                    const float* __restrict__ d_scale, int bits) {
    const float s = q ? *d_scale : 1.f;
    const float qm = (float)((1 << (bits - 1)) - 1);
    const float inv_n = (float)HW;
    const int64_t total = N * C;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += gs) {
        const int64_t n = i / C, c = i - n * C;
        const float* xp = x + n * HW * C + c;
        float acc = 0.f;
        for (int64_t p = 0; p < HW; ++p) acc = __fadd_rn(acc, xp[p * C]);
        const float v = __fdiv_rn(acc, inv_n);
        if (y) y[i] = v;
        if (q) q[i] = epi_quant(v, s, qm);
    }
}

// ---- LSTM cell (pinned transcendentals: pinned_math.cuh, A18) ----
__global__ void lstm_cell_kernel(int64_t B, int64_t Hd, const float* __restrict__ gih,
                                 const float* __restrict__ ghh, float* __restrict__ c,
                                 float* __restrict__ h, int8_t* __restrict__ qh,
                                 const float* __restrict__ d_scale_h, int bits) {
    const float s = qh ? *d_scale_h : 1.f;
    const float qm = (float)((1 << (bits - 1)) - 1);
    const int64_t total = B * Hd;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += gs) {
        const int64_t b = i / Hd, j = i - b * Hd;
        const int64_t base = b * 4 * Hd + j;
        const float gi = __fadd_rn(gih[base], ghh[base]);
        const float gf = __fadd_rn(gih[base + Hd], ghh[base + Hd]);
        const float gg = __fadd_rn(gih[base + 2 * Hd], ghh[base + 2 * Hd]);
        const float go = __fadd_rn(gih[base + 3 * Hd], ghh[base + 3 * Hd]);
        const float ig = pinned_sigmoid(gi), fg = pinned_sigmoid(gf);
        const float g = pinned_tanh(gg), og = pinned_sigmoid(go);
        const float cn = __fadd_rn(__fmul_rn(fg, c[i]), __fmul_rn(ig, g));
        const float hn = __fmul_rn(og, pinned_tanh(cn));
        c[i] = cn;
        h[i] = hn;
        if (qh) qh[i] = epi_quant(hn, s, qm);
    }
}

// ---- explicit im2col of int8 NHWC codes (the stem: C = 3 valid channels stored as 4) ----
// A[m][k] for k = (r*S + s)*cv + c < K = R*S*cv: X[img][hi][wi][c] inside the image, 0 at a
// padded tap (the paper's im2col, P:119 -- a padded 0 is still looked up downstream, A11);
// k in [K, lda) is 0 (storage padding).  taps[k] = (r*dh) | (s*dw) << 8 | c << 16, ~0 past K.
__global__ void im2col_nhwc_i8_kernel(const int8_t* __restrict__ X, int64_t M, int H, int W, int C,
                                      int Ho, int Wo, int sh, int sw, int ph, int pw, int S, int cv, int K,
                                      int lda, int8_t* __restrict__ A) {
    extern __shared__ uint32_t taps[];
    for (int k = threadIdx.x; k < lda; k += blockDim.x) {
        uint32_t t = ~0u;
        if (k < K) {
            const int rs = k / cv, c = k - rs * cv, r = rs / S, s_ = rs - r * S;
            t = (uint32_t)r | ((uint32_t)s_ << 8) | ((uint32_t)c << 16);
        }
        taps[k] = t;
    }
    __syncthreads();
    const int chunks = lda / 16;
    const int64_t total = M * chunks;
    const int64_t hw = (int64_t)Ho * Wo;
    if (cv == C && (C & 15) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 && total < ((int64_t)1 << 31) &&
        (int64_t)H * W * C < ((int64_t)1 << 31)) {
        // 16 consecutive k = 16 channels of one tap: one 16-byte load per chunk, 32-bit index math
        const int hw32 = Ho * Wo, tot = (int)total;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
            const int m = i / chunks, j = i - m * chunks;
            const int img = m / hw32, rem = m - img * hw32;
            const int ho = rem / Wo, wo = rem - ho * Wo;
            const uint32_t t = taps[16 * j];
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (t != ~0u) {
                const int hi = ho * sh - ph + (int)(t & 0xffu), wi = wo * sw - pw + (int)((t >> 8) & 0xffu);
                if ((unsigned)hi < (unsigned)H && (unsigned)wi < (unsigned)W)
                    v = __ldg(reinterpret_cast<const uint4*>(X + (int64_t)img * H * W * C + (hi * W + wi) * C +
                                                             (int)(t >> 16)));
            }
            reinterpret_cast<uint4*>(A + (int64_t)m * lda)[j] = v;
        }
        return;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = i / chunks;
        const int j = (int)(i - m * chunks);
        const int64_t img = m / hw, rem = m - img * hw;
        const int ho = (int)(rem / Wo), wo = (int)(rem - (int64_t)ho * Wo);
        const int hb = ho * sh - ph, wb = wo * sw - pw;
        const int8_t* xb = X + img * (int64_t)H * W * C;
        uint32_t w4[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const uint32_t t = taps[16 * j + b];
            if (t == ~0u) continue;
            const int hi = hb + (int)(t & 0xffu), wi = wb + (int)((t >> 8) & 0xffu);
            if ((unsigned)hi < (unsigned)H && (unsigned)wi < (unsigned)W)
                w4[b >> 2] |= (uint32_t)(uint8_t)__ldg(xb + ((int64_t)hi * W + wi) * C + (int)(t >> 16)) << (8 * (b & 3));
        }
        reinterpret_cast<uint4*>(A + m * lda)[j] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
}

// The stem's shape specialised (C = 4 stored, 3 valid channels, R x S taps): one thread builds
// one whole row in registers -- one 4-byte load per tap (its 3 channels), bytes placed at
// compile-time positions -- then writes it with 16-byte stores.
template <int R, int S, int CV, int LDA>
__global__ void __launch_bounds__(256) im2col_c4_kernel(const int8_t* __restrict__ X, int64_t M, int H, int W,
                                                        int Ho, int Wo, int sh, int sw, int ph, int pw,
                                                        int8_t* __restrict__ A) {
    // a block builds 256 consecutive rows in shared memory, then writes the contiguous
    // 256 x LDA-byte block with coalesced 16-byte stores (per-thread row stores at a 160-byte
    // stride left most of each store's sectors partial)
    constexpr int NW = LDA / 4, NV = LDA / 16;
    __shared__ uint4 tile[256 * NV];
    const int64_t hw = (int64_t)Ho * Wo;
    for (int64_t mb = (int64_t)blockIdx.x * 256; mb < M; mb += (int64_t)gridDim.x * 256) {
        const int64_t m = mb + threadIdx.x;
        if (m < M) {
            const int64_t img = m / hw, rem = m - img * hw;
            const int ho = (int)(rem / Wo), wo = (int)(rem - (int64_t)ho * Wo);
            const int hb = ho * sh - ph, wb = wo * sw - pw;
            const uint32_t* xb = reinterpret_cast<const uint32_t*>(X) + img * (int64_t)H * W;
            uint32_t out[NW];
#pragma unroll
            for (int i = 0; i < NW; ++i) out[i] = 0u;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int hi = hb + r;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const int wi = wb + s;
                    const uint32_t v = ((unsigned)hi < (unsigned)H && (unsigned)wi < (unsigned)W)
                                           ? __ldg(xb + (int64_t)hi * W + wi) : 0u;
#pragma unroll
                    for (int c = 0; c < CV; ++c) {
                        const int k = (r * S + s) * CV + c;
                        out[k >> 2] |= ((v >> (8 * c)) & 0xffu) << (8 * (k & 3));
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < NV; ++i)
                tile[threadIdx.x * NV + i] = make_uint4(out[4 * i], out[4 * i + 1], out[4 * i + 2], out[4 * i + 3]);
        }
        __syncthreads();
        const int rows = (int)min((int64_t)256, M - mb);
        uint4* dst = reinterpret_cast<uint4*>(A + mb * LDA);
        for (int j = threadIdx.x; j < rows * NV; j += 256) dst[j] = tile[j];
        __syncthreads();
    }
}

}  // namespace axq

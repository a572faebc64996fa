// gconv.cuh -- grouped / depthwise approximate convolution (NEXT-3; "groups"; the conv
// of Eq. 2, with each output channel reading only its group's input channels).
//
// out[n][ho][wo][co] = sum_{ci < C/G, r, s} LUT[a][w],  a = X[n][hi][wi][g*C/G + ci] (0 at a padded
// tap, still looked up, A11), w = W[co][r][s][ci], g = co / (K/G).  int32, exact.
//
// Design: a grouped layer has K = R*S*C/G lookups per output -- 9 for a depthwise 3x3 -- too
// few to amortise the packed-table staging, so the table stays resident (the v1 transposed
// layout [uw][ua]) in shared memory of a persistent CTA that walks (32-pixel, 8-channel)
// work items: lane = consecutive output pixels, warp = consecutive output channels, so a
// gather's 32 lanes share the weight and read one 256-byte table row (no bank conflicts) and
// neighbouring warps re-read the same activation sectors from L1.  The exact part of delta8
// tables is one integer multiply-add per lookup.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lut_mm.cuh"

namespace axq {

template <uint32_t SEL>
__device__ __forceinline__ int gc_sext(uint32_t v) {   // sign-extend a byte (PTX prmt sign mode)
    int r;
    asm("prmt.b32 %0, %1, 0, %2;\n" : "=r"(r) : "r"(v), "n"(SEL));
    return r;
}

struct GConvArgs {
    const int8_t* X;        // NHWC [N][H][W][C]
    const int8_t* W;        // [K][R][S][C/G]
    int64_t M;              // N * Ho * Wo
    int N, H, Wd, C, K, R, S, G, Ho, Wo, sh, sw, ph, pw, dh, dw;
    const void* table;      // representation-specific [uw][ua]
    int table_bytes;
    int32_t* C_out;         // raw int32 [M][K] (NHWC) or null -> fused epilogue
    EpiArgs ep;
};

template <int REPR>
__global__ void __launch_bounds__(256) lut_gconv_kernel(const GConvArgs a) {
    extern __shared__ __align__(16) int8_t gsm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if constexpr (REPR != REPR_I32) {
        const uint4* src = reinterpret_cast<const uint4*>(a.table);
        uint4* dst = reinterpret_cast<uint4*>(gsm);
        for (int i = tid; i < a.table_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
        __syncthreads();
    }
    const int32_t* tab_g = reinterpret_cast<const int32_t*>(a.table);
    const int cin_g = a.C / a.G, cout_g = a.K / a.G;
    const int64_t m_blocks = (a.M + 31) / 32, c_blocks = (a.K + 7) / 8;
    const int64_t work = m_blocks * c_blocks;
    const int64_t hw = (int64_t)a.Ho * a.Wo;
    float sc = 0.f, s_out = 1.f, qm = 127.f;
    if (!a.C_out) {
        sc = __fmul_rn(*a.ep.sa, *a.ep.sw);
        if (a.ep.q) {
            s_out = *a.ep.s_out;
            qm = (float)((1 << (a.ep.bits_out - 1)) - 1);
        }
    }
    for (int64_t it = blockIdx.x; it < work; it += gridDim.x) {
        const int64_t mb = it % m_blocks, cb = it / m_blocks;   // pixel blocks fastest: warps share W
        const int64_t m = mb * 32 + lane;
        const int co = (int)(cb * 8 + warp);
        if (m >= a.M || co >= a.K) continue;
        const uint32_t m32 = (uint32_t)m, img = m32 / (uint32_t)hw, rem = m32 - img * (uint32_t)hw;
        const int ho = (int)(rem / (uint32_t)a.Wo), wo = (int)rem - ho * a.Wo;
        const int g = co / cout_g;
        const int8_t* xb = a.X + (int64_t)img * a.H * a.Wd * a.C + g * cin_g;
        const int8_t* wb = a.W + (int64_t)co * a.R * a.S * cin_g;
        int acc = 0;
        for (int r = 0; r < a.R; ++r) {
            const int hi = ho * a.sh - a.ph + r * a.dh;
            const bool hok = (unsigned)hi < (unsigned)a.H;
            for (int s = 0; s < a.S; ++s) {
                const int wi = wo * a.sw - a.pw + s * a.dw;
                const bool ok = hok && (unsigned)wi < (unsigned)a.Wd;
                const int8_t* xp = xb + ((int64_t)hi * a.Wd + wi) * a.C;
                const int8_t* wp = wb + (r * a.S + s) * cin_g;
                for (int ci = 0; ci < cin_g; ++ci) {
                    const int av = ok ? (int)__ldg(xp + ci) : 0;
                    const int wv = (int)__ldg(wp + ci);
                    const uint32_t idx = ((uint32_t)(wv & 0xff) << 8) | (uint32_t)(av & 0xff);
                    if constexpr (REPR == REPR_DELTA8)
                        acc += (int)gsm[idx] + av * wv;
                    else
                        acc += lut_fetch<REPR>(gsm, tab_g, idx);
                }
            }
        }
        if (a.C_out) {
            a.C_out[m * a.K + co] = acc;
        } else {
            epi_store(epi_value(acc, m, co, sc, a.ep), m, co, a.K, a.ep, s_out, qm);
        }
    }
}

// Depthwise (C/G == 1, K == C): a thread owns 4 consecutive channels for a run of output
// pixels.  Its 4 x R*S weights live in registers for the whole run; per tap one coalesced
// 32-bit load brings the 4 activations (a warp reads 128 consecutive bytes of one pixel), then
// 4 lookups in the resident transposed table (+ 4 exact products for delta8).  The epilogue
// writes the 4 channels with one 16-byte fp32 / 4-byte code store where the layout allows.
template <int REPR, int KR, int KS>
__global__ void __launch_bounds__(256) lut_dwconv_kernel(const GConvArgs a) {
    constexpr int RS = KR * KS;
    extern __shared__ __align__(16) int8_t dsm[];
    const int tid = threadIdx.x;
    if constexpr (REPR != REPR_I32) {
        const uint4* src = reinterpret_cast<const uint4*>(a.table);
        uint4* dst = reinterpret_cast<uint4*>(dsm);
        for (int i = tid; i < a.table_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
        __syncthreads();
    }
    const int32_t* tab_g = reinterpret_cast<const int32_t*>(a.table);
    const int C4 = a.C / 4;
    // thread t of the grid: channel quad t % C4, pixel lane t / C4 (strided over pixels)
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + tid;
    const int q = (int)(t0 % C4);
    const int64_t pstride = nthreads / C4;                 // host guarantees nthreads % C4 == 0
    const int c0 = 4 * q;
    uint32_t wq[RS];                                       // the quad's weights, 4 per tap
#pragma unroll
    for (int t = 0; t < RS; ++t) {
        uint32_t v = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) v |= (uint32_t)(uint8_t)a.W[(int64_t)(c0 + j) * RS + t] << (8 * j);
        wq[t] = v;
    }
    const int64_t hw = (int64_t)a.Ho * a.Wo;
    float sc = 0.f, s_out = 1.f, qm = 127.f;
    if (!a.C_out) {
        sc = __fmul_rn(*a.ep.sa, *a.ep.sw);
        if (a.ep.q) {
            s_out = *a.ep.s_out;
            qm = (float)((1 << (a.ep.bits_out - 1)) - 1);
        }
    }
    for (int64_t m = t0 / C4; m < a.M; m += pstride) {
        // M < 2^31 (host check): 32-bit divisions, not the 64-bit subroutine
        const uint32_t m32 = (uint32_t)m, img = m32 / (uint32_t)hw, rem = m32 - img * (uint32_t)hw;
        const int ho = (int)(rem / (uint32_t)a.Wo), wo = (int)rem - ho * a.Wo;
        const int8_t* xb = a.X + (int64_t)img * a.H * a.Wd * a.C + c0;
        int acc[4] = {0, 0, 0, 0};
        uint32_t avs[RS];
#pragma unroll
        for (int r = 0; r < KR; ++r) {                     // all taps' loads first (ILP)
            const int hi = ho * a.sh - a.ph + r * a.dh;
#pragma unroll
            for (int s = 0; s < KS; ++s) {
                const int wi = wo * a.sw - a.pw + s * a.dw;
                avs[r * KS + s] = ((unsigned)hi < (unsigned)a.H && (unsigned)wi < (unsigned)a.Wd)
                                      ? __ldg(reinterpret_cast<const uint32_t*>(xb + ((int64_t)hi * a.Wd + wi) * a.C))
                                      : 0u;
            }
        }
#pragma unroll
        for (int t = 0; t < RS; ++t) {
            const uint32_t av = avs[t], wv = wq[t];
            if constexpr (REPR == REPR_DELTA8) {
                // exact part: the 4 channels' a*w from sign-extended byte pairs
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t idx = __byte_perm(av, wv, 0x4440u + j + ((4u + j) << 4) - 0x40u);  // [ua, uw, 0, 0]
                    acc[j] += (int)dsm[idx & 0xffffu];
                }
                acc[0] += gc_sext<0x8880>(av) * gc_sext<0x8880>(wv);
                acc[1] += gc_sext<0x9991>(av) * gc_sext<0x9991>(wv);
                acc[2] += gc_sext<0xaaa2>(av) * gc_sext<0xaaa2>(wv);
                acc[3] += gc_sext<0xbbb3>(av) * gc_sext<0xbbb3>(wv);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t idx = __byte_perm(av, wv, 0x4440u + j + ((4u + j) << 4) - 0x40u);
                    acc[j] += lut_fetch<REPR>(dsm, tab_g, idx & 0xffffu);
                }
            }
        }
        if (a.C_out) {
            *reinterpret_cast<int4*>(a.C_out + m * a.K + c0) = make_int4(acc[0], acc[1], acc[2], acc[3]);
        } else if (!a.ep.y_nchw && !a.ep.y && a.ep.q && (a.ep.ldq & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(a.ep.q) & 3) == 0) {
            uint32_t w = 0;                                   // 4 codes, one 32-bit store
#pragma unroll
            for (int j = 0; j < 4; ++j)
                w |= (uint32_t)(uint8_t)epi_quant(epi_value(acc[j], m, c0 + j, sc, a.ep), s_out, qm) << (8 * j);
            *reinterpret_cast<uint32_t*>(a.ep.q + m * a.ep.ldq + c0) = w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                epi_store(epi_value(acc[j], m, c0 + j, sc, a.ep), m, c0 + j, a.K, a.ep, s_out, qm);
        }
    }
}

}  // namespace axq

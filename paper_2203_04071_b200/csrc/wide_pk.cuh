// wide_pk.cuh -- packed weight-specialised LUT-GEMM for wide ACUs (NEXT-2: b = 9..12, the
// paper's 12-bit multipliers; the bitwidth experiment of P:322), int16 codes.
//
// acc[m][n] = sum_k LUT[a[m][k]][w[n][k]] (int32, exact) = sum_k a*w + sum_k E[a][w] with
// E = LUT - a*w in int16 (the WIDE16 representation).
//
// The compact 2^b x 2^b table (32 MiB at b = 12) cannot be shared-memory resident, and a
// gather from L2 moves a 32-byte sector per 2-byte lookup (the lut_wide_kernel bound).  Here the
// table is tiled instead: for every k and every quad of 4 output columns the weights are fixed,
// so the slab of the table those 4 weights select, T[k][q][ua] = 4 x (E[ua][w(4q+j, k)] + 2^15),
// is a contiguous 2^b x 8-byte run that one cp.async.bulk stages into shared memory, and ONE
// 64-bit LDS then serves 4 lookups of the lane's row.  A tile of BM rows reuses every staged
// slab BM times (2048 rows at b = 11, 12), which is what bounds the L2 -> shared traffic.
//
//  * Per-stage slab: KS k x NQ quads x 2^b codes x 8 B = 64 KiB (b = 12: KS 2, NQ 1; b = 11:
//    KS 4, NQ 1; b = 10: KS 4, NQ 2; b = 9: KS 4, NQ 4), three stages in flight, with the tile's
//    packed weights; one producer warp issues the bulk copies (mbarrier complete_tx), 16
//    consumer warps look up (lanes = rows, R = 4 / NQ rows per lane).
//  * E sums: biased 16-bit lanes of a 32-bit word v (columns 2i, 2i+1) accumulated as
//    pa = sum v (mod 2^32) and ph = sum (v >> 16); column 2i = pa - 2^16 ph, 2i+1 = ph, exact
//    for K < 2^16 -- no flushes.  The exact part a*w: one IMAD per lookup (12-bit codes do not
//    fit the int8 tensor-core path).
//  * K is padded to whole stages with a = 0 / w = 0 lookups, removed as (Kp - K) * LUT[0][0].
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "async_copy.cuh"
#include "epilogue.cuh"
#include "wide_args.h"
#include "wide_pk_geo.h"

namespace axq {

namespace wpk {
constexpr int CWARPS = 16;                  // consumer warps
constexpr int NT = (CWARPS + 1) * 32;       // + 1 producer warp
template <int BITS>
struct Geo {
    static constexpr int NCODES = 1 << BITS;
    static constexpr int TQB = NCODES * 8;                       // bytes per (k, quad) slab
    static constexpr int NQ = BITS >= 11 ? 1 : (BITS == 10 ? 2 : 4);
    static constexpr int R = 4 / NQ;                             // rows per lane
    static constexpr int BM = 32 * CWARPS * R;
    static constexpr int TN = 4 * NQ;
    static constexpr int KS = 65536 / (NQ * TQB);
    static constexpr int TBL_STAGE = KS * NQ * TQB;              // 64 KiB
    static constexpr int W_STAGE = KS * NQ * 8;                  // packed int16 weights
    static constexpr int STAGES = 3;
    static constexpr int SMEM_W = STAGES * TBL_STAGE;
    static constexpr int SMEM_BAR = SMEM_W + ((STAGES * W_STAGE + 15) / 16) * 16;
    static constexpr int SMEM_BYTES = SMEM_BAR + 8 * 2 * STAGES;
    static_assert(KS >= 1 && 8 % KS == 0, "k per stage must divide the 8-code A loads");
};
}  // namespace wpk


template <int BITS>
__global__ void __launch_bounds__(wpk::NT, 1) lut_widepk_kernel(const __grid_constant__ WidePkArgs P) {
    using G = wpk::Geo<BITS>;
    constexpr int KS = G::KS, NQ = G::NQ, R = G::R, BM = G::BM, TN = G::TN, STAGES = G::STAGES;
    extern __shared__ __align__(16) uint8_t wpk_smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t s_base = smem_u32(wpk_smem);
    const uint32_t bar_full = s_base + G::SMEM_BAR, bar_empty = bar_full + 8 * STAGES;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, wpk::CWARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int64_t n_blocks = (P.N + TN - 1) / TN, m_tiles = (P.M + BM - 1) / BM;
    const int64_t tiles = n_blocks * m_tiles;
    const int nst = (int)(P.Kp / KS);

    if (warp == wpk::CWARPS) {
        // ---- producer: one lane streams the slabs (tile order as the consumers') ----
        if (lane == 0) {
            uint32_t item = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int64_t nb = t / m_tiles;    // m fastest: concurrent CTAs share a slab stream
                for (int st = 0; st < nst; ++st, ++item) {
                    const int buf = (int)(item % STAGES);
                    if (item >= (uint32_t)STAGES) mbar_wait(bar_empty + 8 * buf, ((item / STAGES) - 1) & 1u);
                    const uint32_t bar = bar_full + 8 * buf;
                    mbar_expect_tx(bar, G::TBL_STAGE + G::W_STAGE);
                    const size_t k0 = (size_t)st * KS;
                    bulk_g2s(s_base + buf * G::TBL_STAGE,
                             P.tables + ((size_t)nb * P.Kp + k0) * NQ * G::NCODES, G::TBL_STAGE, bar);
                    bulk_g2s(s_base + G::SMEM_W + buf * G::W_STAGE,
                             P.wts + ((size_t)nb * P.Kp + k0) * NQ * 4, G::W_STAGE, bar);
                }
            }
        }
        return;
    }

    // ---- consumers ----
    const uint32_t mask = (uint32_t)G::NCODES - 1u;
    float sc = 0.f, s_out = 1.f, qm = 127.f;
    if (!P.C_out) {
        sc = __fmul_rn(*P.ep.sa, *P.ep.sw);
        if (P.ep.q) {
            s_out = *P.ep.s_out;
            qm = (float)((1 << (P.ep.bits_out - 1)) - 1);
        }
    }
    uint32_t item = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t nb = t / m_tiles, m0 = (t - nb * m_tiles) * BM;
        int64_t mrow[R];
        bool valid[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            mrow[r] = m0 + (int64_t)r * (32 * wpk::CWARPS) + warp * 32 + lane;
            valid[r] = mrow[r] < P.M;
        }
        uint32_t pa[R][NQ][2], ph[R][NQ][2];
        int ex[R][NQ][4];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                pa[r][q][0] = pa[r][q][1] = ph[r][q][0] = ph[r][q][1] = 0u;
#pragma unroll
                for (int j = 0; j < 4; ++j) ex[r][q][j] = 0;
            }
        // 8 codes per row, zero beyond K (a padded k looks up a = 0); loaded one k8 step ahead
        auto load_codes = [&](int k8, uint4 (&dst)[R]) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int16_t* src = P.A + (valid[r] ? mrow[r] : 0) * P.lda + k8;
                if (valid[r] && k8 + 8 <= P.K && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
                    dst[r] = __ldg(reinterpret_cast<const uint4*>(src));
                } else {
                    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (valid[r] && k8 + j < P.K) w[j >> 1] |= (uint32_t)(uint16_t)src[j] << (16 * (j & 1));
                    dst[r] = make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
        };
        uint4 acode[R], anext[R];
        load_codes(0, anext);
        for (int k8 = 0; k8 < (int)P.Kp; k8 += 8) {
#pragma unroll
            for (int r = 0; r < R; ++r) acode[r] = anext[r];
            if (k8 + 8 < (int)P.Kp) load_codes(k8 + 8, anext);
#pragma unroll
            for (int sub = 0; sub < 8 / KS; ++sub, ++item) {
                const int buf = (int)(item % STAGES);
                mbar_wait(bar_full + 8 * buf, (item / STAGES) & 1u);
                const uint8_t* tb = wpk_smem + buf * G::TBL_STAGE;
                const uint8_t* wb = wpk_smem + G::SMEM_W + buf * G::W_STAGE;
#pragma unroll
                for (int kk = 0; kk < KS; ++kk) {
                    const int kc = sub * KS + kk;              // code slot (compile-time after unrolling)
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        const uint2 wv = *reinterpret_cast<const uint2*>(wb + (kk * NQ + q) * 8);   // broadcast
                        const int w0 = (int)(int16_t)(wv.x & 0xffffu), w1 = (int)(int16_t)(wv.x >> 16);
                        const int w2 = (int)(int16_t)(wv.y & 0xffffu), w3 = (int)(int16_t)(wv.y >> 16);
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            const uint32_t cw = kc < 2 ? acode[r].x : kc < 4 ? acode[r].y : kc < 6 ? acode[r].z : acode[r].w;
                            const int a = (int)(int16_t)((kc & 1) ? (cw >> 16) : (cw & 0xffffu));
                            const uint32_t ua = (uint32_t)a & mask;
                            const uint2 v = *reinterpret_cast<const uint2*>(tb + ((kk * NQ + q) * G::NCODES + ua) * 8);
                            pa[r][q][0] += v.x;
                            ph[r][q][0] += v.x >> 16;
                            pa[r][q][1] += v.y;
                            ph[r][q][1] += v.y >> 16;
                            ex[r][q][0] += a * w0;
                            ex[r][q][1] += a * w1;
                            ex[r][q][2] += a * w2;
                            ex[r][q][3] += a * w3;
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_empty + 8 * buf);
            }
        }
        // ---- epilogue: E sums decoded, bias and padded lookups removed ----
        const int32_t corr = (int32_t)(32768 * P.Kp + (P.Kp - P.K) * (int64_t)P.t00);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (!valid[r]) continue;
            const int64_t m = mrow[r];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const uint32_t e[4] = {pa[r][q][0] - (ph[r][q][0] << 16), ph[r][q][0],
                                       pa[r][q][1] - (ph[r][q][1] << 16), ph[r][q][1]};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t n = nb * TN + q * 4 + j;
                    if (n >= P.N) continue;
                    const int32_t acc = (int32_t)((uint32_t)ex[r][q][j] + e[j] - (uint32_t)corr);
                    if (P.C_out) P.C_out[m * P.ldc + n] = acc;
                    else epi_store(epi_value(acc, m, n, sc, P.ep), m, n, P.N, P.ep, s_out, qm);
                }
            }
        }
    }
}

// wide packing: tables[nb][k][q][ua] = 4 x (E[ua][w(nb*TN + 4q + j, k)] + 2^15) (w = 0 outside
// N / K), from the WIDE16 device table e16 [uw][ua] (b-bit patterns); wts[nb][k][q][j] = w.
__global__ void widepk_pack_kernel(const int16_t* __restrict__ W, int64_t N, int64_t K, int64_t ldw, int64_t Kp,
                                   int bits, int nq, const int16_t* __restrict__ e16, uint2* __restrict__ tables,
                                   int16_t* __restrict__ wts) {
    const int64_t ncodes = (int64_t)1 << bits, tn = 4 * nq;
    const int64_t n_blocks = (N + tn - 1) / tn;
    const int64_t total = n_blocks * Kp * nq * ncodes;
    const uint32_t mask = (uint32_t)ncodes - 1u;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ua = i & (ncodes - 1);
        int64_t t = i >> bits;
        const int q = (int)(t % nq);
        t /= nq;
        const int64_t k = t % Kp, nb = t / Kp;
        uint32_t h[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t n = nb * tn + 4 * q + j;
            const int w = (n < N && k < K) ? (int)W[n * ldw + k] : 0;
            const int e = (int)e16[(((uint32_t)w & mask) << bits) | (uint32_t)ua];
            h[j] = (uint32_t)(e + 32768) & 0xffffu;
            if (ua == 0) wts[((nb * Kp + k) * nq + q) * 4 + j] = (int16_t)w;
        }
        tables[i] = make_uint2(h[0] | (h[1] << 16), h[2] | (h[3] << 16));
    }
}

}  // namespace axq

// lut_p4_args.h -- tile constants and launch arguments of the P4 kernel (lut_p4.cuh).
#pragma once
#include <cstdint>
#include <cuda.h>   // CUtensorMap (the type only; the encoder is fetched from the driver at run time)

#include "lut_mm.cuh"

namespace axq {

namespace p4 {
constexpr int TN = 16;                     // output columns per CTA tile (4 quads)
constexpr int WARPS = 16;
constexpr int NT = WARPS * 32;             // 512 threads
constexpr int KS = 16;                     // k per stage
constexpr int A_STAGE = 1024 * KS;         // activation tile per stage (1024 rows max)
constexpr int W_STAGE = TN * KS;           // 256 B weight tile per stage
constexpr int SCR_WARP = 64 * TN * 4;      // per-warp int32 [64 rows][16 cols] scratch
constexpr int FLUSH_STAGES = 16;           // 16-bit packed E sums: flush every 256 k
constexpr int E_BIAS = 128;                // tables hold E + 128 (unsigned bytes)
constexpr int TAP_BYTES = 2048;            // tap table of the 4-byte conv loader: Kp <= 2048

// Table geometry: full range (ua = 0..255, any activation code) or half range (ua = 0..127,
// non-negative activation codes, e.g. ReLU outputs): half the table bytes, one more stage.
template <bool HALF>
struct Geo {
    static constexpr int TROWS = HALF ? 128 : 256;         // entries per (k, quad) table
    static constexpr int TQ = TROWS * 4;                   // bytes per (k, quad) table
    static constexpr int TBL_STAGE = KS * (TN / 4) * TQ;   // 32 / 64 KiB per stage
    static constexpr int STAGES = HALF ? 3 : 2;
    static constexpr int SMEM_TBL = 0;
    static constexpr int SMEM_A = SMEM_TBL + STAGES * TBL_STAGE;
    static constexpr int SMEM_W = SMEM_A + STAGES * A_STAGE;
    static constexpr int SMEM_BAR = SMEM_W + STAGES * W_STAGE;
    static constexpr int SMEM_SCR = SMEM_BAR + 64;
    static constexpr int SMEM_TAP = SMEM_SCR + WARPS * SCR_WARP;   // 4-byte loader tap table
    static constexpr int SMEM_BYTES = SMEM_TAP + TAP_BYTES;
};
}  // namespace p4

struct P4Args {
    MMArgs mm;                  // geometry, loader info, t00, epilogue (k_split unused)
    const uint32_t* tables;     // [n_blocks][Kp][4][256 or 128] u32
    const int8_t* wpk;          // [n_blocks][Kp/16][16 n][16 k]
    int64_t Kp;                 // K rounded up to a multiple of 16
    int is_conv;
    uint32_t one;
    int splits;                 // K splits (>1: atomic int32 into C_out, epilogue run after)
    int stages_per_split;       // 16-k stages per split
    int rpl;                    // rows per lane: 2 (1024-row tiles) or 1 (512-row tiles)
    int half;                   // tables cover ua = 0..127 only (non-negative activations)
    int c4;                     // conv with C % 16 != 0 (C % 4 == 0): 4-byte tap copies
    int streamk;                // stream-K decomposition (needs ws and cnt): 1 whole waves + cut
                                // tail; 2 (P4W) every iteration cut, one slice per CTA
    int32_t* ws;                // P4W stream-K per-CTA partial slots [grid][2][BM][16] (caller's
                                // epilogue workspace, after the counters)
    int32_t* cnt;               // stream-K tile counters (>= sk_ctas), zero on entry, left zero
    int sk_ctas;                // P4W stream-K: CTAs sharing the tail (0 = all)
    int ks;                     // P4W: k per stage (16 or 32; 16 with half tables = 4 stages)
    int transposed;             // P4W: output element (row r, col c) goes to [c][r] (gemm_xs)
    int cw;                     // P4W consumer warps (tile rows / 32): 28 (default) or 16
    int e16;                    // P4W16: int16 E tables, 2 columns per packed word
    int grp_cout, grp_cin;      // grouped conv (P4W): output / input channels per group (0: none);
                                // a 16-column tile lies in group n0 / grp_cout, whose input
                                // channels start at that group * grp_cin of the pixel (stride cs)
    int pointwise;              // conv that is a plain GEMM of its NHWC input (1x1, stride 1,
                                // pad 0): rows loaded as GEMM rows (lda = C), no per-row division
    int nb_fast;                // tile order: column block fastest (the layer's tables stay in
                                // L2 and each activation tile is read from HBM once) instead of
                                // row tile fastest (concurrent CTAs share one table stream)
    int tma_a;                  // P4W GEMM-row loader: activation planes by TMA (tmap_a) instead
                                // of per-row cp.async (no LSU wavefronts for the operand stream)
    alignas(64) CUtensorMap tmap_a;   // 2D u8 [M][K] (row stride lda), box 16 k x 128 rows,
                                      // out-of-range rows and k >= K read as zeros
    int tma_res;                // P4W residual layers: the epilogue's fp32 residual rows by TMA
    int tma_y;                  // ... and its fp32 y rows written back by TMA stores
    alignas(64) CUtensorMap tmap_res; // 2D fp32 [M][N] (row stride ldr), box 16 cols x 128 rows,
                                      // 64-byte swizzle (conflict-free row reads)
    alignas(64) CUtensorMap tmap_y;   // 2D fp32 [M][N] (row stride ldy), same box and swizzle
};

}  // namespace axq

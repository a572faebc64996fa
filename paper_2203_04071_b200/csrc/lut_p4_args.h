// lut_p4_args.h -- tile constants and launch arguments of the P4 kernel (lut_p4.cuh).
#pragma once
#include <cstdint>

#include "lut_mm.cuh"

namespace axq {

namespace p4 {
constexpr int TN = 16;                     // output columns per CTA tile (4 quads)
constexpr int WARPS = 16;
constexpr int NT = WARPS * 32;             // 512 threads
constexpr int RPL = 2;                     // rows per lane (lookups)
constexpr int BM = WARPS * 32 * RPL;       // 1024 rows per CTA tile
constexpr int KS = 16;                     // k per stage
constexpr int STAGES = 2;
constexpr int TBL_STAGE = KS * (TN / 4) * 1024;   // 64 KiB of E tables per stage
constexpr int A_STAGE = BM * KS;                  // 16 KiB activation tile per stage
constexpr int W_STAGE = TN * KS;                  // 256 B weight tile per stage
constexpr int SMEM_TBL = 0;
constexpr int SMEM_A = SMEM_TBL + STAGES * TBL_STAGE;
constexpr int SMEM_W = SMEM_A + STAGES * A_STAGE;
constexpr int SMEM_BAR = SMEM_W + STAGES * W_STAGE;
constexpr int SMEM_SCR = SMEM_BAR + 64;           // per-warp int32 [64 rows][16 cols] scratch
constexpr int SCR_WARP = 64 * TN * 4;
constexpr int SMEM_BYTES = SMEM_SCR + WARPS * SCR_WARP;
constexpr int FLUSH_STAGES = 16;                  // 16-bit packed E sums: flush every 256 k
constexpr int E_BIAS = 128;                       // tables hold E + 128 (unsigned bytes)
}  // namespace p4

struct P4Args {
    MMArgs mm;                  // geometry, loader info, t00, epilogue (k_split unused)
    const uint32_t* tables;     // [n_blocks][Kp][4][256] u32
    const int8_t* wpk;          // [n_blocks][Kp/16][16 n][16 k]
    int64_t Kp;                 // K rounded up to a multiple of 16
    int is_conv;
    uint32_t one;               // = 1 (opaque to the compiler: keeps the adds on the FMA pipe)
};

}  // namespace axq

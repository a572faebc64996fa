// wide_args.h -- launch arguments of the wide-ACU LUT-GEMM (wide.cuh, NEXT-2).
#pragma once
#include <cstdint>

#include "epilogue.cuh"

namespace axq {

struct WideArgs {
    const int16_t* A;       // [M][lda] codes
    int64_t lda;
    const int16_t* W;       // [N][ldw] codes
    int64_t ldw;
    int64_t M, N, K;
    int bits;
    const void* table;      // [uw][ua] (b-bit patterns): int16 E (delta16) or int32 LUT
    int delta16;
    int32_t* C_out;         // raw int32 [M][ldc] or null -> fused epilogue
    int64_t ldc;
    EpiArgs ep;
};

// packed weight-specialised wide LUT-GEMM (wide_pk.cuh)
struct WidePkArgs {
    const int16_t* A;        // [M][lda] codes
    int64_t lda;
    int64_t M, N, K, Kp;
    int bits;
    const uint2* tables;     // [N/TN][Kp][NQ][2^b] x 4 biased int16 E
    const int16_t* wts;      // [N/TN][Kp][NQ][4] weight codes (0 outside)
    int32_t t00;             // LUT[0][0] (a padded k's lookup)
    int32_t* C_out;          // raw int32 [M][ldc] or null -> fused epilogue
    int64_t ldc;
    EpiArgs ep;
};

}  // namespace axq

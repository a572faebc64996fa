// mm_launch.h -- host-side entry points of the LUT-MM kernel instantiations.
#pragma once
#include <cuda_runtime.h>

#include "lut_mm.cuh"

namespace axq {

struct Cfg {
    int warps, R, tn;
};
// BIG: 16 warps x 1 row per lane x 32 columns (512 x 32 CTA tile, one CTA per SM shares
// one table copy); SMALL: 4 warps x 1 x 32 (128 x 32).
constexpr Cfg CFG_BIG{16, 1, 32};
constexpr Cfg CFG_SMALL{4, 1, 32};

// Return 0 or a cudaError_t code.
int launch_mm_delta8(int epi, int loader, const MMArgs& p, const Cfg& c, dim3 grid, cudaStream_t st);
int launch_mm_i16(int epi, int loader, const MMArgs& p, const Cfg& c, dim3 grid, cudaStream_t st);
int launch_mm_i32(int epi, int loader, const MMArgs& p, const Cfg& c, dim3 grid, cudaStream_t st);

}  // namespace axq

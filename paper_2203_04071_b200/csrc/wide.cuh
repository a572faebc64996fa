// wide.cuh -- LUT-GEMM for wide ACUs (NEXT-2: b = 9..12 bits, the paper's 12-bit multipliers,
// P:237), int16 operand codes.
//
// acc[m][n] = sum_k LUT[a[m][k]][w[n][k]] (int32, exact), the table indexed by b-bit patterns.
// A b = 12 table has 2^24 entries: it cannot live in shared memory (64 MiB as int32, 32 MiB as
// the delta16 split LUT = a*w + E with E in int16), so it is read through L1/L2 -- the 126 MB
// L2 holds it whole -- with lanes = output rows sharing the weight: one gather touches one
// 2^b-entry table row (8 KiB at b = 12), which the 8 warps of a CTA tile reuse from L1.  This
// is the GPU face of the paper's observation that wider LUTs run slower (cache misses).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "epilogue.cuh"
#include "wide_args.h"

namespace axq {


namespace wide {
constexpr int NT = 256;     // 8 warps, one output row per lane
constexpr int TN = 16;      // columns per CTA tile
}

__global__ void __launch_bounds__(wide::NT) lut_wide_kernel(const WideArgs a) {
    using namespace wide;
    const int tid = threadIdx.x;
    const int64_t m_tiles = (a.M + NT - 1) / NT, n_tiles = (a.N + TN - 1) / TN;
    const uint32_t mask = (1u << a.bits) - 1u;
    const int16_t* t16 = reinterpret_cast<const int16_t*>(a.table);
    const int32_t* t32 = reinterpret_cast<const int32_t*>(a.table);
    float sc = 0.f, s_out = 1.f, qm = 127.f;
    if (!a.C_out) {
        sc = __fmul_rn(*a.ep.sa, *a.ep.sw);
        if (a.ep.q) {
            s_out = *a.ep.s_out;
            qm = (float)((1 << (a.ep.bits_out - 1)) - 1);
        }
    }
    for (int64_t tile = blockIdx.x; tile < m_tiles * n_tiles; tile += gridDim.x) {
        const int64_t n0 = (tile / m_tiles) * TN;      // column-major tiles: concurrent CTAs share
        const int64_t m = (tile % m_tiles) * NT + tid; // the same weight columns / table rows
        const bool valid = m < a.M;
        int acc[TN];
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[j] = 0;
        const int16_t* arow = a.A + (valid ? m : 0) * a.lda;
        for (int64_t k = 0; k < a.K; ++k) {
            const int av = valid ? (int)__ldg(arow + k) : 0;
            const uint32_t ua = (uint32_t)av & mask;
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int64_t n = n0 + j;
                const int wv = n < a.N ? (int)__ldg(a.W + n * a.ldw + k) : 0;
                const uint32_t idx = (((uint32_t)wv & mask) << a.bits) | ua;
                acc[j] += a.delta16 ? (int)__ldg(t16 + idx) + av * wv : __ldg(t32 + idx);
            }
        }
        if (!valid) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int64_t n = n0 + j;
            if (n >= a.N) continue;
            if (a.C_out) a.C_out[m * a.ldc + n] = acc[j];
            else epi_store(epi_value(acc[j], m, n, sc, a.ep), m, n, a.N, a.ep, s_out, qm);
        }
    }
}

// int16 codes: q = clamp(rint(fl(x / s))) with qmax = 2^(b-1) - 1 (O4 for b <= 16)
__global__ void quantize16_kernel(const float* __restrict__ x, int64_t n, const float* __restrict__ d_scale,
                                  int bits, int16_t* __restrict__ q) {
    const float s = *d_scale, qm = (float)((1 << (bits - 1)) - 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float t = div_rn_nz(x[i], s);
        t = fminf(fmaxf(t, -qm), qm);
        q[i] = (int16_t)__float2int_rn(t);
    }
}

}  // namespace axq

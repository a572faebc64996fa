// mm_launch.cuh -- template dispatch of lut_mm_kernel instantiations for one table
// representation (included once per representation .cu so they compile in parallel).
#pragma once
#include "mm_launch.h"

namespace axq {

template <int REPR, int TN, int R, int WARPS, int LOADER, int EPI, int WC = 1>
int launch_one(const MMArgs& p, dim3 grid, cudaStream_t st) {
    auto kern = lut_mm_kernel<REPR, TN, R, WARPS, LOADER, EPI, WC>;
    const int smem = (REPR == REPR_I32 ? 0 : REPR == REPR_I32H ? I32_HALF_BYTES : p.table_bytes) + 2 * (KC / 4) * TN * WC * 4 +
                     (LOADER == LOAD_CONV_C4 ? 4 * (MAX_TAP_GROUPS + 4) : 0);
    static unsigned configured = 0;  // bit per device
    static int resident[32] = {0};   // CTAs per SM, per device
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 31;
    if (!(configured & (1u << dev))) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return (int)e;
        int nb = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, WARPS * 32, smem);
        if (e != cudaSuccess) return (int)e;
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        resident[dev] = (nb > 0 ? nb : 1) * (sms > 0 ? sms : 148);
        configured |= 1u << dev;
    }
    // persistent grid: every CTA stages the table once and loops over the tiles
    const long long work = (long long)grid.x * grid.y * grid.z;
    const unsigned g = (unsigned)(work < resident[dev] ? work : resident[dev]);
    kern<<<g, WARPS * 32, smem, st>>>(p);
    return (int)cudaGetLastError();
}

// Byte-wise loaders (unaligned / tiny C) and the int32 table use only the SMALL tile.
template <int REPR, int LOADER, int EPI>
int launch_cfg(const MMArgs& p, const Cfg& c, dim3 grid, cudaStream_t st) {
    constexpr bool big_ok = (REPR != REPR_I32) && (LOADER == LOAD_GEMM || LOADER == LOAD_CONV || LOADER == LOAD_CONV_C4);
    if constexpr (big_ok) {
        if (c.wc == CFG_TINY.wc && c.warps == CFG_TINY.warps && LOADER == LOAD_GEMM)
            return launch_one<REPR, CFG_TINY.tn, CFG_TINY.R, CFG_TINY.warps, LOADER, EPI, CFG_TINY.wc>(p, grid, st);
        if (c.wc == CFG_SQ.wc && c.warps == CFG_SQ.warps && LOADER == LOAD_GEMM)
            return launch_one<REPR, CFG_SQ.tn, CFG_SQ.R, CFG_SQ.warps, LOADER, EPI, CFG_SQ.wc>(p, grid, st);
        if (c.wc == CFG_MID.wc && c.warps == CFG_MID.warps && LOADER == LOAD_GEMM)
            return launch_one<REPR, CFG_MID.tn, CFG_MID.R, CFG_MID.warps, LOADER, EPI, CFG_MID.wc>(p, grid, st);
        if (c.warps == CFG_BIG.warps && c.R == CFG_BIG.R && c.wc == 1)
            return launch_one<REPR, CFG_BIG.tn, CFG_BIG.R, CFG_BIG.warps, LOADER, EPI>(p, grid, st);
    }
    return launch_one<REPR, CFG_SMALL.tn, CFG_SMALL.R, CFG_SMALL.warps, LOADER, EPI>(p, grid, st);
}

template <int REPR, int EPI>
int launch_loader(int loader, const MMArgs& p, const Cfg& c, dim3 grid, cudaStream_t st) {
    switch (loader) {
        case LOAD_GEMM: return launch_cfg<REPR, LOAD_GEMM, EPI>(p, c, grid, st);
        case LOAD_GEMM_BYTES: return launch_cfg<REPR, LOAD_GEMM_BYTES, EPI>(p, c, grid, st);
        case LOAD_CONV: return launch_cfg<REPR, LOAD_CONV, EPI>(p, c, grid, st);
        case LOAD_CONV_C4: return launch_cfg<REPR, LOAD_CONV_C4, EPI>(p, c, grid, st);
        case LOAD_GEMM_F32: return launch_cfg<REPR, LOAD_GEMM_F32, EPI>(p, c, grid, st);
        case LOAD_CONV_F32: return launch_cfg<REPR, LOAD_CONV_F32, EPI>(p, c, grid, st);
        default: return launch_cfg<REPR, LOAD_CONV_BYTES, EPI>(p, c, grid, st);
    }
}

template <int REPR>
int launch_mm_repr(int epi, int loader, const MMArgs& p, const Cfg& c, dim3 grid, cudaStream_t st) {
    switch (epi) {
        case EPI_RAW: return launch_loader<REPR, EPI_RAW>(loader, p, c, grid, st);
        case EPI_RAW_ATOMIC: return launch_loader<REPR, EPI_RAW_ATOMIC>(loader, p, c, grid, st);
        default: return launch_loader<REPR, EPI_FUSED>(loader, p, c, grid, st);
    }
}

}  // namespace axq

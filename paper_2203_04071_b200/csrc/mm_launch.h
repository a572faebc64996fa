// mm_launch.h -- host-side entry points of the LUT-MM kernel instantiations.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>

#include "lut_mm.cuh"

namespace axq {

// LOAD_CONV_C4 keeps one 4-byte tap entry per 4 k in shared memory: K <= 4 * MAX_TAP_GROUPS.
constexpr int MAX_TAP_GROUPS = 1024;

struct Cfg {
    int warps, R, tn;
    int wc;        // warps along the columns (CTA tile 32R*(warps/wc) x wc*tn)
};
// BIG: 8 warps x 1 row per lane x 32 columns (256 x 32 CTA tile), two resident CTAs per SM
// (each with its own table copy) so one CTA's epilogue overlaps the other's lookups;
// SMALL: 4 warps x 1 x 32 (128 x 32).
constexpr Cfg CFG_BIG{8, 1, 32, 1};
constexpr Cfg CFG_SMALL{4, 1, 32, 1};
// TINY (M <= 64): 8 warps x 32 columns each over the same 64 rows (2 rows per lane).
constexpr Cfg CFG_TINY{8, 2, 32, 8};
// MID: 16 warps as 2 row groups x 8 column groups of 4 columns (64 x 32 CTA tile, whole K
// per tile).  Measured no faster than SMALL + K split on the 256-row linear layer of BJ
// configs[1] (86 vs 83 us), so pick_cfg does not select it; kept instantiated for A/B runs.
constexpr Cfg CFG_MID{16, 1, 4, 8};
// SQ (M <= 64 and N <= 64, e.g. BJ configs[0]): 4 warps as 2 x 2 over a 64 x 64 tile, K split
// down to one 16-k chunk per CTA, so a latency-bound small GEMM spreads over many SMs.
constexpr Cfg CFG_SQ{4, 1, 32, 2};

// Return 0 or a cudaError_t code.
int launch_mm_delta8(int epi, int loader, const MMArgs& p, const Cfg& c, dim3 grid, cudaStream_t st);
int launch_mm_i16(int epi, int loader, const MMArgs& p, const Cfg& c, dim3 grid, cudaStream_t st);
int launch_mm_i32(int epi, int loader, const MMArgs& p, const Cfg& c, dim3 grid, cudaStream_t st);
int launch_mm_i32h(int epi, int loader, const MMArgs& p, const Cfg& c, dim3 grid, cudaStream_t st);

// P4 kernel (lut_p4.cuh); declared here with an opaque argument struct.
struct P4Args;
int p4_pack(const int8_t* W, int64_t N, int64_t K, int64_t ldw, int64_t Kp, const int8_t* dtab,
            uint32_t* tables, int8_t* wpk, int half, int swap, cudaStream_t st);
int p4_pack_w(const int8_t* W, int64_t N, int64_t K, int64_t ldw, int64_t Kp, int8_t* wpk, cudaStream_t st);
int p4_pack16(const int8_t* W, int64_t N, int64_t K, int64_t ldw, int64_t Kp, const int16_t* e16,
              uint32_t* tables, cudaStream_t st);
int launch_p4(const P4Args& a, cudaStream_t st);
int launch_p4w(const P4Args& a, cudaStream_t st);
// P4W tile rows of a shape (cw consumer warps: 28 -> 896, 24 -> 768, 20 -> 640, 16 -> 512);
// launch_p4w serves cw = 16 for non-residual layers (full-range, or half-range 32-k tables),
// 20 / 24 for residual layers (half-range 32-k tables), 28 otherwise
int p4w_bm(int cw);
extern int g_p4w_pdl;   // warp-specialised P4T (lut_p4w.cuh)
struct LstmRecArgs;
struct GConvArgs;
struct WideArgs;
int launch_wide(const WideArgs& a, int sms, cudaStream_t st);   // wide.cuh (NEXT-2)
struct WidePkArgs;
int launch_widepk(const WidePkArgs& a, int sms, cudaStream_t st);   // wide_pk.cuh (NEXT-2 packed)
int widepk_tn(int bits);
int widepk_pack(const int16_t* W, int64_t N, int64_t K, int64_t ldw, int64_t Kp, int bits, const int16_t* e16,
                uint2* tables, int16_t* wts, int sms, cudaStream_t st);
int launch_quantize16(const float* x, int64_t n, const float* d_scale, int bits, int16_t* q, int sms,
                      cudaStream_t st);
int launch_gconv(int repr, const GConvArgs& a, cudaStream_t st);   // gconv.cuh (groups > 1)
int launch_lstm_rec(const LstmRecArgs& a, int sms, cudaStream_t st);   // lstm_rec.cuh
void p4w_plan(int64_t M, int64_t N, int64_t Kp, int ks, int bm, int sms, bool can_split, int& splits, int& sps);
void p4_plan(int64_t M, int64_t N, int64_t Kp, int sms, bool can_split, int& rpl, int& splits,
             int& sps);

}  // namespace axq

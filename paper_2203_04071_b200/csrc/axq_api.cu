// axq_api.cu -- the extern "C" boundary (include/axq.h): argument validation, ACU table
// representation, kernel selection and launch.  Compiled for sm_100a only.
#include "../../include/axq.h"

#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <vector>

#include "lut_p4_args.h"
#include "gconv.cuh"
#include "wide_args.h"
#include "wide_pk_geo.h"
#include "lstm_rec_args.h"
#include "mm_launch.h"
#include "glue_kernels.cuh"
#include "quant_kernels.cuh"

struct axq_wpack {
    int device;
    int half;
    int e16;                   // P4W16 tables (int16 E, 2 columns per packed word)
    int wide_bits;             // > 0: a wide (b = 9..12) pack for axq_lut_gemm16_wp
    int swap;                  // tables specialised on activations (axq_lut_gemm_xs)
    const int8_t* dtab;        // packing table: the LUT's [uw][ua] delta8 table, or (swap) a
                               // transposed [ua][uw] copy owned by the wpack (dtab_own)
    int8_t* dtab_own;
    int32_t t00;
    int64_t N, K, Kp;
    uint32_t* tables;
    int8_t* wpk;
    int64_t bytes;
};

struct axq_lut {
    int bits;
    int repr;
    int device;
    int32_t tmin, tmax, t00;
    int64_t absmax;
    void* d_table;
    int table_bytes;
    int16_t* d_e16;            // int16 E = LUT - a*w [uw8][ua8] when every E fits int16 and the
                               // table is not delta8 (feeds the P4W16 packer), else null
    int32_t* d_i32h;           // AXQ_LUT_I32: the table as two 128 KiB halves by the activation's
                               // high bit, [h][uw8][ua8 & 127] (lut_mm_kernel<REPR_I32H>), else null
    int i32_resident;          // AXQ_LUT_I32: 1 -> the SM-resident halves kernel, 0 -> L1 gather
};

namespace {

thread_local int g_last_cuda = 0;
thread_local int g_last_path = 0;   // axq_last_path: AXQ_PATH_* of the last LUT launch on this thread

inline axq_status cuda_fail(cudaError_t e) {
    g_last_cuda = (int)e;
    return AXQ_ERR_CUDA;
}

int sm_count();

inline axq_status check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e);
    return AXQ_OK;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
        cached[dev] = n;
    }
    return cached[dev];
}

int stream_grid(int64_t n_items, int per_block) {
    int64_t g = (n_items + per_block - 1) / per_block;
    int64_t cap = (int64_t)sm_count() * 8;
    return (int)std::max<int64_t>(1, std::min(g, cap));
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---------------------------------------------------------------------------------------
// LUT-MM launch plumbing (kernels are instantiated in mm_delta8.cu / mm_i16.cu / mm_i32.cu)
// ---------------------------------------------------------------------------------------
using axq::Cfg;
using axq::CFG_BIG;
using axq::CFG_SMALL;

// kernel representation beyond axq_lut_repr: the int32 table as SM-resident halves
constexpr int KREPR_I32H = 16;

axq_status launch_mm(int epi, int loader, int repr, const axq::MMArgs& p, const Cfg& c,
                     dim3 grid, cudaStream_t st) {
    int rc;
    switch (repr) {
        case AXQ_LUT_DELTA8: rc = axq::launch_mm_delta8(epi, loader, p, c, grid, st); break;
        case AXQ_LUT_I16: rc = axq::launch_mm_i16(epi, loader, p, c, grid, st); break;
        case KREPR_I32H: rc = axq::launch_mm_i32h(epi, loader, p, c, grid, st); break;
        default: rc = axq::launch_mm_i32(epi, loader, p, c, grid, st); break;
    }
    if (rc != 0) return cuda_fail((cudaError_t)rc);
    return AXQ_OK;
}

// Must agree with mm_launch.cuh::launch_cfg: byte-wise loaders and the int32 table only
// have the SMALL tile instantiated.
Cfg pick_cfg(int64_t M, int64_t N, int loader, int repr) {
    const bool big_ok = repr != AXQ_LUT_I32 &&
                        (loader == axq::LOAD_GEMM || loader == axq::LOAD_CONV || loader == axq::LOAD_CONV_C4);
    static int forced = -1;   // AXQ_V1_CFG (measurement switch): 1 SMALL, 2 BIG, 3 TINY, 4 MID
    if (forced < 0) {
        const char* v = std::getenv("AXQ_V1_CFG");
        forced = v ? std::atoi(v) : 0;
    }
    if (forced && big_ok && loader == axq::LOAD_GEMM) {
        if (forced == 2) return CFG_BIG;
        if (forced == 3) return axq::CFG_TINY;
        if (forced == 4) return axq::CFG_MID;
        return CFG_SMALL;
    }
    if (big_ok && loader == axq::LOAD_GEMM && M <= 64 && N <= 64) return axq::CFG_SQ;
    if (big_ok && loader == axq::LOAD_GEMM && M <= 64) return axq::CFG_TINY;
    return (M > 2048 && big_ok) ? CFG_BIG : CFG_SMALL;
}

inline int64_t cfg_bm(const Cfg& c) { return (int64_t)32 * c.R * (c.warps / c.wc); }
inline int64_t cfg_bn(const Cfg& c) { return (int64_t)c.tn * c.wc; }

// K-splitting so that small M*N problems still fill the SMs (exact: integer atomics).
int64_t pick_k_split(int64_t M, int64_t N, int64_t K, const Cfg& c, bool allow) {
    int64_t kr = ((K + axq::KC - 1) / axq::KC) * axq::KC;
    if (!allow || K <= 0) return std::max<int64_t>(kr, axq::KC);
    int64_t bm = cfg_bm(c);
    int64_t tiles = ((M + bm - 1) / bm) * ((N + cfg_bn(c) - 1) / cfg_bn(c));
    // 16-warp MID tiles: one wave of SMs suffices (no split from 3/4 of the SMs up)
    const bool mid = c.warps == axq::CFG_MID.warps && c.wc == axq::CFG_MID.wc;
    int64_t want = (int64_t)sm_count() * (mid ? 1 : 2);
    if (tiles >= (mid ? want * 3 / 4 : want)) return kr;
    int64_t splits = (want + tiles - 1) / tiles;
    // >= 64 k per split; the SQ tile (tiny GEMMs, latency-bound) down to one 16-k chunk
    const bool sq = c.warps == axq::CFG_SQ.warps && c.wc == axq::CFG_SQ.wc;
    int64_t max_splits = std::max<int64_t>(1, kr / ((sq ? 1 : 4) * axq::KC));
    splits = std::min(splits, max_splits);
    int64_t ks = (kr + splits - 1) / splits;
    ks = ((ks + axq::KC - 1) / axq::KC) * axq::KC;
    return std::max<int64_t>(ks, axq::KC);
}

axq_status check_lut(axq_lut_t lut) {
    if (!lut || !lut->d_table) return AXQ_ERR_INVALID;
    if (lut->bits > 8) return AXQ_ERR_UNSUPPORTED;   // wide tables: axq_lut_gemm16 only
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != lut->device) return AXQ_ERR_INVALID;
    return AXQ_OK;
}

axq_status overflow_guard(axq_lut_t lut, int64_t K) {
    // int32 accumulation is exact iff every partial sum fits; K * max|T| < 2^31 suffices.
    if (K > 0 && (double)K * (double)lut->absmax >= 2147483648.0) return AXQ_ERR_OVERFLOW;
    return AXQ_OK;
}

void fill_common(axq::MMArgs& p, axq_lut_t lut) {
    p.table = lut->d_table;
    p.table_bytes = lut->table_bytes;
    p.t00 = lut->t00;
}

}  // namespace

extern "C" {

int axq_last_cuda_error(void) { return g_last_cuda; }

const char* axq_status_string(axq_status s) {
    switch (s) {
        case AXQ_OK: return "ok";
        case AXQ_ERR_INVALID: return "invalid argument";
        case AXQ_ERR_OVERFLOW: return "int32 accumulator could overflow (K * max|LUT| >= 2^31)";
        case AXQ_ERR_UNSUPPORTED: return "unsupported case";
        case AXQ_ERR_CUDA: return "CUDA error";
    }
    return "unknown status";
}

int axq_version(void) { return 100; }

// ---------------------------------------------------------------------------------------
// ACU table
// ---------------------------------------------------------------------------------------
// NEXT-2: wide ACUs (b = 9..12).  Device layout [uw][ua] in the b-bit pattern space; int16 E =
// LUT - a*w when every E fits (delta16), else int32 LUT values.
static axq_status lut_create_wide(int bits, const int32_t* host_table, axq_lut_t* out) {
    const int64_t n = (int64_t)1 << bits, mask = n - 1;
    int64_t tmin = INT32_MAX, tmax = INT32_MIN;
    bool d16 = true;
    for (int64_t ua = 0; ua < n; ++ua)
        for (int64_t uw = 0; uw < n; ++uw) {
            const int64_t v = host_table[(ua << bits) | uw];
            tmin = std::min(tmin, v);
            tmax = std::max(tmax, v);
            const int64_t a = ua >= n / 2 ? ua - n : ua, w = uw >= n / 2 ? uw - n : uw;
            const int64_t e = v - a * w;
            if (e < INT16_MIN || e > INT16_MAX) d16 = false;
        }
    const int esz = d16 ? 2 : 4;
    std::vector<uint8_t> dev_tab((size_t)(n * n) * esz);
    for (int64_t uw = 0; uw < n; ++uw)
        for (int64_t ua = 0; ua < n; ++ua) {
            const int64_t a = ua >= n / 2 ? ua - n : ua, w = uw >= n / 2 ? uw - n : uw;
            const int32_t v = host_table[(ua << bits) | uw];
            const size_t idx = (size_t)((uw << bits) | ua);
            if (d16) {
                const int16_t e = (int16_t)(v - a * w);
                std::memcpy(&dev_tab[idx * 2], &e, 2);
            } else {
                std::memcpy(&dev_tab[idx * 4], &v, 4);
            }
        }
    (void)mask;
    axq_lut* L = new axq_lut();
    L->bits = bits;
    L->repr = d16 ? AXQ_LUT_WIDE16 : AXQ_LUT_WIDE32;
    cudaGetDevice(&L->device);
    L->tmin = (int32_t)tmin;
    L->tmax = (int32_t)tmax;
    L->t00 = host_table[0];
    L->absmax = std::max<int64_t>(std::llabs(tmin), std::llabs(tmax));
    L->table_bytes = (int)std::min<size_t>(dev_tab.size(), (size_t)INT32_MAX);
    cudaError_t e = cudaMalloc(&L->d_table, dev_tab.size());
    if (e == cudaSuccess) e = cudaMemcpy(L->d_table, dev_tab.data(), dev_tab.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        if (L->d_table) cudaFree(L->d_table);
        delete L;
        return cuda_fail(e);
    }
    *out = L;
    return AXQ_OK;
}

axq_status axq_lut_create(int bits, const int32_t* host_table, axq_lut_t* out) {
    if (!out || !host_table || bits < 2 || bits > 12) return AXQ_ERR_INVALID;
    *out = nullptr;
    if (bits > 8) return lut_create_wide(bits, host_table, out);
    const int n = 1 << bits, mask = n - 1;
    int64_t tmin = INT32_MAX, tmax = INT32_MIN;
    bool delta_ok = true;
    for (int ua = 0; ua < n; ++ua) {
        for (int uw = 0; uw < n; ++uw) {
            int64_t v = host_table[(ua << bits) | uw];
            tmin = std::min(tmin, v);
            tmax = std::max(tmax, v);
            int a = (ua >= n / 2) ? ua - n : ua, w = (uw >= n / 2) ? uw - n : uw;
            int64_t e = v - (int64_t)a * w;
            if (e < -128 || e > 127) delta_ok = false;
        }
    }
    int repr = delta_ok ? AXQ_LUT_DELTA8
                        : (tmin >= INT16_MIN && tmax <= INT16_MAX) ? AXQ_LUT_I16 : AXQ_LUT_I32;
    const int esz = repr == AXQ_LUT_DELTA8 ? 1 : repr == AXQ_LUT_I16 ? 2 : 4;
    // Device layout: 8-bit two's-complement pattern space, TRANSPOSED: entry [uw8][ua8].
    // Patterns that are not sign-extended b-bit codes are never produced by the quantizer
    // and hold 0.
    std::vector<uint8_t> dev_tab((size_t)65536 * esz, 0);
    for (int uw8 = 0; uw8 < 256; ++uw8) {
        int w = (int)(int8_t)uw8;
        if (w < -(n / 2) || w >= n / 2) continue;
        for (int ua8 = 0; ua8 < 256; ++ua8) {
            int a = (int)(int8_t)ua8;
            if (a < -(n / 2) || a >= n / 2) continue;
            int32_t v = host_table[((a & mask) << bits) | (w & mask)];
            size_t idx = ((size_t)uw8 << 8) | (size_t)ua8;
            if (repr == AXQ_LUT_DELTA8) {
                dev_tab[idx] = (uint8_t)(int8_t)(v - a * w);
            } else if (repr == AXQ_LUT_I16) {
                int16_t s = (int16_t)v;
                std::memcpy(&dev_tab[idx * 2], &s, 2);
            } else {
                std::memcpy(&dev_tab[idx * 4], &v, 4);
            }
        }
    }
    axq_lut* L = new axq_lut();
    L->bits = bits;
    L->repr = repr;
    L->d_e16 = nullptr;
    L->d_i32h = nullptr;
    L->i32_resident = 0;
    cudaGetDevice(&L->device);
    if (repr != AXQ_LUT_DELTA8) {
        // E16 copy for the packed int16-E kernel (P4W16): E = LUT - a*w within int16
        bool e16_ok = true;
        std::vector<int16_t> e16((size_t)65536, 0);
        for (int uw8 = 0; uw8 < 256 && e16_ok; ++uw8) {
            const int w = (int)(int8_t)uw8;
            if (w < -(n / 2) || w >= n / 2) continue;
            for (int ua8 = 0; ua8 < 256; ++ua8) {
                const int a = (int)(int8_t)ua8;
                if (a < -(n / 2) || a >= n / 2) continue;
                const int64_t ev = (int64_t)host_table[((a & mask) << bits) | (w & mask)] - (int64_t)a * w;
                if (ev < INT16_MIN || ev > INT16_MAX) { e16_ok = false; break; }
                e16[((size_t)uw8 << 8) | (size_t)ua8] = (int16_t)ev;
            }
        }
        if (e16_ok) {
            cudaError_t e = cudaMalloc(&L->d_e16, 131072);
            if (e == cudaSuccess) e = cudaMemcpy(L->d_e16, e16.data(), 131072, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) {
                if (L->d_e16) cudaFree(L->d_e16);
                delete L;
                return cuda_fail(e);
            }
        }
    }
    L->tmin = (int32_t)tmin;
    L->tmax = (int32_t)tmax;
    L->t00 = host_table[0];
    L->absmax = std::max<int64_t>(std::llabs(tmin), std::llabs(tmax));
    L->table_bytes = 65536 * esz;
    cudaError_t e = cudaMalloc(&L->d_table, L->table_bytes);
    if (e != cudaSuccess) {
        delete L;
        return cuda_fail(e);
    }
    e = cudaMemcpy(L->d_table, dev_tab.data(), L->table_bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && repr == AXQ_LUT_I32) {
        // halves by the activation's high bit: entry [uw8][ua8] -> [ua8 >> 7][uw8][ua8 & 127]
        std::vector<int32_t> h((size_t)65536);
        const int32_t* t = reinterpret_cast<const int32_t*>(dev_tab.data());
        for (int uw8 = 0; uw8 < 256; ++uw8)
            for (int ua8 = 0; ua8 < 256; ++ua8)
                h[((size_t)(ua8 >> 7) << 15) | ((size_t)uw8 << 7) | (size_t)(ua8 & 127)] =
                    t[((size_t)uw8 << 8) | (size_t)ua8];
        e = cudaMalloc(&L->d_i32h, 262144);
        if (e == cudaSuccess) e = cudaMemcpy(L->d_i32h, h.data(), 262144, cudaMemcpyHostToDevice);
        static const int resident_default = [] {
            const char* v = std::getenv("AXQ_I32_RESIDENT");   // measurement switch
            return v ? std::atoi(v) : 0;
        }();
        L->i32_resident = resident_default;
    }
    if (e != cudaSuccess) {
        cudaFree(L->d_table);
        if (L->d_i32h) cudaFree(L->d_i32h);
        if (L->d_e16) cudaFree(L->d_e16);
        delete L;
        return cuda_fail(e);
    }
    *out = L;
    return AXQ_OK;
}

axq_status axq_lut_destroy(axq_lut_t lut) {
    if (!lut) return AXQ_OK;
    cudaDeviceSynchronize();
    cudaFree(lut->d_table);
    if (lut->d_e16) cudaFree(lut->d_e16);
    if (lut->d_i32h) cudaFree(lut->d_i32h);
    delete lut;
    return AXQ_OK;
}

axq_status axq_lut_set_i32_resident(axq_lut_t lut, int resident) {
    if (!lut) return AXQ_ERR_INVALID;
    if (lut->repr != AXQ_LUT_I32) return AXQ_ERR_UNSUPPORTED;
    lut->i32_resident = resident ? 1 : 0;
    return AXQ_OK;
}

axq_status axq_lut_info(axq_lut_t lut, int* bits, int* repr, int32_t* tmin, int32_t* tmax) {
    if (!lut) return AXQ_ERR_INVALID;
    if (bits) *bits = lut->bits;
    if (repr) *repr = lut->repr;
    if (tmin) *tmin = lut->tmin;
    if (tmax) *tmax = lut->tmax;
    return AXQ_OK;
}

// ---------------------------------------------------------------------------------------
// Quantizer
// ---------------------------------------------------------------------------------------
axq_status axq_amax(const float* x, int64_t n, float* d_amax, void* stream) {
    if (n < 0 || !d_amax || (n > 0 && !x)) return AXQ_ERR_INVALID;
    cudaError_t e = cudaMemsetAsync(d_amax, 0, sizeof(float), S(stream));
    if (e != cudaSuccess) return cuda_fail(e);
    if (n == 0) return AXQ_OK;
    axq::amax_kernel<<<stream_grid(n / 4 + 1, 256 * 4), 256, 0, S(stream)>>>(
        x, n, reinterpret_cast<unsigned int*>(d_amax));
    return check_launch();
}

axq_status axq_scale(const float* d_amax, int bits, float* d_scale, void* stream) {
    if (!d_amax || !d_scale || bits < 2 || bits > 16) return AXQ_ERR_INVALID;
    axq::scale_kernel<<<1, 1, 0, S(stream)>>>(d_amax, bits, d_scale);
    return check_launch();
}

// ---- NEXT-1: the paper's quantizer (A30-A32) ----
axq_status axq_amax_rows(const float* W, int64_t rows, int64_t cols, float* d_amax, void* stream) {
    if (rows < 0 || cols < 0 || (rows > 0 && (!W || !d_amax))) return AXQ_ERR_INVALID;
    if (rows == 0) return AXQ_OK;
    if (cols == 0) return cudaMemsetAsync(d_amax, 0, rows * sizeof(float), S(stream)) == cudaSuccess ? AXQ_OK : AXQ_ERR_CUDA;
    axq::amax_rows_kernel<<<(unsigned)std::min<int64_t>(rows, 148 * 8), 256, 0, S(stream)>>>(W, rows, cols, d_amax);
    return check_launch();
}

axq_status axq_scale_vec(const float* d_amax, int64_t n, int bits, float* d_scale, void* stream) {
    if (n < 0 || bits < 2 || bits > 8 || (n > 0 && (!d_amax || !d_scale))) return AXQ_ERR_INVALID;
    if (n == 0) return AXQ_OK;
    axq::scale_vec_kernel<<<stream_grid(n, 256), 256, 0, S(stream)>>>(d_amax, n, bits, d_scale);
    return check_launch();
}

axq_status axq_quantize_rows(const float* W, int64_t rows, int64_t cols, const float* d_scale_rows,
                             int bits, int8_t* q, void* stream) {
    if (rows < 0 || cols < 0 || bits < 2 || bits > 8) return AXQ_ERR_INVALID;
    if (rows == 0 || cols == 0) return AXQ_OK;
    if (!W || !d_scale_rows || !q) return AXQ_ERR_INVALID;
    axq::quantize_rows_kernel<<<stream_grid(rows * cols, 256 * 4), 256, 0, S(stream)>>>(W, rows, cols, d_scale_rows,
                                                                                    bits, q);
    return check_launch();
}

axq_status axq_calib_histogram(const float* x, int64_t n, const float* d_amax, int bins,
                               uint32_t* d_hist, void* stream) {
    if (n < 0 || bins < 1 || bins > 8192 || !d_amax || !d_hist || (n > 0 && !x)) return AXQ_ERR_INVALID;
    cudaError_t e = cudaMemsetAsync(d_hist, 0, (size_t)bins * sizeof(uint32_t), S(stream));
    if (e != cudaSuccess) return cuda_fail(e);
    if (n == 0) return AXQ_OK;
    const int copies = bins <= 2048 ? 8 : (bins <= 4096 ? 4 : 2);   // per-warp sub-histograms
    const size_t sm = (size_t)bins * copies * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(axq::hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        attr = true;
    }
    axq::hist_kernel<<<stream_grid(n / 4 + 1, 256 * 8), 256, sm, S(stream)>>>(x, n, d_amax, bins, copies, d_hist);
    return check_launch();
}

axq_status axq_calib_percentile(const uint32_t* d_hist, int bins, int64_t n, const float* d_amax,
                                int64_t p_num, int64_t p_den, int bits, float* d_calib_max,
                                float* d_scale, void* stream) {
    if (!d_hist || bins < 1 || n < 0 || !d_amax || p_num < 0 || p_den <= 0 || p_num > p_den ||
        bits < 2 || bits > 8 || (!d_calib_max && !d_scale))
        return AXQ_ERR_INVALID;
    axq::percentile_kernel<<<1, 1024, 0, S(stream)>>>(d_hist, bins, n, d_amax, p_num, p_den, bits, d_calib_max,
                                                    d_scale);
    return check_launch();
}

axq_status axq_quantize(const float* x, int64_t n, const float* d_scale, int bits, int8_t* q,
                        void* stream) {
    if (n < 0 || !d_scale || bits < 2 || bits > 8 || (n > 0 && (!x || !q))) return AXQ_ERR_INVALID;
    if (n == 0) return AXQ_OK;
    axq::quantize_kernel<<<stream_grid(n / 4 + 1, 256 * 4), 256, 0, S(stream)>>>(x, n, d_scale, bits, q);
    return check_launch();
}

axq_status axq_quantize_nchw_to_nhwc(const float* x, int64_t N, int64_t C, int64_t H, int64_t W,
                                     int64_t Cq, const float* d_scale, int bits, int8_t* q,
                                     void* stream) {
    if (N < 0 || C < 0 || H < 0 || W < 0 || Cq < C || !d_scale || bits < 2 || bits > 8)
        return AXQ_ERR_INVALID;
    if (N == 0 || Cq == 0 || H == 0 || W == 0) return AXQ_OK;
    if (!x || !q || N > 65535) return AXQ_ERR_INVALID;
    const int64_t HW = H * W;
    if (Cq == 4 && C <= 4 && N * HW < ((int64_t)1 << 30) && (reinterpret_cast<uintptr_t>(q) & 3) == 0) {
        axq::quantize_nchw_to_nhwc_c4_kernel<<<stream_grid(N * HW, 256), 256, 0, S(stream)>>>(
            x, (int)C, (int)HW, (int)(N * HW), d_scale, bits, q);
    } else if (Cq <= 16) {  // few channels (network input): one pixel per thread
        axq::quantize_nchw_to_nhwc_small_kernel<<<stream_grid(N * HW, 256), 256, 0, S(stream)>>>(
            x, N, C, HW, Cq, d_scale, bits, q);
    } else {
        dim3 grid((unsigned)((HW + 63) / 64), (unsigned)((Cq + 63) / 64), (unsigned)N);
        axq::quantize_nchw_to_nhwc_kernel<<<grid, 256, 0, S(stream)>>>(x, C, HW, Cq, d_scale, bits, q);
    }
    return check_launch();
}

// ---------------------------------------------------------------------------------------
// LUT-GEMM
// ---------------------------------------------------------------------------------------
static axq_status gemm_common(int64_t M, int64_t N, int64_t K, const int8_t* A, int64_t lda,
                              const int8_t* W, int64_t ldw, axq_lut_t lut) {
    if (M < 0 || N < 0 || K < 0) return AXQ_ERR_INVALID;
    axq_status s = check_lut(lut);
    if (s != AXQ_OK) return s;
    if (M > 0 && N > 0 && K > 0) {
        if (!A || !W || lda < K || ldw < K) return AXQ_ERR_INVALID;
    }
    return overflow_guard(lut, K);
}

// The caller's epilogue workspace if it can hold `need` int32 elements (split-K accumulators),
// else null (no K split).  workspace_elems == 0 means "M*N", the documented minimum.
static int32_t* ws_if_fits(const axq_epilogue* ep, int64_t need) {
    if (!ep || !ep->workspace) return nullptr;
    if (ep->workspace_elems > 0 && ep->workspace_elems < need) return nullptr;
    return ep->workspace;
}

static axq_status check_epilogue(const axq_epilogue* ep, int64_t N, bool conv) {
    if (!ep || !ep->d_scale_a || !ep->d_scale_w) return AXQ_ERR_INVALID;
    const bool rows = !conv || ep->y_nhwc;
    if (ep->y && rows && ep->ldy < N) return AXQ_ERR_INVALID;
    if (ep->residual && (ep->ldr < N || (conv && !ep->y_nhwc && ep->y))) return AXQ_ERR_INVALID;
    if (ep->q_out && (ep->ldq < N || !ep->d_scale_out || ep->bits_out < 2 || ep->bits_out > 8))
        return AXQ_ERR_INVALID;
    return AXQ_OK;
}

static axq::EpiArgs to_epi(const axq_epilogue* ep, bool nchw, int64_t hw) {
    axq::EpiArgs e{};
    e.sa = ep->d_scale_a;
    e.sw = ep->d_scale_w;
    e.sw_ch = ep->d_scale_w_ch;
    e.bias = ep->bias;
    e.residual = ep->residual;
    e.ldr = ep->ldr;
    e.relu = ep->relu;
    e.y = ep->y;
    e.ldy = ep->ldy;
    e.y_nchw = nchw ? 1 : 0;
    e.hw = hw;
    e.q = ep->q_out;
    e.ldq = ep->ldq;
    e.s_out = ep->d_scale_out;
    e.bits_out = ep->bits_out;
    return e;
}

static axq_status launch_epilogue(int64_t M, int64_t N, const int32_t* acc, int64_t ldacc,
                                  const axq::EpiArgs& e, cudaStream_t st, int32_t* zero_acc = nullptr) {
    axq::epilogue_kernel<<<stream_grid(M * N, 256 * 4), 256, 0, st>>>(M, N, acc, ldacc, e, zero_acc);
    return check_launch();
}

// Common driver: plan split-K, launch the fused or the split (atomic + epilogue) variant.
static axq_status run_mm(axq::MMArgs& p, int loader, axq_lut_t lut, const axq::EpiArgs* epi,
                         int32_t* workspace, int32_t* C_raw, int64_t ldc, cudaStream_t st) {
    int krepr = lut->repr;
    if (krepr == AXQ_LUT_I32 && lut->i32_resident && lut->d_i32h) {
        krepr = KREPR_I32H;
        p.table = lut->d_i32h;
    }
    Cfg c = pick_cfg(p.M, p.N, loader, krepr);
    const bool can_split = epi ? (workspace != nullptr) : true;
    p.k_split = pick_k_split(p.M, p.N, p.K, c, can_split);
    const int64_t splits = p.K > 0 ? (p.K + p.k_split - 1) / p.k_split : 1;
    const int64_t bm = cfg_bm(c), bn = cfg_bn(c);
    dim3 grid((unsigned)((p.M + bm - 1) / bm), (unsigned)((p.N + bn - 1) / bn), (unsigned)splits);
    g_last_path = AXQ_PATH_V1 | (splits > 1 ? AXQ_PATH_SPLITK : 0);
    if (!epi) {
        p.C_out = C_raw;
        p.ldc = ldc;
        if (splits > 1) {
            cudaError_t e = cudaMemset2DAsync(C_raw, ldc * 4, 0, p.N * 4, p.M, st);
            if (e != cudaSuccess) return cuda_fail(e);
            return launch_mm(axq::EPI_RAW_ATOMIC, loader, krepr, p, c, grid, st);
        }
        return launch_mm(axq::EPI_RAW, loader, krepr, p, c, grid, st);
    }
    if (splits > 1) {
        p.C_out = workspace;
        p.ldc = p.N;
        cudaError_t e = cudaMemsetAsync(workspace, 0, (size_t)p.M * p.N * 4, st);
        if (e != cudaSuccess) return cuda_fail(e);
        axq_status s = launch_mm(axq::EPI_RAW_ATOMIC, loader, krepr, p, c, grid, st);
        if (s != AXQ_OK) return s;
        return launch_epilogue(p.M, p.N, workspace, p.N, *epi, st, workspace);
    }
    p.ep = *epi;
    return launch_mm(axq::EPI_FUSED, loader, krepr, p, c, grid, st);
}

axq_status axq_lut_gemm(int64_t M, int64_t N, int64_t K, const int8_t* A, int64_t lda,
                        const int8_t* W, int64_t ldw, axq_lut_t lut, int32_t* C, int64_t ldc,
                        void* stream) {
    axq_status s = gemm_common(M, N, K, A, lda, W, ldw, lut);
    if (s != AXQ_OK) return s;
    if (M == 0 || N == 0) return AXQ_OK;
    if (!C || ldc < N) return AXQ_ERR_INVALID;
    if (K == 0) {
        cudaError_t e = cudaMemset2DAsync(C, ldc * 4, 0, N * 4, M, S(stream));
        return e == cudaSuccess ? AXQ_OK : cuda_fail(e);
    }
    axq::MMArgs p{};
    p.A = A; p.lda = lda; p.W = W; p.ldw = ldw; p.M = M; p.N = N; p.K = K;
    fill_common(p, lut);
    int loader = (aligned16(A) && (lda & 15) == 0) ? axq::LOAD_GEMM : axq::LOAD_GEMM_BYTES;
    return run_mm(p, loader, lut, nullptr, nullptr, C, ldc, S(stream));
}

axq_status axq_lut_gemm_dq(int64_t M, int64_t N, int64_t K, const int8_t* A, int64_t lda,
                           const int8_t* W, int64_t ldw, axq_lut_t lut, const axq_epilogue* ep,
                           void* stream) {
    axq_status s = gemm_common(M, N, K, A, lda, W, ldw, lut);
    if (s != AXQ_OK) return s;
    s = check_epilogue(ep, N, false);
    if (s != AXQ_OK) return s;
    if (M == 0 || N == 0) return AXQ_OK;
    axq::MMArgs p{};
    p.A = A; p.lda = lda; p.W = W; p.ldw = ldw; p.M = M; p.N = N; p.K = K;
    fill_common(p, lut);
    axq::EpiArgs e = to_epi(ep, false, 0);
    int loader = (aligned16(A) && (lda & 15) == 0) ? axq::LOAD_GEMM : axq::LOAD_GEMM_BYTES;
    return run_mm(p, loader, lut, &e, ws_if_fits(ep, p.M * p.N), nullptr, 0, S(stream));
}

// ---------------------------------------------------------------------------------------
// LUT convolution (implicit im2col)
// ---------------------------------------------------------------------------------------
axq_status axq_conv2d_out_hw(const axq_conv_desc* d, int64_t* Ho, int64_t* Wo) {
    if (!d || !Ho || !Wo) return AXQ_ERR_INVALID;
    if (d->stride_h <= 0 || d->stride_w <= 0 || d->dil_h <= 0 || d->dil_w <= 0 || d->pad_h < 0 ||
        d->pad_w < 0 || d->R <= 0 || d->S <= 0)
        return AXQ_ERR_INVALID;
    *Ho = (d->H + 2 * d->pad_h - d->dil_h * (d->R - 1) - 1) / d->stride_h + 1;
    *Wo = (d->W + 2 * d->pad_w - d->dil_w * (d->S - 1) - 1) / d->stride_w + 1;
    return AXQ_OK;
}

// groups > 1 (NEXT-3): grouped / depthwise conv on the resident-table kernel (gconv.cuh)
static axq_status gconv_run(const axq_conv_desc* d, const int8_t* X, const int8_t* Wt, axq_lut_t lut,
                            const axq_epilogue* ep, int32_t* Y, cudaStream_t st) {
    if (d->groups < 1 || d->C % d->groups || d->K % d->groups) return AXQ_ERR_INVALID;
    if (d->c_valid != 0 && d->c_valid != d->C) return AXQ_ERR_UNSUPPORTED;
    int64_t Ho, Wo;
    axq_status s = axq_conv2d_out_hw(d, &Ho, &Wo);
    if (s != AXQ_OK) return s;
    if (Ho <= 0 || Wo <= 0) return AXQ_ERR_INVALID;
    s = check_lut(lut);
    if (s != AXQ_OK) return s;
    s = overflow_guard(lut, d->R * d->S * (d->C / d->groups));
    if (s != AXQ_OK) return s;
    if (d->N > 0 && d->K > 0 && (!X || !Wt)) return AXQ_ERR_INVALID;
    if (d->H * d->W * d->C >= (int64_t)1 << 31 || Ho * Wo >= (int64_t)1 << 31) return AXQ_ERR_INVALID;
    if (d->N * Ho * Wo >= (int64_t)1 << 31) return AXQ_ERR_UNSUPPORTED;   // 32-bit pixel indexing
    axq::GConvArgs a{};
    a.X = X; a.W = Wt; a.M = d->N * Ho * Wo;
    a.N = (int)d->N; a.H = (int)d->H; a.Wd = (int)d->W; a.C = (int)d->C; a.K = (int)d->K;
    a.R = (int)d->R; a.S = (int)d->S; a.G = (int)d->groups; a.Ho = (int)Ho; a.Wo = (int)Wo;
    a.sh = (int)d->stride_h; a.sw = (int)d->stride_w; a.ph = (int)d->pad_h; a.pw = (int)d->pad_w;
    a.dh = (int)d->dil_h; a.dw = (int)d->dil_w;
    a.table = lut->d_table;
    a.table_bytes = lut->table_bytes;
    if (ep) {
        s = check_epilogue(ep, d->K, true);
        if (s != AXQ_OK) return s;
        a.ep = to_epi(ep, !ep->y_nhwc, Ho * Wo);
        a.C_out = nullptr;
    } else {
        if (!Y) return AXQ_ERR_INVALID;
        a.C_out = Y;
    }
    if (a.M == 0 || a.K == 0) return AXQ_OK;
    const int64_t cin_g = d->C / d->groups, cout_g = d->K / d->groups;
    if (cin_g % 4 == 0 && cin_g >= 16 && lut->repr != AXQ_LUT_I32 &&
        (reinterpret_cast<uintptr_t>(X) & 3) == 0) {
        // wide groups: one dense implicit-im2col LUT-GEMM per group on the v1 kernel, the group's
        // channels addressed through the pixel stride (cs) and the outputs through offsets
        const int64_t Kg = d->R * d->S * cin_g, hw = Ho * Wo;
        for (int64_t g = 0; g < d->groups; ++g) {
            axq::MMArgs p{};
            p.A = X + g * cin_g; p.lda = 0; p.W = Wt + g * cout_g * Kg; p.ldw = Kg;
            p.M = a.M; p.N = cout_g; p.K = Kg;
            p.H = a.H; p.Wd = a.Wd; p.C = (int)cin_g; p.cs = a.C; p.Ho = a.Ho; p.Wo = a.Wo;
            p.S = a.S; p.sh = a.sh; p.sw = a.sw; p.ph = a.ph; p.pw = a.pw; p.dh = a.dh; p.dw = a.dw;
            fill_common(p, lut);
            const int loader = (cin_g % 16 == 0 && aligned16(X) && (a.C % 16) == 0) ? axq::LOAD_CONV
                             : (Kg <= 4 * axq::MAX_TAP_GROUPS && d->R * d->dil_h < 256 && d->S * d->dil_w < 256)
                                   ? axq::LOAD_CONV_C4 : axq::LOAD_CONV_BYTES;
            axq_status r;
            if (ep) {
                axq::EpiArgs e = a.ep;
                const int64_t off = g * cout_g;
                if (e.y) e.y += e.y_nchw ? off * hw : off;
                if (e.y_nchw) e.nchw_ld = d->K;
                if (e.bias) e.bias += off;
                if (e.residual) e.residual += off;
                if (e.q) e.q += off;
                if (e.sw_ch) e.sw_ch += off;
                r = run_mm(p, loader, lut, &e, ws_if_fits(ep, p.M * p.N), nullptr, 0, st);
            } else {
                r = run_mm(p, loader, lut, nullptr, nullptr, Y + g * cout_g, d->K, st);
            }
            if (r != AXQ_OK) return r;
        }
        return AXQ_OK;
    }
    g_last_path = AXQ_PATH_GCONV;
    const int rc = axq::launch_gconv(lut->repr, a, st);
    return rc ? cuda_fail((cudaError_t)rc) : AXQ_OK;
}

static axq_status conv_setup(const axq_conv_desc* d, const int8_t* X, const int8_t* Wt,
                             axq_lut_t lut, axq::MMArgs& p, int& loader) {
    if (!d) return AXQ_ERR_INVALID;
    if (d->N < 0 || d->H <= 0 || d->W <= 0 || d->C <= 0 || d->K < 0) return AXQ_ERR_INVALID;
    if (d->c_valid < 0 || d->c_valid > d->C) return AXQ_ERR_INVALID;
    if (d->groups != 1) return d->groups < 1 ? AXQ_ERR_INVALID : AXQ_ERR_UNSUPPORTED;
    int64_t Ho, Wo;
    axq_status s = axq_conv2d_out_hw(d, &Ho, &Wo);
    if (s != AXQ_OK) return s;
    if (Ho <= 0 || Wo <= 0) return AXQ_ERR_INVALID;
    s = check_lut(lut);
    if (s != AXQ_OK) return s;
    const int64_t K = d->R * d->S * d->C;
    const int64_t cv = d->c_valid ? d->c_valid : d->C;
    s = overflow_guard(lut, d->R * d->S * cv);
    if (s != AXQ_OK) return s;
    if (d->N > 0 && d->K > 0 && (!X || !Wt)) return AXQ_ERR_INVALID;
    if (d->H * d->W * d->C >= (int64_t)1 << 31 || Ho * Wo >= (int64_t)1 << 31) return AXQ_ERR_INVALID;
    p = axq::MMArgs{};
    p.A = X; p.lda = 0; p.W = Wt; p.ldw = K;
    p.M = d->N * Ho * Wo; p.N = d->K; p.K = K;
    p.H = (int)d->H; p.Wd = (int)d->W; p.C = (int)d->C; p.Ho = (int)Ho; p.Wo = (int)Wo;
    p.S = (int)d->S; p.sh = (int)d->stride_h; p.sw = (int)d->stride_w;
    p.ph = (int)d->pad_h; p.pw = (int)d->pad_w; p.dh = (int)d->dil_h; p.dw = (int)d->dil_w;
    fill_common(p, lut);
    p.pad_lookups = (int32_t)(d->R * d->S * (d->C - cv));
    if ((d->C & 15) == 0 && aligned16(X))
        loader = axq::LOAD_CONV;
    else if ((d->C & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 3) == 0 &&
             K <= 4 * axq::MAX_TAP_GROUPS && d->R * d->dil_h < 256 && d->S * d->dil_w < 256)
        loader = axq::LOAD_CONV_C4;
    else
        loader = axq::LOAD_CONV_BYTES;
    return AXQ_OK;
}

axq_status axq_lut_conv2d(const axq_conv_desc* d, const int8_t* X, const int8_t* Wt,
                          axq_lut_t lut, int32_t* Y, void* stream) {
    if (d && d->groups != 1) return gconv_run(d, X, Wt, lut, nullptr, Y, S(stream));
    axq::MMArgs p;
    int loader;
    axq_status s = conv_setup(d, X, Wt, lut, p, loader);
    if (s != AXQ_OK) return s;
    if (p.M == 0 || p.N == 0) return AXQ_OK;
    if (!Y) return AXQ_ERR_INVALID;
    return run_mm(p, loader, lut, nullptr, nullptr, Y, p.N, S(stream));
}

axq_status axq_lut_conv2d_dq(const axq_conv_desc* d, const int8_t* X, const int8_t* Wt,
                             axq_lut_t lut, const axq_epilogue* ep, void* stream) {
    if (d && d->groups != 1) {
        if (!ep) return AXQ_ERR_INVALID;
        return gconv_run(d, X, Wt, lut, ep, nullptr, S(stream));
    }
    axq::MMArgs p;
    int loader;
    axq_status s = conv_setup(d, X, Wt, lut, p, loader);
    if (s != AXQ_OK) return s;
    s = check_epilogue(ep, d->K, true);
    if (s != AXQ_OK) return s;
    if (p.M == 0 || p.N == 0) return AXQ_OK;
    const bool nchw = !ep->y_nhwc;
    axq::EpiArgs e = to_epi(ep, nchw, (int64_t)p.Ho * p.Wo);
    return run_mm(p, loader, lut, &e, ws_if_fits(ep, p.M * p.N), nullptr, 0, S(stream));
}

// ---------------------------------------------------------------------------------------
// Quantize-on-load variants (SURVEY §8(b) conventions; P:74 quantizer fused into the operand
// load, "~10% Q/DQ"): fp32 activations + their device scale, quantized by the loader of
// the resident-table kernel with axq_quantize's pinned rule, so the result equals the unfused
// axq_quantize -> axq_lut_gemm(_dq) / axq_lut_conv2d(_dq) chain bit for bit.
// ---------------------------------------------------------------------------------------
axq_status axq_lut_gemm_f32a(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                             const float* d_scale_a, const int8_t* W, int64_t ldw, axq_lut_t lut,
                             const axq_epilogue* ep, int32_t* C, int64_t ldc, void* stream) {
    axq_status s = gemm_common(M, N, K, reinterpret_cast<const int8_t*>(A), lda, W, ldw, lut);
    if (s != AXQ_OK) return s;
    if (!d_scale_a) return AXQ_ERR_INVALID;
    if (ep) {
        s = check_epilogue(ep, N, false);
        if (s != AXQ_OK) return s;
    } else if (M > 0 && N > 0 && (!C || ldc < N)) {
        return AXQ_ERR_INVALID;
    }
    if (M == 0 || N == 0) return AXQ_OK;
    if (K == 0 && !ep) {
        cudaError_t e = cudaMemset2DAsync(C, ldc * 4, 0, N * 4, M, S(stream));
        return e == cudaSuccess ? AXQ_OK : cuda_fail(e);
    }
    axq::MMArgs p{};
    p.Af = A; p.lda = lda; p.W = W; p.ldw = ldw; p.M = M; p.N = N; p.K = K;
    p.qscale = d_scale_a; p.qbits = lut->bits;
    fill_common(p, lut);
    axq_status r;
    if (ep) {
        axq::EpiArgs e = to_epi(ep, false, 0);
        r = run_mm(p, axq::LOAD_GEMM_F32, lut, &e, ws_if_fits(ep, M * N), nullptr, 0, S(stream));
    } else {
        r = run_mm(p, axq::LOAD_GEMM_F32, lut, nullptr, nullptr, C, ldc, S(stream));
    }
    g_last_path = AXQ_PATH_F32A | (g_last_path & AXQ_PATH_SPLITK);
    return r;
}

axq_status axq_lut_conv2d_f32(const axq_conv_desc* d, const float* X, const float* d_scale_a,
                              const int8_t* Wt, axq_lut_t lut, const axq_epilogue* ep, int32_t* Y,
                              void* stream) {
    if (!d || !d_scale_a) return AXQ_ERR_INVALID;
    if (d->c_valid != 0 && d->c_valid != d->C) return AXQ_ERR_UNSUPPORTED;   // no storage padding in NCHW fp32
    axq::MMArgs p;
    int loader;
    axq_status s = conv_setup(d, reinterpret_cast<const int8_t*>(X), Wt, lut, p, loader);
    if (s != AXQ_OK) return s;
    if (ep) {
        s = check_epilogue(ep, d->K, true);
        if (s != AXQ_OK) return s;
    } else if (p.M > 0 && p.N > 0 && !Y) {
        return AXQ_ERR_INVALID;
    }
    if (p.M == 0 || p.N == 0) return AXQ_OK;
    if (d->C * d->H * d->W * d->N >= ((int64_t)1 << 40)) return AXQ_ERR_UNSUPPORTED;
    p.A = nullptr;
    p.Af = X;
    p.qscale = d_scale_a;
    p.qbits = lut->bits;
    p.pad_lookups = 0;
    axq_status r;
    if (ep) {
        axq::EpiArgs e = to_epi(ep, !ep->y_nhwc, (int64_t)p.Ho * p.Wo);
        r = run_mm(p, axq::LOAD_CONV_F32, lut, &e, ws_if_fits(ep, p.M * p.N), nullptr, 0, S(stream));
    } else {
        r = run_mm(p, axq::LOAD_CONV_F32, lut, nullptr, nullptr, Y, p.N, S(stream));
    }
    g_last_path = AXQ_PATH_F32A | (g_last_path & AXQ_PATH_SPLITK);
    return r;
}

// ---------------------------------------------------------------------------------------
// Prepared weights + packed-table (P4) kernel
// ---------------------------------------------------------------------------------------
axq_status axq_wpack_create(axq_lut_t lut, const int8_t* W, int64_t N, int64_t K, int64_t ldw,
                            int a_nonneg, axq_wpack_t* out) {
    if (!out || N <= 0 || K <= 0 || ldw < K || !W) return AXQ_ERR_INVALID;
    *out = nullptr;
    axq_status s = check_lut(lut);
    if (s != AXQ_OK) return s;
    // delta8 tables: packed int8 E (P4W / P4); other tables whose E fits int16, for
    // non-negative activations: packed int16 E (P4W16); anything else: the resident-table kernel
    const bool e16 = lut->repr != AXQ_LUT_DELTA8;
    if (e16 && (!lut->d_e16 || !(a_nonneg & AXQ_WPACK_NONNEG) || (a_nonneg & AXQ_WPACK_ACTIVATIONS)))
        return AXQ_ERR_UNSUPPORTED;
    s = overflow_guard(lut, K);
    if (s != AXQ_OK) return s;
    axq_wpack* w = new axq_wpack();
    cudaGetDevice(&w->device);
    w->t00 = lut->t00;
    w->N = N;
    w->K = K;
    w->Kp = (K + 31) / 32 * 32;   // a whole number of 32-k stages (P4T half-range tables)
    w->half = (a_nonneg & AXQ_WPACK_NONNEG) ? 1 : 0;
    w->e16 = e16 ? 1 : 0;
    w->swap = (a_nonneg & AXQ_WPACK_ACTIVATIONS) ? 1 : 0;
    w->dtab = reinterpret_cast<const int8_t*>(lut->d_table);
    w->dtab_own = nullptr;
    if (w->swap) {   // activation packing reads E[x][*] rows: keep a transposed copy
        std::vector<int8_t> h(65536), ht(65536);
        cudaError_t e0 = cudaMemcpy(h.data(), lut->d_table, 65536, cudaMemcpyDeviceToHost);
        for (int uw = 0; uw < 256 && e0 == cudaSuccess; ++uw)
            for (int ua = 0; ua < 256; ++ua) ht[(ua << 8) | uw] = h[(uw << 8) | ua];
        if (e0 == cudaSuccess) e0 = cudaMalloc(&w->dtab_own, 65536);
        if (e0 == cudaSuccess) e0 = cudaMemcpy(w->dtab_own, ht.data(), 65536, cudaMemcpyHostToDevice);
        if (e0 != cudaSuccess) {
            cudaFree(w->dtab_own);
            delete w;
            return cuda_fail(e0);
        }
        w->dtab = w->dtab_own;
    }
    const int64_t nb = (N + axq::p4::TN - 1) / axq::p4::TN;
    const size_t tb = (size_t)nb * w->Kp * (w->e16 ? 8 : 4) * (w->half ? 128 : 256) * 4,
                 wb = (size_t)nb * w->Kp * axq::p4::TN;
    w->bytes = (int64_t)(tb + wb);
    cudaError_t e = cudaMalloc(&w->tables, tb);
    if (e == cudaSuccess) e = cudaMalloc(&w->wpk, wb);
    if (e == cudaSuccess) {
        int rc = w->e16 ? axq::p4_pack16(W, N, K, ldw, w->Kp, lut->d_e16, w->tables, 0)
                        : axq::p4_pack(W, N, K, ldw, w->Kp, w->dtab, w->tables, w->wpk, w->half, w->swap, 0);
        if (!rc && w->e16)   // the packed weight tile of the exact part (p4_pack writes both)
            rc = axq::p4_pack_w(W, N, K, ldw, w->Kp, w->wpk, 0);
        e = rc ? (cudaError_t)rc : cudaDeviceSynchronize();
    }
    if (e != cudaSuccess) {
        cudaFree(w->tables);
        cudaFree(w->wpk);
        delete w;
        return cuda_fail(e);
    }
    *out = w;
    return AXQ_OK;
}

axq_status axq_wpack_repack(axq_wpack_t wp, const int8_t* W, int64_t ldw, void* stream) {
    if (!wp || !W || ldw < wp->K) return AXQ_ERR_INVALID;
    if (wp->wide_bits) return AXQ_ERR_UNSUPPORTED;
    if (wp->e16) return AXQ_ERR_UNSUPPORTED;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != wp->device) return AXQ_ERR_INVALID;
    const int rc = axq::p4_pack(W, wp->N, wp->K, ldw, wp->Kp, wp->dtab, wp->tables, wp->wpk, wp->half, wp->swap,
                                S(stream));
    return rc ? cuda_fail((cudaError_t)rc) : AXQ_OK;
}

axq_status axq_wpack_destroy(axq_wpack_t wp) {
    if (!wp) return AXQ_OK;
    cudaDeviceSynchronize();
    cudaFree(wp->tables);
    cudaFree(wp->wpk);
    if (wp->dtab_own) cudaFree(wp->dtab_own);
    delete wp;
    return AXQ_OK;
}

axq_status axq_wpack_info(axq_wpack_t wp, int64_t* N, int64_t* K, int64_t* device_bytes) {
    if (!wp) return AXQ_ERR_INVALID;
    if (N) *N = wp->N;
    if (K) *K = wp->K;
    if (device_bytes) *device_bytes = wp->bytes;
    return AXQ_OK;
}

// Kernel-choice knobs (measurement switches).  Atomics: a setter racing a launch on another
// thread sees either value, both of which give bit-identical results.
static std::atomic<int> g_p4w_main_cw{28};        // AXQ_P4W_MAIN_CW: consumer warps of the half-range 32-k shape
static std::atomic<int64_t> g_p4w_main_cw_max_k{1 << 30};   // ... for layers with K up to this
static std::atomic<int> g_p4w_res_cw{20};         // AXQ_P4W_RES_CW: consumer warps of the residual-layer shape (r2: 20 after the specialised epilogue)
static std::atomic<int64_t> g_nbfast_mib{24};     // AXQ_NBFAST_MIB: column-block-fastest tile order up to this table size
static std::atomic<int> g_p4w_tma_res{2};         // AXQ_P4W_TMA_RES: residual rows by TMA (RESBUF shapes), 2: + y stores
static std::atomic<int> g_p4w_tma{2};             // AXQ_P4W_TMA: activation planes by TMA (0 off, 1 GEMM rows, 2 + im2col)
static std::atomic<int> g_p4w_cw{0};              // AXQ_P4W_CW: 0 auto (16 for M <= 1024), 16 or 28 forced
static std::atomic<int64_t> g_sk_full_waves{8};   // AXQ_SK_FULL_WAVES: P4W layers of fewer than this many waves of
                                                  // tiles cut every iteration (no whole-wave phase): measured
                                                  // 73.5 -> 73.2 ms at 256 images, 10.79 -> 10.60 at 32 (4, 16 close)
static std::atomic<int64_t> g_sk_min_stages{4};   // AXQ_SK_MIN_STAGES: stream-K pieces of >= 4 stages (measured
                                                  // with the 512-row residual shape: 1 -> 4 saves 0.3-0.7 ms per
                                                  // forward at 256-32 images; 6 is worse again)
static std::atomic<int64_t> g_p4w_ks16_max_k{0};  // AXQ_P4W_KS16_MAX_K: measured slower, off
static std::atomic<int> g_wpack_kernel{0};        // axq_wpack_kernel: 0 default (P4W; P4 for c4 convs), 1 P4, 3 P4W

static void p4w_read_env() {
    static std::once_flag once;
    std::call_once(once, [] {
        if (const char* v = std::getenv("AXQ_P4W_KS16_MAX_K")) g_p4w_ks16_max_k = std::atoll(v);
        if (const char* v = std::getenv("AXQ_SK_MIN_STAGES")) g_sk_min_stages = std::max(1LL, std::atoll(v));
        if (const char* v = std::getenv("AXQ_P4W_PDL")) axq::g_p4w_pdl = std::atoi(v);
        if (const char* v = std::getenv("AXQ_P4W_CW")) g_p4w_cw = std::atoi(v);
        if (const char* v = std::getenv("AXQ_P4W_RES_CW")) g_p4w_res_cw = std::atoi(v);
        if (const char* v = std::getenv("AXQ_P4W_MAIN_CW")) g_p4w_main_cw = std::atoi(v);
        if (const char* v = std::getenv("AXQ_SK_FULL_WAVES")) g_sk_full_waves = std::atoll(v);
        if (const char* v = std::getenv("AXQ_P4W_MAIN_CW_MAX_K")) g_p4w_main_cw_max_k = std::atoll(v);
        if (const char* v = std::getenv("AXQ_P4W_TMA")) g_p4w_tma = std::atoi(v);
        if (const char* v = std::getenv("AXQ_P4W_TMA_RES")) g_p4w_tma_res = std::atoi(v);
        if (const char* v = std::getenv("AXQ_NBFAST_MIB")) g_nbfast_mib = std::atoll(v);
    });
}

// cuTensorMapEncodeTiled from the driver (no link-time libcuda dependency)
static PFN_cuTensorMapEncodeIm2col_v12000 tmap_encoder_im2col() {
    static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(ptr);
    });
    return fn;
}

static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

// P4W GEMM-row operand (plain GEMM, 1x1 / stride-1 / unpadded conv): a 2D u8 tensor map over
// [M][K] with row stride lda, box 16 k x 128 rows (one MMA slice of one 16-k plane); rows >= M
// and k >= K are zero-filled by the copy engine like the cp.async loader's zero-fill.  False
// (cp.async loader kept) when the layout does not meet the copy engine's rules.
static bool p4w_encode_tma(axq::P4Args& a) {
    const axq::MMArgs& p = a.mm;
    if (!g_p4w_tma.load() || a.is_conv || a.c4 || a.grp_cout || p.M <= 0 || p.M >= ((int64_t)1 << 31) ||
        p.K <= 0 || p.K >= ((int64_t)1 << 31) || (p.lda & 15) != 0 || p.lda >= ((int64_t)1 << 40) ||
        (reinterpret_cast<uintptr_t>(p.A) & 15) != 0)
        return false;
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)p.K, (cuuint64_t)p.M};
    cuuint64_t strides[1] = {(cuuint64_t)p.lda};
    cuuint32_t box[2] = {16u, 128u};
    cuuint32_t es[2] = {1u, 1u};
    CUresult r = enc(&a.tmap_a, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(p.A), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// P4W residual layers: the epilogue's fp32 residual [M][N] (row stride ldr) as a 2D tensor map,
// box 16 columns x 128 rows (one MMA slice of one column tile); used by the residual-layer
// shapes that have room for the tile's rows in shared memory (lut_p4w.cuh Geo::RESBUF)
static bool p4w_encode_rows_f32(CUtensorMap* map, const float* base, int64_t M, int64_t N, int64_t ld) {
    if (!base || M <= 0 || M >= ((int64_t)1 << 31) || N <= 0 || (ld & 3) != 0 || ld < N ||
        (reinterpret_cast<uintptr_t>(base) & 15) != 0)
        return false;
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
    cuuint32_t box[2] = {16u, 128u};
    cuuint32_t es[2] = {1u, 1u};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool p4w_encode_res(axq::P4Args& a, const axq::EpiArgs& e) {
    if (!g_p4w_tma_res.load() || a.transposed || !e.residual) return false;
    if (!p4w_encode_rows_f32(&a.tmap_res, e.residual, a.mm.M, a.mm.N, e.ldr)) return false;
    a.tma_y = (g_p4w_tma_res.load() >= 2 && e.y && !e.y_nchw &&
               p4w_encode_rows_f32(&a.tmap_y, e.y, a.mm.M, a.mm.N, e.ldy)) ? 1 : 0;
    return true;
}

// P4W implicit-im2col operand (a conv, any padding / stride, 16-channel planes): an im2col
// tensor map over the NHWC input [N][H][W][pix] -- each copy loads 128 consecutive output
// pixels' 16 channels of one tap (row, image boundaries and padding taps handled by the copy
// engine's traversal of the window-corner box, padding zero-filled), i.e. one MMA slice of one
// plane.  Square, symmetric windows only (the box corners are then order-free); the host checks
// that the box's traversal yields exactly Ho x Wo positions.
static bool p4w_encode_im2col(axq::P4Args& a) {
    const axq::MMArgs& p = a.mm;
    if (!g_p4w_tma.load() || !a.is_conv || a.c4 || a.grp_cout || p.M <= 0 || p.M >= ((int64_t)1 << 31) ||
        (p.C & 15) != 0 || (reinterpret_cast<uintptr_t>(p.A) & 15) != 0 || p.ph != p.pw || p.sh != p.sw ||
        p.dh != p.dw || p.sh < 1 || p.sh > 8)
        return false;
    const int64_t pix = p.cs ? p.cs : p.C;
    const int64_t rs = p.K / p.C, R = rs / p.S;
    if (R * p.S * p.C != p.K || R != p.S || (pix & 15) != 0) return false;
    const int64_t hw = (int64_t)p.Ho * p.Wo, n_img = p.M / hw;
    if (n_img * hw != p.M) return false;
    const int lo = -p.pw, up = p.pw - (int)(R - 1) * p.dw;
    if (lo < -128 || lo > 127 || up < -128 || up > 127) return false;
    // positions the traversal visits per row / column must be the output extents
    if ((p.Wd - 1 + up - lo) < 0 || (p.Wd - 1 + up - lo) / p.sw + 1 != p.Wo ||
        (p.H - 1 + up - lo) / p.sh + 1 != p.Ho)
        return false;
    auto enc = tmap_encoder_im2col();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)pix, (cuuint64_t)p.Wd, (cuuint64_t)p.H, (cuuint64_t)n_img};
    cuuint64_t strides[3] = {(cuuint64_t)pix, (cuuint64_t)(pix * p.Wd), (cuuint64_t)(pix * p.Wd * p.H)};
    int lower[2] = {lo, lo}, upper[2] = {up, up};
    cuuint32_t es[4] = {1u, (cuuint32_t)p.sw, (cuuint32_t)p.sh, 1u};
    CUresult r = enc(&a.tmap_a, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(p.A), dims, strides, lower,
                     upper, 16u, 128u, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

axq_status axq_wpack_shapes(int main_cw, int res_cw, int small_cw) {
    p4w_read_env();
    if ((main_cw && main_cw != 16 && main_cw != 20 && main_cw != 24 && main_cw != 28) ||
        (res_cw && res_cw != 16 && res_cw != 20 && res_cw != 24 && res_cw != 28) ||
        (small_cw && small_cw != 16 && small_cw != 28))
        return AXQ_ERR_INVALID;
    if (main_cw) g_p4w_main_cw = main_cw;
    if (res_cw) g_p4w_res_cw = res_cw;
    if (small_cw) g_p4w_cw = small_cw == 16 ? 0 : 28;
    return AXQ_OK;
}

int axq_wpack_kernel(int variant) {
    if (variant < 0 || variant > 3 || variant == 2) return -1;   // 2 was the superseded P4T kernel
    return g_wpack_kernel.exchange(variant);
}

// Stream-K scratch of the P4W kernel, carved from the caller's epilogue workspace (so two
// launches on two streams with two workspaces never share it): [STREAMK_CNT] int32 tile
// counters (zero on entry, left zero by the kernel), then one pair of [BM][16] int32 partial
// slots per CTA.
static constexpr int64_t STREAMK_CNT = 256;
static int64_t streamk_elems(int bm) { return STREAMK_CNT + (int64_t)sm_count() * 2 * bm * axq::p4::TN; }

axq_status axq_last_path(int* out) {
    if (!out) return AXQ_ERR_INVALID;
    *out = g_last_path;
    return AXQ_OK;
}

int64_t axq_workspace_elems(int64_t M, int64_t N) {
    if (M < 0 || N < 0) return -1;
    return std::max<int64_t>(M * N, streamk_elems(896));
}

static axq_status p4_run(axq::P4Args& a, axq_wpack_t wp, const axq_epilogue* ep, bool conv,
                         int32_t* C, int64_t ldc, cudaStream_t st) {
    if (wp->wide_bits) return AXQ_ERR_INVALID;   // wide packs: axq_lut_gemm16_wp
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != wp->device) return AXQ_ERR_INVALID;
    a.tables = wp->tables;
    a.wpk = wp->wpk;
    a.Kp = wp->Kp;
    a.is_conv = (conv && !a.pointwise) ? 1 : 0;
    a.one = 1u;
    a.half = wp->half;
    a.mm.t00 = wp->t00;
    axq::EpiArgs epi{};
    if (ep) {
        axq_status s = check_epilogue(ep, a.transposed ? a.mm.M : a.mm.N, conv);
        if (s != AXQ_OK) return s;
        epi = to_epi(ep, conv && !ep->y_nhwc, (int64_t)a.mm.Ho * a.mm.Wo);
        if (a.transposed && (ep->ldy < a.mm.M && ep->y)) return AXQ_ERR_INVALID;
    } else if (!C || ldc < (a.transposed ? a.mm.M : a.mm.N)) {
        return AXQ_ERR_INVALID;
    }
    if (a.mm.M == 0) return AXQ_OK;
    // raw output may always split K (atomics into C); the fused epilogue needs a workspace of
    // M*N elements for that
    const int64_t ws_elems = (ep && ep->workspace) ? (ep->workspace_elems > 0 ? ep->workspace_elems
                                                                             : a.mm.M * a.mm.N) : 0;
    const int64_t out_rows = a.transposed ? a.mm.N : a.mm.M, out_cols = a.transposed ? a.mm.M : a.mm.N;
    const bool can_split = ep ? (ws_elems >= out_rows * out_cols) : true;
    // default: P4W, except the 4-byte-tap conv loader (e.g. the padded 3-channel stem), where
    // P4's 2 rows per lane measure faster
    const int kv = g_wpack_kernel.load();
    const int variant = wp->e16 ? 3 : (kv != 0 ? kv : (a.c4 ? 1 : 3));
    a.e16 = wp->e16;
    if (wp->e16 && (a.c4 || kv == 1)) return AXQ_ERR_UNSUPPORTED;   // P4W16: 16-byte loaders, P4W only
    const bool use_tc = variant == 3;                                 // P4W: tcgen05 exact part
    // P4W shape: 512-row tiles (16 consumer warps) for small row counts, where 896-row tiles
    // would leave lanes idle or cut a ragged second tile; not for residual epilogues or the
    // half-range 16-k stages (no such instantiation)
    // k per stage: 32 for half-range tables, 16 for full-range ones, except half-range tables
    // with K <= AXQ_P4W_KS16_MAX_K (16-k stages, 4 deep)
    p4w_read_env();
    a.ks = wp->e16 ? 16 : wp->half ? ((variant == 3 && wp->Kp <= g_p4w_ks16_max_k) ? 16 : 32) : 16;
    const bool res_ep = ep && ep->residual;
    a.cw = 28;
    // 512-row tiles when they pad fewer rows than 896-row ones (M <= 1024 always: one or two
    // nearly empty 896-row tiles), e.g. the LSTM input projection (M = 8192 = 16 x 512, 9.1 x 896)
    const int64_t pad512 = (a.mm.M + 511) / 512 * 512 - a.mm.M, pad896 = (a.mm.M + 895) / 896 * 896 - a.mm.M;
    const int cw_forced = g_p4w_cw, res_cw = g_p4w_res_cw, main_cw = g_p4w_main_cw;
    if (variant == 3 && !res_ep && !a.c4 && (!wp->half || a.ks == 32) && cw_forced != 28 &&
        (cw_forced == 16 || a.mm.M <= 1024 || pad512 < pad896))
        a.cw = 16;
    if (variant == 3 && res_ep && wp->half && a.ks == 32 && !a.c4 && (res_cw == 16 || res_cw == 20 || res_cw == 24))
        a.cw = res_cw;
    if (variant == 3 && !res_ep && wp->half && a.ks == 32 && !a.c4 && a.cw == 28 &&
        (main_cw == 16 || main_cw == 20 || main_cw == 24) && wp->Kp <= g_p4w_main_cw_max_k)
        a.cw = main_cw;
    if (wp->e16) a.cw = (res_ep || a.mm.M <= 1024 || pad512 < pad896) ? 16 : 28;
    const int bm = variant == 3 ? axq::p4w_bm(a.cw) : 1024;
    if (use_tc)
        axq::p4w_plan(a.mm.M, a.mm.N, wp->Kp, a.ks, bm, sm_count(), can_split && !a.transposed, a.splits,
                      a.stages_per_split);
    else
        axq::p4_plan(a.mm.M, a.mm.N, wp->Kp, sm_count(), can_split, a.rpl, a.splits, a.stages_per_split);
    a.tma_a = variant != 3 ? 0 : p4w_encode_tma(a) ? 1 : (g_p4w_tma.load() >= 2 && p4w_encode_im2col(a)) ? 2 : 0;
    a.tma_y = 0;
    a.tma_res = (variant == 3 && ep && ep->residual && p4w_encode_res(a, epi)) ? 1 : 0;
    auto launch = [&](const axq::P4Args& x) { return variant == 3 ? axq::launch_p4w(x, st) : axq::launch_p4(x, st); };
    int path = wp->e16 ? AXQ_PATH_P4W16 : variant == 3 ? AXQ_PATH_P4W : AXQ_PATH_P4;
    path |= a.tma_a == 1 ? AXQ_PATH_TMA : a.tma_a == 2 ? AXQ_PATH_TMA_IM2COL : 0;
    if (use_tc && ep && ep->workspace && ws_elems >= streamk_elems(bm) &&
        (reinterpret_cast<uintptr_t>(ep->workspace) & 15) == 0) {
        // stream-K whenever whole tiles would leave a partial wave (exact int32 pieces in the
        // caller's workspace; finished by the kernel itself, no extra launch)
        const int64_t tiles = ((a.mm.M + bm - 1) / bm) * ((a.mm.N + axq::p4::TN - 1) / axq::p4::TN);
        if (tiles % sm_count() != 0) {
            const bool full = tiles < g_sk_full_waves * sm_count();
            a.streamk = full ? 2 : 1;
            a.splits = 1;
            a.stages_per_split = 0;
            // pieces of at least ~4 stages: a small tail is shared by fewer CTAs
            const int64_t tail_it = (full ? tiles : tiles % sm_count()) * (wp->Kp / a.ks);
            a.sk_ctas = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)sm_count(), STREAMK_CNT,
                                                                      tail_it / g_sk_min_stages}));
            a.cnt = ep->workspace;
            a.ws = ep->workspace + STREAMK_CNT;
            path |= AXQ_PATH_STREAMK;
        }
    }
    // column-block-fastest order when all of the layer's tables fit comfortably in L2
    a.nb_fast = (wp->bytes <= (g_nbfast_mib.load() << 20)) ? 1 : 0;
    if (a.splits > 1) {
        int32_t* acc = ep ? ep->workspace : C;
        const int64_t ld = ep ? a.mm.N : ldc;
        cudaError_t e = cudaMemset2DAsync(acc, ld * 4, 0, a.mm.N * 4, a.mm.M, st);
        if (e != cudaSuccess) return cuda_fail(e);
        a.mm.C_out = acc;
        a.mm.ldc = ld;
        g_last_path = path | AXQ_PATH_SPLITK;
        int rc = launch(a);
        if (rc) return cuda_fail((cudaError_t)rc);
        return ep ? launch_epilogue(a.mm.M, a.mm.N, acc, ld, epi, st, acc) : AXQ_OK;
    }
    if (ep) {
        a.mm.ep = epi;
        a.mm.C_out = nullptr;
    } else {
        a.mm.C_out = C;
        a.mm.ldc = ldc;
    }
    g_last_path = path;
    int rc = launch(a);
    return rc ? cuda_fail((cudaError_t)rc) : AXQ_OK;
}

axq_status axq_lut_gemm_xs(int64_t N, const int8_t* W, int64_t ldw, axq_wpack_t xp,
                           const axq_epilogue* ep, int32_t* C, int64_t ldc, void* stream) {
    // acc[m][n] = sum_k LUT[x[m][k]][W[n][k]] with x packed (activation-specialised) in xp: the
    // P4W kernel runs with the weight rows as its row operand and writes the result transposed
    if (!xp || !xp->swap || N < 0 || (N > 0 && (!W || ldw < xp->K))) return AXQ_ERR_INVALID;
    if (!aligned16(W) || (ldw & 15)) return AXQ_ERR_UNSUPPORTED;
    if (g_wpack_kernel.load() == 1) return AXQ_ERR_UNSUPPORTED;   // P4W only
    axq::P4Args a{};
    a.mm.A = W; a.mm.lda = ldw; a.mm.M = N; a.mm.N = xp->N; a.mm.K = xp->K;
    a.transposed = 1;
    return p4_run(a, xp, ep, false, C, ldc, S(stream));
}

axq_status axq_lut_gemm_wp(int64_t M, const int8_t* A, int64_t lda, axq_wpack_t wp,
                           const axq_epilogue* ep, int32_t* C, int64_t ldc, void* stream) {
    if (!wp || M < 0 || (M > 0 && (!A || lda < wp->K))) return AXQ_ERR_INVALID;
    if (!aligned16(A) || (lda & 15)) return AXQ_ERR_UNSUPPORTED;
    axq::P4Args a{};
    a.mm.A = A; a.mm.lda = lda; a.mm.M = M; a.mm.N = wp->N; a.mm.K = wp->K;
    return p4_run(a, wp, ep, false, C, ldc, S(stream));
}

axq_status axq_lut_conv2d_wp(const axq_conv_desc* d, const int8_t* X, axq_wpack_t wp,
                             const axq_epilogue* ep, int32_t* Y, void* stream) {
    if (!wp || !d) return AXQ_ERR_INVALID;
    if (d->groups < 1 || d->C % d->groups || d->K % d->groups) return AXQ_ERR_INVALID;
    const int64_t cin_g = d->C / d->groups, cout_g = d->K / d->groups;
    // grouped (NEXT-3): every 16-column tile inside one group, 16-byte channel runs per group
    if (d->groups > 1 && ((cout_g & 15) || (cin_g & 15) || !aligned16(X) || d->c_valid || wp->e16 ||
                          g_wpack_kernel.load() == 1))
        return AXQ_ERR_UNSUPPORTED;
    if ((d->C & 3) || (reinterpret_cast<uintptr_t>(X) & 3)) return AXQ_ERR_UNSUPPORTED;
    const bool c4 = (d->C & 15) || !aligned16(X);
    if (c4 && wp->Kp > axq::p4::TAP_BYTES) return AXQ_ERR_UNSUPPORTED;   // tap table capacity
    if (d->K != wp->N || d->R * d->S * cin_g != wp->K) return AXQ_ERR_INVALID;
    axq::P4Args a{};
    int loader = 0;
    // reuse the generic conv validation (LUT-independent parts) through a shim LUT view
    if (d->N < 0 || d->H <= 0 || d->W <= 0 || d->c_valid < 0 || d->c_valid > d->C) return AXQ_ERR_INVALID;
    int64_t Ho, Wo;
    axq_status s = axq_conv2d_out_hw(d, &Ho, &Wo);
    if (s != AXQ_OK) return s;
    if (Ho <= 0 || Wo <= 0 || (d->N > 0 && !X)) return AXQ_ERR_INVALID;
    if (d->H * d->W * d->C >= (int64_t)1 << 31 || Ho * Wo >= (int64_t)1 << 31) return AXQ_ERR_INVALID;
    (void)loader;
    axq::MMArgs& p = a.mm;
    p.A = X; p.M = d->N * Ho * Wo; p.N = d->K; p.K = wp->K;
    p.H = (int)d->H; p.Wd = (int)d->W; p.C = (int)cin_g; p.Ho = (int)Ho; p.Wo = (int)Wo;
    if (d->groups > 1) {
        p.cs = (int)d->C;
        a.grp_cout = (int)cout_g;
        a.grp_cin = (int)cin_g;
    }
    p.S = (int)d->S; p.sh = (int)d->stride_h; p.sw = (int)d->stride_w;
    p.ph = (int)d->pad_h; p.pw = (int)d->pad_w; p.dh = (int)d->dil_h; p.dw = (int)d->dil_w;
    const int64_t cv = d->c_valid ? d->c_valid : d->C;
    p.pad_lookups = (int32_t)(d->R * d->S * (d->C - cv));
    a.c4 = c4 ? 1 : 0;
    // a 1x1 / stride-1 / unpadded conv is the GEMM of its NHWC rows (P:119 with a trivial im2col)
    a.pointwise = (!c4 && d->R == 1 && d->S == 1 && d->stride_h == 1 && d->stride_w == 1 && d->pad_h == 0 &&
                   d->pad_w == 0) ? 1 : 0;
    if (a.pointwise) p.lda = d->C;   // (grouped: the group's channel offset is added per tile)
    return p4_run(a, wp, ep, true, Y, d->K, S(stream));
}

// ---------------------------------------------------------------------------------------
// Dequantize / epilogue
// ---------------------------------------------------------------------------------------
axq_status axq_dequantize(int64_t M, int64_t N, const int32_t* acc, int64_t ldacc,
                          const float* d_scale_a, const float* d_scale_w, const float* bias,
                          float* y, int64_t ldy, void* stream) {
    if (M < 0 || N < 0 || !d_scale_a || !d_scale_w) return AXQ_ERR_INVALID;
    if (M == 0 || N == 0) return AXQ_OK;
    if (!acc || !y || ldacc < N || ldy < N) return AXQ_ERR_INVALID;
    axq::dequant_rows_kernel<<<stream_grid(M * N, 256 * 4), 256, 0, S(stream)>>>(
        M, N, acc, ldacc, d_scale_a, d_scale_w, bias, y, ldy);
    return check_launch();
}

axq_status axq_dequantize_nhwc_to_nchw(int64_t N, int64_t HW, int64_t C, const int32_t* acc,
                                       const float* d_scale_a, const float* d_scale_w,
                                       const float* bias, float* y, void* stream) {
    if (N < 0 || HW < 0 || C < 0 || !d_scale_a || !d_scale_w) return AXQ_ERR_INVALID;
    if (N == 0 || HW == 0 || C == 0) return AXQ_OK;
    if (!acc || !y || N > 65535) return AXQ_ERR_INVALID;
    dim3 grid((unsigned)((HW + 31) / 32), (unsigned)((C + 31) / 32), (unsigned)N);
    axq::dequant_nhwc_to_nchw_kernel<<<grid, dim3(32, 8), 0, S(stream)>>>(acc, HW, C, d_scale_a,
                                                                        d_scale_w, bias, y);
    return check_launch();
}

axq_status axq_epilogue_apply(int64_t M, int64_t N, const int32_t* acc, int64_t ldacc,
                              const axq_epilogue* ep, void* stream) {
    if (M < 0 || N < 0 || ldacc < N) return AXQ_ERR_INVALID;
    axq_status s = check_epilogue(ep, N, false);
    if (s != AXQ_OK) return s;
    if (M == 0 || N == 0) return AXQ_OK;
    if (!acc) return AXQ_ERR_INVALID;
    return launch_epilogue(M, N, acc, ldacc, to_epi(ep, false, 0), S(stream));
}

// ---------------------------------------------------------------------------------------
// Model glue
// ---------------------------------------------------------------------------------------
axq_status axq_maxpool2d_nhwc_i8(const int8_t* x, int64_t N, int64_t H, int64_t W, int64_t C,
                                 int64_t R, int64_t Sz, int64_t stride, int64_t pad, int8_t* y,
                                 void* stream) {
    if (N < 0 || H <= 0 || W <= 0 || C <= 0 || R <= 0 || Sz <= 0 || stride <= 0 || pad < 0 ||
        pad >= R || pad >= Sz)
        return AXQ_ERR_INVALID;
    const int64_t Ho = (H + 2 * pad - R) / stride + 1, Wo = (W + 2 * pad - Sz) / stride + 1;
    if (Ho <= 0 || Wo <= 0) return AXQ_ERR_INVALID;
    if (N == 0) return AXQ_OK;
    if (!x || !y) return AXQ_ERR_INVALID;
    if ((C & 15) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 &&
        N * Ho * Wo * (C / 16) < ((int64_t)1 << 31) && N * H * W * C < ((int64_t)1 << 40)) {
        axq::maxpool_nhwc_i8x16_kernel<<<stream_grid(N * Ho * Wo * (C / 16), 256), 256, 0, S(stream)>>>(
            x, (int)N, (int)H, (int)W, (int)C, (int)R, (int)Sz, (int)stride, (int)pad, (int)Ho, (int)Wo, y);
    } else if ((C & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 3) == 0 && (reinterpret_cast<uintptr_t>(y) & 3) == 0) {
        axq::maxpool_nhwc_i8_kernel<<<stream_grid(N * Ho * Wo * (C / 4), 256), 256, 0, S(stream)>>>(
            x, N, (int)H, (int)W, (int)C, (int)R, (int)Sz, (int)stride, (int)pad, (int)Ho, (int)Wo, y);
    } else {
        axq::maxpool_nhwc_i8_bytes_kernel<<<stream_grid(N * Ho * Wo * C, 256), 256, 0, S(stream)>>>(
            x, N, (int)H, (int)W, (int)C, (int)R, (int)Sz, (int)stride, (int)pad, (int)Ho, (int)Wo, y);
    }
    return check_launch();
}

axq_status axq_im2col_nhwc_i8(const int8_t* X, int64_t N, int64_t H, int64_t W, int64_t C, int64_t c_valid,
                              int64_t R, int64_t Sz, int64_t stride_h, int64_t stride_w, int64_t pad_h,
                              int64_t pad_w, int8_t* A, int64_t lda, void* stream) {
    if (N < 0 || H <= 0 || W <= 0 || C <= 0 || R <= 0 || Sz <= 0 || stride_h <= 0 || stride_w <= 0 ||
        pad_h < 0 || pad_w < 0)
        return AXQ_ERR_INVALID;
    const int64_t cv = c_valid ? c_valid : C;
    const int64_t K = R * Sz * cv;
    if (cv > C || lda < K || (lda & 15) || lda > 8192 || R > 255 || Sz > 255) return AXQ_ERR_INVALID;
    const int64_t Ho = (H + 2 * pad_h - R) / stride_h + 1, Wo = (W + 2 * pad_w - Sz) / stride_w + 1;
    if (Ho <= 0 || Wo <= 0) return AXQ_ERR_INVALID;
    if (N == 0) return AXQ_OK;
    if (!X || !A || (reinterpret_cast<uintptr_t>(A) & 15)) return AXQ_ERR_INVALID;
    const int64_t M = N * Ho * Wo;
    if (C == 4 && cv == 3 && R == 7 && Sz == 7 && lda == 160 && (reinterpret_cast<uintptr_t>(X) & 3) == 0) {
        axq::im2col_c4_kernel<7, 7, 3, 160><<<stream_grid(M, 256), 256, 0, S(stream)>>>(
            X, M, (int)H, (int)W, (int)Ho, (int)Wo, (int)stride_h, (int)stride_w, (int)pad_h, (int)pad_w, A);
        const cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? AXQ_OK : cuda_fail(e);
    }
    axq::im2col_nhwc_i8_kernel<<<stream_grid(M * (lda / 16), 256), 256, lda * 4, S(stream)>>>(
        X, M, (int)H, (int)W, (int)C, (int)Ho, (int)Wo, (int)stride_h, (int)stride_w, (int)pad_h, (int)pad_w,
        (int)Sz, (int)cv, (int)K, (int)lda, A);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? AXQ_OK : cuda_fail(e);
}

axq_status axq_maxpool2d_nhwc_f32(const float* x, int64_t N, int64_t H, int64_t W, int64_t C,
                                  int64_t R, int64_t Sz, int64_t stride, int64_t pad, float* y,
                                  void* stream) {
    if (N < 0 || H <= 0 || W <= 0 || C <= 0 || R <= 0 || Sz <= 0 || stride <= 0 || pad < 0 ||
        pad >= R || pad >= Sz)
        return AXQ_ERR_INVALID;
    const int64_t Ho = (H + 2 * pad - R) / stride + 1, Wo = (W + 2 * pad - Sz) / stride + 1;
    if (Ho <= 0 || Wo <= 0) return AXQ_ERR_INVALID;
    if (N == 0) return AXQ_OK;
    if (!x || !y) return AXQ_ERR_INVALID;
    axq::maxpool_nhwc_f32_kernel<<<stream_grid(N * Ho * Wo * C, 256), 256, 0, S(stream)>>>(
        x, N, (int)H, (int)W, (int)C, (int)R, (int)Sz, (int)stride, (int)pad, (int)Ho, (int)Wo, y);
    return check_launch();
}

axq_status axq_avgpool_nhwc(const float* x, int64_t N, int64_t HW, int64_t C, float* y,
                            int8_t* q, const float* d_scale, int bits, void* stream) {
    if (N < 0 || HW <= 0 || C <= 0) return AXQ_ERR_INVALID;
    if (q && (!d_scale || bits < 2 || bits > 8)) return AXQ_ERR_INVALID;
    if (N == 0) return AXQ_OK;
    if (!x || (!y && !q)) return AXQ_ERR_INVALID;
    axq::avgpool_nhwc_kernel<<<stream_grid(N * C, 256), 256, 0, S(stream)>>>(x, N, HW, C, y, q,
                                                                            d_scale, q ? bits : 8);
    return check_launch();
}

axq_status axq_lstm_cell(int64_t B, int64_t Hd, const float* gates_ih, const float* gates_hh,
                         float* c, float* h_out, int8_t* q_h, const float* d_scale_h, int bits,
                         void* stream) {
    if (B < 0 || Hd < 0) return AXQ_ERR_INVALID;
    if (q_h && (!d_scale_h || bits < 2 || bits > 8)) return AXQ_ERR_INVALID;
    if (B == 0 || Hd == 0) return AXQ_OK;
    if (!gates_ih || !gates_hh || !c || !h_out) return AXQ_ERR_INVALID;
    axq::lstm_cell_kernel<<<stream_grid(B * Hd, 256), 256, 0, S(stream)>>>(
        B, Hd, gates_ih, gates_hh, c, h_out, q_h, d_scale_h, q_h ? bits : 8);
    return check_launch();
}

// ---- NEXT-2: wide ACUs, int16 codes ----
axq_status axq_quantize16(const float* x, int64_t n, const float* d_scale, int bits, int16_t* q,
                          void* stream) {
    if (n < 0 || !d_scale || bits < 2 || bits > 16 || (n > 0 && (!x || !q))) return AXQ_ERR_INVALID;
    if (n == 0) return AXQ_OK;
    const int rc = axq::launch_quantize16(x, n, d_scale, bits, q, sm_count(), S(stream));
    return rc ? cuda_fail((cudaError_t)rc) : AXQ_OK;
}

axq_status axq_lut_gemm16(int64_t M, int64_t N, int64_t K, const int16_t* A, int64_t lda,
                          const int16_t* W, int64_t ldw, axq_lut_t lut, const axq_epilogue* ep,
                          int32_t* C, int64_t ldc, void* stream) {
    if (!lut || !lut->d_table || M < 0 || N < 0 || K < 0) return AXQ_ERR_INVALID;
    if (lut->repr != AXQ_LUT_WIDE16 && lut->repr != AXQ_LUT_WIDE32) return AXQ_ERR_UNSUPPORTED;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != lut->device) return AXQ_ERR_INVALID;
    if (M > 0 && N > 0 && K > 0 && (!A || !W || lda < K || ldw < K)) return AXQ_ERR_INVALID;
    axq_status s = overflow_guard(lut, K);
    if (s != AXQ_OK) return s;
    axq::WideArgs a{};
    a.A = A; a.lda = lda; a.W = W; a.ldw = ldw; a.M = M; a.N = N; a.K = K; a.bits = lut->bits;
    a.table = lut->d_table; a.delta16 = lut->repr == AXQ_LUT_WIDE16;
    if (ep) {
        s = check_epilogue(ep, N, false);
        if (s != AXQ_OK) return s;
        a.ep = to_epi(ep, false, 0);
    } else {
        if (!C || ldc < N) return AXQ_ERR_INVALID;
        a.C_out = C;
        a.ldc = ldc;
    }
    if (M == 0 || N == 0) return AXQ_OK;
    g_last_path = AXQ_PATH_WIDE;
    const int rc = axq::launch_wide(a, sm_count(), S(stream));
    return rc ? cuda_fail((cudaError_t)rc) : AXQ_OK;
}

// ---- NEXT-2, packed: weight-specialised wide tables (wide_pk.cuh) ----
axq_status axq_wpack16_create(axq_lut_t lut, const int16_t* W, int64_t N, int64_t K, int64_t ldw,
                              axq_wpack_t* out) {
    if (!out || !lut || !lut->d_table || N <= 0 || K <= 0 || ldw < K || !W) return AXQ_ERR_INVALID;
    *out = nullptr;
    if (lut->repr != AXQ_LUT_WIDE16) return AXQ_ERR_UNSUPPORTED;   // E must fit int16
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != lut->device) return AXQ_ERR_INVALID;
    if (K >= 65536 - axq::wpk::KP_ALIGN) return AXQ_ERR_UNSUPPORTED;   // 16-bit-lane sums exact below 2^16 k
    axq_status s = overflow_guard(lut, K);
    if (s != AXQ_OK) return s;
    const int bits = lut->bits, tn = axq::widepk_tn(bits);
    axq_wpack* w = new axq_wpack();
    w->device = dev;
    w->wide_bits = bits;
    w->t00 = lut->t00;
    w->N = N;
    w->K = K;
    w->Kp = (K + axq::wpk::KP_ALIGN - 1) / axq::wpk::KP_ALIGN * axq::wpk::KP_ALIGN;
    const int64_t nb = (N + tn - 1) / tn;
    const size_t tb = (size_t)nb * w->Kp * (tn / 4) * ((size_t)1 << bits) * 8, wb = (size_t)nb * w->Kp * tn * 2;
    w->bytes = (int64_t)(tb + wb);
    cudaError_t e = cudaMalloc(&w->tables, tb);
    if (e == cudaSuccess) e = cudaMalloc(&w->wpk, wb);
    if (e == cudaSuccess) {
        const int rc = axq::widepk_pack(W, N, K, ldw, w->Kp, bits, reinterpret_cast<const int16_t*>(lut->d_table),
                                        reinterpret_cast<uint2*>(w->tables), reinterpret_cast<int16_t*>(w->wpk),
                                        sm_count(), 0);
        e = rc ? (cudaError_t)rc : cudaDeviceSynchronize();
    }
    if (e != cudaSuccess) {
        cudaFree(w->tables);
        cudaFree(w->wpk);
        delete w;
        return cuda_fail(e);
    }
    *out = w;
    return AXQ_OK;
}

axq_status axq_lut_gemm16_wp(int64_t M, const int16_t* A, int64_t lda, axq_wpack_t wp,
                             const axq_epilogue* ep, int32_t* C, int64_t ldc, void* stream) {
    if (!wp || !wp->wide_bits || M < 0 || (M > 0 && (!A || lda < wp->K))) return AXQ_ERR_INVALID;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != wp->device) return AXQ_ERR_INVALID;
    axq::WidePkArgs a{};
    a.A = A; a.lda = lda; a.M = M; a.N = wp->N; a.K = wp->K; a.Kp = wp->Kp; a.bits = wp->wide_bits;
    a.tables = reinterpret_cast<const uint2*>(wp->tables);
    a.wts = reinterpret_cast<const int16_t*>(wp->wpk);
    a.t00 = wp->t00;
    if (ep) {
        axq_status s = check_epilogue(ep, wp->N, false);
        if (s != AXQ_OK) return s;
        a.ep = to_epi(ep, false, 0);
    } else {
        if (!C || ldc < wp->N) return AXQ_ERR_INVALID;
        a.C_out = C;
        a.ldc = ldc;
    }
    if (M == 0) return AXQ_OK;
    g_last_path = AXQ_PATH_WIDEPK;
    const int rc = axq::launch_widepk(a, sm_count(), S(stream));
    return rc ? cuda_fail((cudaError_t)rc) : AXQ_OK;
}

axq_status axq_lstm_recurrent(int64_t T, int64_t B, int64_t H, const float* gates_ih,
                              const int8_t* qw_hh, const float* d_scale_w_hh, const float* b_hh,
                              const float* d_scale_h, int bits, axq_lut_t lut, float* hs,
                              float* c_out, int8_t* workspace, void* stream) {
    if (T < 0 || B < 0 || H < 0) return AXQ_ERR_INVALID;
    if (T == 0 || B == 0 || H == 0) return AXQ_OK;
    if (!gates_ih || !qw_hh || !d_scale_w_hh || !b_hh || !d_scale_h || !hs || !c_out || !workspace)
        return AXQ_ERR_INVALID;
    axq_status s = check_lut(lut);
    if (s != AXQ_OK) return s;
    if (bits != lut->bits) return AXQ_ERR_INVALID;
    if (lut->repr != AXQ_LUT_DELTA8) return AXQ_ERR_UNSUPPORTED;
    s = overflow_guard(lut, H);
    if (s != AXQ_OK) return s;
    if (T > INT32_MAX || B > INT32_MAX || H > INT32_MAX || (reinterpret_cast<uintptr_t>(workspace) & 15) ||
        (reinterpret_cast<uintptr_t>(qw_hh) & 15))
        return AXQ_ERR_UNSUPPORTED;
    axq::LstmRecArgs a{};
    a.T = (int)T; a.B = (int)B; a.H = (int)H;
    a.gih = gates_ih; a.qw = qw_hh; a.sw = d_scale_w_hh; a.b_hh = b_hh; a.sh = d_scale_h;
    a.bits = bits; a.table = reinterpret_cast<const int8_t*>(lut->d_table);
    a.hs = hs; a.c_out = c_out; a.hq = workspace;
    a.bar = reinterpret_cast<unsigned int*>(workspace + ((2 * B * H + 15) / 16) * 16);
    g_last_path = AXQ_PATH_LSTM_REC;
    const int rc = axq::launch_lstm_rec(a, sm_count(), S(stream));
    if (rc == -1) return AXQ_ERR_UNSUPPORTED;
    return rc ? cuda_fail((cudaError_t)rc) : AXQ_OK;
}

}  // extern "C"

namespace axq {
// for the other translation units' entry points (mm_ste.cu): record a failed CUDA call
axq_status cuda_fail_ext(int e) { return cuda_fail((cudaError_t)e); }
}  // namespace axq

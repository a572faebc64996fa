// lut_mm.cuh -- the approximate LUT-GEMM / implicit-im2col LUT-conv core (sm_100a).
//
// Computes acc[m][n] = sum_k LUT[a[m][k]][w[n][k]] in int32 (BASELINE.json north_star;
// PAPER.md:161 "the inner multiplications between each input and filter values using a
// LUT"), where a[m][k] is a row of A (linear layer) or of the implicit im2col
// matrix of a convolution.
//
// Design:
//  * The ACU table lives in shared memory for the whole CTA, TRANSPOSED (row = weight
//    pattern uw, column = activation pattern ua) so that the 32 lanes of one gather share
//    the weight and differ only in the activation: a row is 256 B (int8) = 2 bank lines,
//    so a gather costs at most 2 wavefronts and 1 for the usual |a| < 64 codes.
//  * Representation DELTA8 stores E = LUT - a*w as int8 (64 KiB); the exact part a*w is
//    added with one dp4a per 4 lookups, so lookups stay 1 byte wide.  I16 stores LUT
//    values directly (128 KiB).  Tables whose values do not fit int16 (256 KiB of int32):
//    I32 gathers through L1 (no shared-memory carve-out, 3 CTAs per SM: the L1 holds the
//    touched rows); I32H keeps the table SM-resident in shared memory as two 128 KiB halves
//    split by the activation's high bit ("populate the cache with the LUTs",
//    north_star "int32 split across SM-resident halves" / "tiled by the a-operand's high
//    bits"): a tile's K loop runs with the resident half, lookups of the other half adding
//    0, and a second pass with the other half runs only if some code of the tile needs it
//    (ReLU inputs: never, so the table is staged once per CTA).
//  * One lane owns R output rows (m) x TN output columns (n); the 32 lanes of a warp own
//    32 consecutive rows.  The gather index (uw << 8) | ua is built by ONE byte-permute
//    (PRMT) from a zero-padded activation word and the packed weight word.
//  * K is streamed in chunks of KC = 16 bytes: activations go global -> registers
//    (lane-private rows, 16-byte loads, prefetched one chunk ahead); the CTA's weight
//    tile [KC/4][TN] (packed 4 k per word) is staged through double-buffered shared
//    memory and read with broadcast 16-byte loads.
//  * K-tail storage padding contributes (0,0) lookups; they are removed exactly by
//    subtracting npad * LUT[0][0] (semantic conv padding is NOT removed: A11).
//  * Persistent: grid = resident CTAs; each stages the table once and walks the (m, n, k-split)
//    tiles.  Split-K uses int32 atomics (exact because integer addition is
//    associative).  Epilogues: raw int32, atomic int32, fused dequant to [M][N] fp32 or to
//    NCHW fp32 (lanes = consecutive pixels -> coalesced stores).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "async_copy.cuh"
#include "epilogue.cuh"

namespace axq {

constexpr int KC = 16;

enum { REPR_DELTA8 = 0, REPR_I16 = 1, REPR_I32 = 2, REPR_I32H = 3 };
enum { EPI_RAW = 0, EPI_RAW_ATOMIC = 1, EPI_FUSED = 2 };
enum { LOAD_GEMM = 0, LOAD_CONV = 1, LOAD_GEMM_BYTES = 2, LOAD_CONV_BYTES = 3, LOAD_CONV_C4 = 4,
       // quantize-on-load (SURVEY §8(b) axq_lut_gemm_f32a / axq_lut_conv2d_f32): the operand is
       // fp32 (GEMM rows [M][lda]; conv NCHW) and each element is quantized with the pinned
       // rule of axq_quantize (A1-A3) as it is loaded -- the codes equal the unfused chain's
       LOAD_GEMM_F32 = 5, LOAD_CONV_F32 = 6 };

struct MMArgs {
    const int8_t* A;  // GEMM: [M][lda]; conv: NHWC input X
    int64_t lda;
    const int8_t* W;  // [N][ldw]  (conv: KRSC flattened, ldw = R*S*C)
    int64_t ldw;
    int64_t M, N, K;
    // conv geometry
    int H, Wd, C, Ho, Wo, S, sh, sw, ph, pw, dh, dw;
    int cs;             // conv: NHWC pixel stride in channels (0 -> C; grouped conv: all C)
    const float* Af;    // LOAD_GEMM_F32 / LOAD_CONV_F32: fp32 operand (A / X unused)
    const float* qscale;  // ... its device quantization scale
    int qbits;          // ... and bit width
    const void* table;  // device table (representation-specific layout, [uw][ua])
    int table_bytes;
    int32_t t00;        // LUT[0][0] (value of one storage-padding lookup)
    int32_t pad_lookups;  // storage-padding lookups per output inside K (padded channels)
    int64_t k_split;    // K extent per split-K slice, multiple of KC
    // outputs
    int32_t* C_out;     // raw / atomic epilogues
    int64_t ldc;
    EpiArgs ep;         // fused epilogue
};

// Global-table form: I32 (through L1) and the grouped-conv kernels (gconv.cuh).
template <int REPR>
__device__ __forceinline__ int lut_fetch(const int8_t* lut_s, const int32_t* lut_g, uint32_t idx) {
    if constexpr (REPR == REPR_DELTA8) {
        return (int)lut_s[idx];
    } else if constexpr (REPR == REPR_I16) {
        return (int)reinterpret_cast<const int16_t*>(lut_s)[idx];
    } else {
        return __ldg(lut_g + idx);
    }
}

// I32H: lut_s holds half h = the entries with (ua >> 7) == h, laid out [uw][ua & 127]
// (axq_lut_create's d_i32h); an index of the other half reads an in-bounds word and
// contributes 0 (its own pass adds it).
constexpr int I32_HALF_BYTES = 131072;

template <int REPR>
__device__ __forceinline__ int lut_fetch(const int8_t* lut_s, uint32_t idx, uint32_t half) {
    if constexpr (REPR == REPR_DELTA8) {
        return (int)lut_s[idx];
    } else if constexpr (REPR == REPR_I16) {
        return (int)reinterpret_cast<const int16_t*>(lut_s)[idx];
    } else {
        const uint32_t j = ((idx >> 1) & 0x7f80u) | (idx & 0x7fu);
        const int v = reinterpret_cast<const int32_t*>(lut_s)[j];
        return ((idx >> 7) & 1u) == half ? v : 0;
    }
}

__device__ __forceinline__ uint4 ldg16(const int8_t* p) {
    return __ldg(reinterpret_cast<const uint4*>(p));
}

// Per-row state of the activation loader.
struct RowInfo {
    int64_t m;       // global row
    int64_t base;    // GEMM: m*lda ; conv: img*H*W*C
    int hb, wb;      // conv: ho*sh - ph, wo*sw - pw
    bool valid;
};

template <int LOADER>
__device__ __forceinline__ RowInfo make_row(const MMArgs& p, int64_t m) {
    RowInfo ri;
    ri.m = m;
    ri.valid = m < p.M;
    if constexpr (LOADER == LOAD_GEMM || LOADER == LOAD_GEMM_BYTES || LOADER == LOAD_GEMM_F32) {
        ri.base = m * p.lda;
        ri.hb = ri.wb = 0;
    } else if (p.M <= 0x7fffffff) {   // 32-bit index arithmetic (uniform branch)
        const uint32_t hw = (uint32_t)p.Ho * (uint32_t)p.Wo;
        const uint32_t mm = ri.valid ? (uint32_t)m : 0u;
        const uint32_t img = mm / hw, rem = mm - img * hw;
        const int ho = (int)(rem / (uint32_t)p.Wo), wo = (int)(rem - (uint32_t)ho * (uint32_t)p.Wo);
        ri.base = (int64_t)img * p.H * p.Wd * (p.cs ? p.cs : p.C);
        ri.hb = ho * p.sh - p.ph;
        ri.wb = wo * p.sw - p.pw;
    } else {
        int64_t hw = (int64_t)p.Ho * p.Wo;
        int64_t mm = ri.valid ? m : 0;
        int64_t img = mm / hw;
        int64_t rem = mm - img * hw;
        int ho = (int)(rem / p.Wo), wo = (int)(rem - (int64_t)ho * p.Wo);
        ri.base = img * (int64_t)p.H * p.Wd * (p.cs ? p.cs : p.C);
        ri.hb = ho * p.sh - p.ph;
        ri.wb = wo * p.sw - p.pw;
    }
    return ri;
}

// Load the 16 activation bytes a[m][k0 .. k0+15] (zeros beyond K or out of range rows;
// zeros at semantic conv padding taps, which ARE looked up).
// One element quantized as axq_quantize does (A1-A3: IEEE x / s, clamp, round half to even).
__device__ __forceinline__ uint32_t qload_byte(float x, float s, float qm) {
    float t = div_rn_nz(x, s);
    t = fminf(fmaxf(t, -qm), qm);
    return (uint32_t)(uint8_t)(int8_t)__float2int_rn(t);
}

template <int LOADER>
__device__ __forceinline__ uint4 load_a(const MMArgs& p, const RowInfo& ri, int64_t k0,
                                      const uint32_t* tap_s, float qs = 1.f, float qm = 127.f) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if constexpr (LOADER == LOAD_GEMM_F32) {
        if (ri.valid) {
            uint32_t w[4] = {0, 0, 0, 0};
            const float* row = p.Af + ri.base + k0;
            if (k0 + KC <= p.K && ((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float4 f = __ldg(reinterpret_cast<const float4*>(row) + j);
                    w[j] = qload_byte(f.x, qs, qm) | (qload_byte(f.y, qs, qm) << 8) |
                           (qload_byte(f.z, qs, qm) << 16) | (qload_byte(f.w, qs, qm) << 24);
                }
            } else {
#pragma unroll
                for (int j = 0; j < KC; ++j)
                    if (k0 + j < p.K) w[j >> 2] |= qload_byte(__ldg(row + j), qs, qm) << (8 * (j & 3));
            }
            v = make_uint4(w[0], w[1], w[2], w[3]);
        }
        return v;
    } else if constexpr (LOADER == LOAD_CONV_F32) {
        // NCHW fp32 input, k = (r, s, c) (KRSC weights); a padded tap is code 0 (A11)
        if (ri.valid && k0 < p.K) {
            uint32_t w[4] = {0, 0, 0, 0};
            int rs = (int)(k0 / p.C);
            int c = (int)(k0 - (int64_t)rs * p.C);
            int r = rs / p.S, s_ = rs - r * p.S;
            const int64_t hw = (int64_t)p.H * p.Wd;
#pragma unroll
            for (int j = 0; j < KC; ++j) {
                if (k0 + j < p.K) {
                    const int hi = ri.hb + r * p.dh, wi = ri.wb + s_ * p.dw;
                    if (hi >= 0 && hi < p.H && wi >= 0 && wi < p.Wd)
                        w[j >> 2] |= qload_byte(__ldg(p.Af + ri.base + (int64_t)c * hw + (int64_t)hi * p.Wd + wi),
                                                qs, qm) << (8 * (j & 3));
                }
                if (++c == p.C) {
                    c = 0;
                    if (++s_ == p.S) { s_ = 0; ++r; }
                }
            }
            v = make_uint4(w[0], w[1], w[2], w[3]);
        }
        return v;
    } else if constexpr (LOADER == LOAD_GEMM) {
        if (ri.valid && k0 + KC <= p.K) return ldg16(p.A + ri.base + k0);
        if (ri.valid) {
            uint32_t w[4] = {0, 0, 0, 0};
            for (int j = 0; j < KC; ++j)
                if (k0 + j < p.K)
                    w[j >> 2] |= (uint32_t)(uint8_t)p.A[ri.base + k0 + j] << (8 * (j & 3));
            v = make_uint4(w[0], w[1], w[2], w[3]);
        }
        return v;
    } else if constexpr (LOADER == LOAD_GEMM_BYTES) {
        if (ri.valid) {
            uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < KC; ++j)
                if (k0 + j < p.K)
                    w[j >> 2] |= (uint32_t)(uint8_t)p.A[ri.base + k0 + j] << (8 * (j & 3));
            v = make_uint4(w[0], w[1], w[2], w[3]);
        }
        return v;
    } else if constexpr (LOADER == LOAD_CONV) {
        // C % 16 == 0: the chunk lies inside one filter tap (r, s).
        int rs = (int)(k0 / p.C);
        int c0 = (int)(k0 - (int64_t)rs * p.C);
        int r = rs / p.S, s = rs - r * p.S;
        int hi = ri.hb + r * p.dh, wi = ri.wb + s * p.dw;
        if (ri.valid && k0 < p.K && hi >= 0 && hi < p.H && wi >= 0 && wi < p.Wd)
            v = ldg16(p.A + ri.base + ((int64_t)hi * p.Wd + wi) * (p.cs ? p.cs : p.C) + c0);
        return v;
    } else if constexpr (LOADER == LOAD_CONV_C4) {
        // C % 4 == 0 (small C, e.g. the padded network input): each 4-byte group of the chunk
        // lies inside one filter tap; tap offsets come from the per-CTA table built at start.
        if (ri.valid) {
            uint32_t w[4] = {0, 0, 0, 0};
            const int g0 = (int)(k0 >> 2);
            const uint4 t4 = *reinterpret_cast<const uint4*>(tap_s + g0);
            const uint32_t tv[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (k0 + 4 * j < p.K) {
                    const int hi = ri.hb + (int)(tv[j] & 0xff);
                    const int wi = ri.wb + (int)((tv[j] >> 8) & 0xff);
                    if (hi >= 0 && hi < p.H && wi >= 0 && wi < p.Wd)
                        w[j] = __ldg(reinterpret_cast<const uint32_t*>(
                            p.A + ri.base + ((int64_t)hi * p.Wd + wi) * (p.cs ? p.cs : p.C) + (tv[j] >> 16)));
                }
            }
            v = make_uint4(w[0], w[1], w[2], w[3]);
        }
        return v;
    } else {  // LOAD_CONV_BYTES: any C
        if (ri.valid) {
            uint32_t w[4] = {0, 0, 0, 0};
            for (int j = 0; j < KC; ++j) {
                int64_t k = k0 + j;
                if (k < p.K) {
                    int rs = (int)(k / p.C);
                    int c = (int)(k - (int64_t)rs * p.C);
                    int r = rs / p.S, s = rs - r * p.S;
                    int hi = ri.hb + r * p.dh, wi = ri.wb + s * p.dw;
                    if (hi >= 0 && hi < p.H && wi >= 0 && wi < p.Wd)
                        w[j >> 2] |= (uint32_t)(uint8_t)p.A[ri.base + ((int64_t)hi * p.Wd + wi) * (p.cs ? p.cs : p.C) + c]
                                     << (8 * (j & 3));
                }
            }
            v = make_uint4(w[0], w[1], w[2], w[3]);
        }
        return v;
    }
}

__device__ __forceinline__ uint4 load_w(const MMArgs& p, int64_t n, int64_t k0, bool vec) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (n >= p.N) return v;
    const int8_t* row = p.W + n * p.ldw;
    if (vec && k0 + KC <= p.K) return ldg16(row + k0);
    uint32_t w[4] = {0, 0, 0, 0};
    for (int j = 0; j < KC; ++j)
        if (k0 + j < p.K) w[j >> 2] |= (uint32_t)(uint8_t)row[k0 + j] << (8 * (j & 3));
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// WC: the CTA's warps form a (WARPS/WC) x WC grid over rows x columns; WC = WARPS splits
// only the columns (small M, e.g. the LSTM's
// recurrent GEMM with M = 64): CTA tile = (32 R) rows x (WARPS TN) columns.
template <int REPR, int TN, int R, int WARPS, int LOADER, int EPI, int WC = 1>
__global__ void __launch_bounds__(WARPS * 32, (WARPS >= 16 || REPR == REPR_I16 || REPR == REPR_I32H || WC > 1) ? 1 : (WARPS >= 8 ? 2 : 3))
lut_mm_kernel(const MMArgs p) {
    constexpr int NT = WARPS * 32;
    constexpr int WR = WARPS / WC;                 // warps along the rows
    constexpr int BM = WR * 32 * R;
    constexpr int CTN = WC * TN;                   // columns per CTA tile
    extern __shared__ __align__(16) int8_t smem[];
    // layout: [table (table_bytes; 0 for I32; one 128 KiB half for I32H)] [W tiles: 2 x KC/4 x TN words]
    int8_t* lut_s = smem;
    const int tbytes = (REPR == REPR_I32) ? 0 : (REPR == REPR_I32H) ? I32_HALF_BYTES : p.table_bytes;
    uint32_t* w_s = reinterpret_cast<uint32_t*>(smem + tbytes);
    const int32_t* lut_g = reinterpret_cast<const int32_t*>(p.table);

    uint32_t* tap_s = w_s + 2 * (KC / 4) * CTN;  // LOAD_CONV_C4 tap table (K/4 entries)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool wvec = ((p.ldw & 15) == 0) && ((reinterpret_cast<uintptr_t>(p.W) & 15) == 0);

    // ---- stage the ACU table in shared memory (once per CTA: the kernel is persistent) ----
    // one bulk copy (TMA, mbarrier complete_tx): the whole 64 / 128 KiB in flight at once, so a
    // small problem (BJ configs[0]) pays one memory latency for it, not one per 16-byte round
    __shared__ __align__(8) uint64_t tbl_bar;
    if (tid == 0) {
        mbar_init(smem_u32(&tbl_bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if constexpr (REPR != REPR_I32 && REPR != REPR_I32H) {
        const uint32_t bar = smem_u32(&tbl_bar);
        if (tid == 0) {
            mbar_expect_tx(bar, (uint32_t)tbytes);
            bulk_g2s(smem_u32(lut_s), p.table, (uint32_t)tbytes, bar);
        }
    }
    if constexpr (LOADER == LOAD_CONV_C4) {
        // entry g (k = 4g .. 4g+3): r*dh | s*dw << 8 | c << 16, padded with zeros
        const int ng = (int)((p.K + 3) / 4);
        for (int g = tid; g < ng + 4; g += NT) {
            uint32_t e = 0;
            if (g < ng) {
                const int k = 4 * g, rs = k / p.C, c = k - rs * p.C, r = rs / p.S, s_ = rs - r * p.S;
                e = (uint32_t)(r * p.dh) | ((uint32_t)(s_ * p.dw) << 8) | ((uint32_t)c << 16);
            }
            tap_s[g] = e;
        }
    }

    float qs = 1.f, qm = 127.f;
    if constexpr (LOADER == LOAD_GEMM_F32 || LOADER == LOAD_CONV_F32) {
        qs = __ldg(p.qscale);
        qm = (float)((1 << (p.qbits - 1)) - 1);
    }
    if constexpr (REPR != REPR_I32 && REPR != REPR_I32H) {
        __syncthreads();                       // barrier initialised before anyone waits on it
        mbar_wait(smem_u32(&tbl_bar), 0u);
    }
    int resident = -1;          // I32H: the half in lut_s (-1: none yet)
    uint32_t tbl_phase = 0;     // I32H: parity of the next table-barrier completion
    const int64_t m_tiles = (p.M + BM - 1) / BM, n_tiles = (p.N + CTN - 1) / CTN;
    const int64_t n_split = (p.K + p.k_split - 1) / p.k_split;
    const int64_t n_work = m_tiles * n_tiles * (n_split > 0 ? n_split : 1);
    for (int64_t tile = blockIdx.x; tile < n_work; tile += gridDim.x) {
    const int64_t ks = n_split > 0 ? tile % n_split : 0;
    const int64_t mn = n_split > 0 ? tile / n_split : tile;
    const int64_t m0 = (mn / n_tiles) * BM;
    const int64_t nc0 = (mn % n_tiles) * CTN;            // CTA's first column
    const int wr = warp % WR, wc = warp / WR;
    const int64_t n0 = nc0 + wc * TN;                    // this warp's first column
    const int64_t kb = ks * p.k_split;
    const int64_t ke = min(p.K, kb + p.k_split);
    const int nchunks = (int)((ke - kb + KC - 1) / KC);

    RowInfo rows[R];
#pragma unroll
    for (int r = 0; r < R; ++r)
        rows[r] = make_row<LOADER>(p, m0 + (int64_t)(wr * R + r) * 32 + lane);

    int acc[R][TN];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int n = 0; n < TN; ++n) acc[r][n] = 0;

    constexpr int NPASS = (REPR == REPR_I32H) ? 2 : 1;
    const int first_half = resident < 0 ? 0 : resident;
    uint32_t a_or = 0, a_nor = 0;   // I32H: OR of the tile's codes / of their complements
    for (int pass = 0; pass < NPASS; ++pass) {
    const uint32_t half = (uint32_t)(first_half ^ pass);
    if constexpr (REPR == REPR_I32H) {
        if (pass == 1) {
            // the other half is needed only if some code of the tile has its high bit
            const uint32_t other = first_half == 0 ? a_or : a_nor;
            if (!__syncthreads_or((other & 0x80808080u) != 0u)) break;
        }
        if ((int)half != resident) {
            __syncthreads();   // every warp is done reading the previous half
            if (tid == 0) {
                const uint32_t bar = smem_u32(&tbl_bar);
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic reads -> async writes
                mbar_expect_tx(bar, (uint32_t)I32_HALF_BYTES);
                bulk_g2s(smem_u32(lut_s), static_cast<const int8_t*>(p.table) + (size_t)half * I32_HALF_BYTES,
                         (uint32_t)I32_HALF_BYTES, bar);
            }
            mbar_wait(smem_u32(&tbl_bar), tbl_phase);
            tbl_phase ^= 1u;
            resident = (int)half;
        }
    }
    uint4 a_cur[R], a_nxt[R];
    uint4 w_nxt = make_uint4(0, 0, 0, 0);
    if (nchunks > 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) a_cur[r] = load_a<LOADER>(p, rows[r], kb, tap_s, qs, qm);
        if (tid < CTN) {
            uint4 wv = load_w(p, nc0 + tid, kb, wvec);
            w_s[0 * CTN + tid] = wv.x;
            w_s[1 * CTN + tid] = wv.y;
            w_s[2 * CTN + tid] = wv.z;
            w_s[3 * CTN + tid] = wv.w;
        }
    }
    __syncthreads();

    for (int ci = 0; ci < nchunks; ++ci) {
        const bool has_next = ci + 1 < nchunks;
        const int64_t kn = kb + (int64_t)(ci + 1) * KC;
        if (has_next) {
#pragma unroll
            for (int r = 0; r < R; ++r) a_nxt[r] = load_a<LOADER>(p, rows[r], kn, tap_s, qs, qm);
            if (tid < CTN) w_nxt = load_w(p, nc0 + tid, kn, wvec);
        }
        const uint32_t* ws = w_s + (ci & 1) * (4 * CTN) + wc * TN;
#pragma unroll
        for (int kq = 0; kq < 4; ++kq) {
            uint32_t a4[R], alo[R], ahi[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                a4[r] = (kq == 0) ? a_cur[r].x : (kq == 1) ? a_cur[r].y : (kq == 2) ? a_cur[r].z : a_cur[r].w;
                if constexpr (REPR == REPR_I32H) {
                    if (pass == 0) { a_or |= a4[r]; a_nor |= ~a4[r]; }
                }
                alo[r] = __byte_perm(a4[r], 0u, 0x4140);  // [a0, 0, a1, 0]
                ahi[r] = __byte_perm(a4[r], 0u, 0x4342);  // [a2, 0, a3, 0]
            }
#pragma unroll
            for (int n4 = 0; n4 < TN / 4; ++n4) {
                const uint4 wv = *reinterpret_cast<const uint4*>(ws + kq * CTN + n4 * 4);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t w4 = (j == 0) ? wv.x : (j == 1) ? wv.y : (j == 2) ? wv.z : wv.w;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        // gather index (uw << 8) | ua for the 4 k of this word
                        const uint32_t i0 = __byte_perm(alo[r], w4, 0x1140);
                        const uint32_t i1 = __byte_perm(alo[r], w4, 0x3352);
                        const uint32_t i2 = __byte_perm(ahi[r], w4, 0x1160);
                        const uint32_t i3 = __byte_perm(ahi[r], w4, 0x3372);
                        const int e0 = (REPR == REPR_I32 ? lut_fetch<REPR>(lut_s, lut_g, i0) : lut_fetch<REPR>(lut_s, i0, half));
                        const int e1 = (REPR == REPR_I32 ? lut_fetch<REPR>(lut_s, lut_g, i1) : lut_fetch<REPR>(lut_s, i1, half));
                        const int e2 = (REPR == REPR_I32 ? lut_fetch<REPR>(lut_s, lut_g, i2) : lut_fetch<REPR>(lut_s, i2, half));
                        const int e3 = (REPR == REPR_I32 ? lut_fetch<REPR>(lut_s, lut_g, i3) : lut_fetch<REPR>(lut_s, i3, half));
                        int s = acc[r][n4 * 4 + j];
                        if constexpr (REPR == REPR_DELTA8) s = __dp4a((int)a4[r], (int)w4, s);
                        acc[r][n4 * 4 + j] = s + e0 + e1 + e2 + e3;
                    }
                }
            }
        }
        if (has_next) {
#pragma unroll
            for (int r = 0; r < R; ++r) a_cur[r] = a_nxt[r];
            if (tid < CTN) {
                uint32_t* wd = w_s + ((ci + 1) & 1) * (4 * CTN);
                wd[0 * CTN + tid] = w_nxt.x;
                wd[1 * CTN + tid] = w_nxt.y;
                wd[2 * CTN + tid] = w_nxt.z;
                wd[3 * CTN + tid] = w_nxt.w;
            }
        }
        __syncthreads();
    }
    }   // pass

    // ---- remove storage-padding lookups (K tail of this split; padded channels) ----
    int64_t npad = (int64_t)nchunks * KC - (ke - kb);
    if (ke == p.K) npad += p.pad_lookups;   // counted once, by the split holding the K end
    if (npad != 0) {
        const int corr = (int)(npad * (int64_t)p.t00);
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int n = 0; n < TN; ++n) acc[r][n] -= corr;
    }

    // ---- epilogue ----
    float sc = 0.f, s_out = 1.f, qm = 127.f;
    if constexpr (EPI == EPI_FUSED) {
        sc = __fmul_rn(*p.ep.sa, *p.ep.sw);
        if (p.ep.q) {
            s_out = *p.ep.s_out;
            qm = (float)((1 << (p.ep.bits_out - 1)) - 1);
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const RowInfo& ri = rows[r];
        if (!ri.valid) continue;
        const int64_t m = ri.m;
        if constexpr (EPI == EPI_RAW) {
            int32_t* c = p.C_out + m * p.ldc + n0;
            if (n0 + TN <= p.N && ((p.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(p.C_out) & 15) == 0)) {
#pragma unroll
                for (int n = 0; n < TN; n += 4)
                    *reinterpret_cast<int4*>(c + n) = make_int4(acc[r][n], acc[r][n + 1], acc[r][n + 2], acc[r][n + 3]);
            } else {
#pragma unroll
                for (int n = 0; n < TN; ++n)
                    if (n0 + n < p.N) c[n] = acc[r][n];
            }
        } else if constexpr (EPI == EPI_RAW_ATOMIC) {
            int32_t* c = p.C_out + m * p.ldc + n0;
#pragma unroll
            for (int n = 0; n < TN; ++n)
                if (n0 + n < p.N) atomicAdd(c + n, acc[r][n]);
        } else {
            const EpiArgs& e = p.ep;
            const bool full = n0 + TN <= p.N;
            // vector path: row layout, 16-byte aligned rows (lane = row writes 4 columns per
            // store: half-sector granularity instead of 4-byte scattered stores)
            const bool vec = full && !e.y_nchw &&
                             (!e.y || (((e.ldy & 3) == 0) && ((reinterpret_cast<uintptr_t>(e.y) & 15) == 0))) &&
                             (!e.residual || (((e.ldr & 3) == 0) && ((reinterpret_cast<uintptr_t>(e.residual) & 15) == 0))) &&
                             (!e.bias || ((reinterpret_cast<uintptr_t>(e.bias) & 15) == 0 && (n0 & 3) == 0)) &&
                             (!e.q || (((e.ldq & 3) == 0) && ((reinterpret_cast<uintptr_t>(e.q) & 3) == 0)));
            if (vec) {
#pragma unroll
                for (int n = 0; n < TN; n += 4) {
                    const int64_t nn = n0 + n;
                    float v[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) v[j] = __fmul_rn(__int2float_rn(acc[r][n + j]), epi_sc(e, sc, nn + j));
                    if (e.bias) {
                        const float4 b = *reinterpret_cast<const float4*>(e.bias + nn);
                        v[0] = __fadd_rn(v[0], b.x); v[1] = __fadd_rn(v[1], b.y);
                        v[2] = __fadd_rn(v[2], b.z); v[3] = __fadd_rn(v[3], b.w);
                    }
                    if (e.residual) {
                        const float4 rr = __ldg(reinterpret_cast<const float4*>(e.residual + m * e.ldr + nn));
                        v[0] = __fadd_rn(v[0], rr.x); v[1] = __fadd_rn(v[1], rr.y);
                        v[2] = __fadd_rn(v[2], rr.z); v[3] = __fadd_rn(v[3], rr.w);
                    }
                    if (e.relu) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) v[j] = v[j] > 0.f ? v[j] : 0.f;
                    }
                    if (e.y) *reinterpret_cast<float4*>(e.y + m * e.ldy + nn) = make_float4(v[0], v[1], v[2], v[3]);
                    if (e.q) {
                        uint32_t w = 0;
#pragma unroll
                        for (int j = 0; j < 4; ++j) w |= (uint32_t)(uint8_t)epi_quant(v[j], s_out, qm) << (8 * j);
                        *reinterpret_cast<uint32_t*>(e.q + m * e.ldq + nn) = w;
                    }
                }
            } else {
#pragma unroll
                for (int n = 0; n < TN; ++n) {
                    const int64_t nn = n0 + n;
                    if (nn < p.N) epi_store(epi_value(acc[r][n], m, nn, sc, e), m, nn, p.N, e, s_out, qm);
                }
            }
        }
    }
    }  // persistent tile loop
}

}  // namespace axq

// lut_p4w.cuh -- "P4W": warp-specialised packed-table LUT-GEMM / implicit-im2col LUT-conv
// (sm_100a).  Same result as lut_p4.cuh / lut_mm.cuh: acc[m][n] = sum_k LUT[a[m][k]][w[n][k]]
// in int32, exact, as  sum_k a*w (tcgen05.mma kind::i8, TMEM)  +  sum_k E[a][w] (packed tables).
//
// Roles inside one persistent CTA (1024 threads, one CTA per SM):
//  * 4 producer warps (warps CW..CW+3) stream the operands of each (tile, stage) item into a
//    ring of STAGES shared-memory buffers: the activation planes (16 k x the tile's rows) by
//    TMA -- a 2D tiled tensor map for GEMM rows, an im2col-mode map for convs (padding taps
//    zero-filled by the copy engine) -- or, where neither applies, by cp.async (implicit
//    im2col, ignore-src zero fill, signalled with cp.async.mbarrier.arrive); the packed E
//    tables and weights by cp.async.bulk; all complete on the stage's full mbarrier.  A buffer
//    is refilled once the consumer warps released it (empty barrier) and the MMA that read it
//    completed.
//  * Residual layers (640-row shape): the tile's fp32 residual rows are staged in shared memory
//    by TMA (64-byte swizzle) and the block output y leaves through TMA stores per slice.
//  * CW consumer warps (one tile row per lane) only wait for full buffers and do the lookups
//    (4 per 32-bit LDS).  E8 tables: per quad and 4 k the 4 words are byte-transposed and each
//    column summed by one dp4a into a 32-bit register sum kept for the whole tile.  E16
//    tables: 16-bit lane sums in registers, flushed to TMEM.  (P4W_TCE = 1, measured slower:
//    the gathered words of 4 k x 4 quads go to a TMEM staging buffer with one tcgen05.st and
//    the tensor core sums them, D[m][n] += sum_j G[m][j] * SEL[j][n] with SEL[j][n] =
//    (j mod 16 == n), G read from TMEM, kind::i8 u8 x u8.)
//  * Each 128-row MMA slice has an issuer (lane 0 of one of its 4 warps, spread over the SM
//    sub-partitions) that issues the slice's exact-part MMAs (M = 128, N = 16, K = 32) per
//    stage -- and the TCE E MMAs -- into one of two TMEM accumulator sets (double-buffered
//    across tiles, so the next tile's MMAs never wait for this tile's epilogue reads); one
//    issuing thread per accumulator keeps them in issue order.  No CTA-wide barrier in the
//    steady state.
//  * Row 32*w + lane of a tile is TMEM lane 32*(w % 4) + lane of MMA slice w / 4, so every
//    consumer warp reads and writes exactly the TMEM lane quarter it may access.
//  * Tile order, stream-K tail (exact int32 pieces in the zero-filled workspace), split-K for
//    raw output and the fused epilogue (tc_common.cuh).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lut_p4.cuh"
#include "tc_common.cuh"

namespace axq {

namespace p4w {
constexpr int PW = 4;                      // producer warps
constexpr int TN = p4::TN;
constexpr int W_STAGE = 512;
constexpr int TMEM_COLS = 512;
// E8: one accumulator set at 0 (exact part + E sums), the E staging buffers from column 128;
// E16: two exact sets at 0 and 128, the E sums at 256
constexpr int STG_COLS = 16;               // one staged chunk: 4 k x 4 quads, 32-bit words
constexpr int STG_BUFS = 3;                // staged chunks per slice
constexpr int STG_BASE = 128;

// CTA shape: CWX consumer warps (one tile row per lane).  28 (896-row tiles, 1024 threads) is
// the default; 16 (512-row tiles, 640 threads) serves small row counts (M <= 1024), where 896-row
// tiles would leave most lanes idle or cut a ragged second tile.
template <int CWX>
struct Shape {
    static constexpr int CW = CWX;                 // consumer warps
    static constexpr int NT = (CW + PW) * 32;      // threads
    static constexpr int BM = CW * 32;             // rows per tile
    static constexpr int SLICES = BM / 128;        // MMA slices of 128 rows
    static constexpr int PT = PW * 32;             // 128 producer threads
    static_assert(BM % 128 == 0, "tile rows must be whole MMA slices");
    static_assert(STG_BASE + SLICES * STG_BUFS * STG_COLS <= TMEM_COLS, "E staging exceeds TMEM");
};
constexpr int CW = 28;
constexpr int BM = CW * 32;                // 896 (host: stream-K partial slots are sized for it)

#ifndef P4W_TCE
#define P4W_TCE 0
#endif
#ifndef P4W_TMA_ON        // A/B builds: 0 compiles the TMA activation loaders out (cp.async only)
#define P4W_TMA_ON 1
#endif
#ifndef P4W_RES_LEAD      // residual rows requested this many stages before the tile's end
#define P4W_RES_LEAD 2
#endif
#ifndef P4W_SMALL_FULL_STAGES
#define P4W_SMALL_FULL_STAGES 3
#endif
// E16 (P4W16, tables whose E = LUT - a*w does not fit int8 but fits int16): a packed word holds
// the biased E of 2 columns (a column pair) instead of 4 (a quad), so NQ = 8 words per k.
template <bool HALF, int KSX = (HALF ? 32 : 16), int CWX = 28, bool E16 = false, bool RESX = false>
struct Geo {
    static constexpr int BM = Shape<CWX>::BM;
    static constexpr int SLICES = Shape<CWX>::SLICES;
    static constexpr int KS = KSX;
    static constexpr int TROWS = HALF ? 128 : 256;
    static constexpr int TQ = TROWS * 4;
    static constexpr int NQ = E16 ? TN / 2 : TN / 4;       // packed words per k
    static constexpr int TBL_STAGE = KS * NQ * TQ;         // 64 KiB
    static constexpr int A_STAGE = BM * KS;                // KS / 16 planes of [BM][16 B]
    // half-range tables in 16-k stages (small-K layers): 4 stages of 32 KiB, a deeper pipeline
    // across the short tiles; the 512-row shape with full-range tables: 3 stages of 64 KiB
    // (few rows per table byte: the table stream, not the lookups, sets the pace); otherwise 2
    static constexpr bool SMALL_FULL = (CWX == 16 && !HALF);
    static constexpr int STAGES = E16 ? 2 : (HALF && KS == 16) ? 4 : SMALL_FULL ? P4W_SMALL_FULL_STAGES : 2;
    // the 4-byte-tap conv loader's tap table (not in the SMALL_FULL shape: no room; the host
    // never picks it for such layers)
    static constexpr bool HAS_TAP = !SMALL_FULL && !E16;
    static constexpr int FLUSH_STAGES = 256 / KS;
    static constexpr int SMEM_TBL = 0;
    static constexpr int SMEM_A = SMEM_TBL + STAGES * TBL_STAGE;
    static constexpr int SMEM_W = SMEM_A + STAGES * A_STAGE;
    static constexpr int SMEM_SEL = SMEM_W + STAGES * W_STAGE;    // E8: the selector SEL (512 B)
    static constexpr int SMEM_ROW = SMEM_SEL + W_STAGE;           // producer row info [BM] x 16 B
    static constexpr int SMEM_BAR = SMEM_ROW + BM * 16;
    // full[S], empty[S], mma[S], tile_full[SLICES][2], tmem_free[SLICES][2],
    // chunk_full[SLICES][STG_BUFS], chunk_free[SLICES][STG_BUFS], then tmem address, flag
    // ... + res_full, res_free (residual-layer shapes with a residual buffer)
    static constexpr int NBAR = 3 * STAGES + 4 * SLICES + 2 * SLICES * STG_BUFS + 2;
    static constexpr int SMEM_MISC = SMEM_BAR + 8 * NBAR;
    static constexpr int SMEM_KC = SMEM_MISC + 16;                 // EpiConst (32 B)
    static constexpr int SMEM_TAP = SMEM_KC + 32;
    static constexpr int SMEM_END = SMEM_TAP + (HAS_TAP ? p4::TAP_BYTES : 0);
    // residual layers whose shape leaves room: the tile's fp32 residual rows [BM][16] staged by
    // TMA (issued by consumer thread 0 as the tile's last stage starts), read from shared memory
    // by the epilogue
    static constexpr int SMEM_RES = (SMEM_END + 1023) / 1024 * 1024;   // 64-byte swizzle atoms
    static constexpr bool RESBUF = RESX && SMEM_RES + BM * 64 <= 232448;
    static constexpr int SMEM_BYTES = RESBUF ? SMEM_RES + BM * 64 : SMEM_END;
    static constexpr int NT_EXTRA = 0;
    static_assert(SMEM_BYTES <= 232448, "P4W shared memory exceeds 227 KiB");
};
}  // namespace p4w

__device__ __forceinline__ void cp_async_mbar_arrive(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}

template <int BM_>
__device__ __forceinline__ void consumer_sync() {   // named barrier 1: the BM_ consumer threads
    asm volatile("bar.sync 1, %0;\n" ::"n"(BM_) : "memory");
}

// RES: a separate instantiation for layers with a residual input, whose epilogue loads the
// residual rows before waiting on the tile's MMAs (their latency overlaps the wait).  Kept out
// of the other layers' instantiation: its extra live registers would spill into their loop.
template <bool HALF, int KSX, bool RES = false, int CWX = 28, bool E16 = false>
__global__ void __launch_bounds__(p4w::Shape<CWX>::NT + p4w::Geo<HALF, KSX, CWX, E16, RES>::NT_EXTRA, 1)
    lut_p4w_kernel(const __grid_constant__ P4Args P) {
    using namespace p4w;
    using G = p4w::Geo<HALF, KSX, CWX, E16, RES>;
    using S = p4w::Shape<CWX>;
    constexpr int CW = S::CW, NT = S::NT, BM = S::BM, SLICES = S::SLICES, PT = S::PT;
    constexpr int KS = G::KS, STAGES = G::STAGES, TBL_STAGE = G::TBL_STAGE, TQ = G::TQ, A_STAGE = G::A_STAGE;
    constexpr int NPL = KS / 16;
    // E8 sums: by dp4a in registers (default) or, with P4W_TCE, on the tensor core from
    // TMEM-staged words (measured slower)
    constexpr bool TCE = !E16 && P4W_TCE;
    constexpr bool DP4 = !E16 && !P4W_TCE;
    extern __shared__ __align__(1024) uint8_t p4w_smem[];
    uint8_t* smem = p4w_smem;
    const MMArgs& p = P.mm;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t s_base = smem_u32(smem);
    const uint32_t bar_full = s_base + G::SMEM_BAR;
    const uint32_t bar_empty = bar_full + 8 * STAGES;
    const uint32_t bar_mma = bar_empty + 8 * STAGES;
    const uint32_t bar_tfull = bar_mma + 8 * STAGES;     // [SLICES][2]
    const uint32_t bar_tfree = bar_tfull + 16 * SLICES;  // [SLICES][2]
    const uint32_t bar_cfull = bar_tfree + 16 * SLICES;  // [SLICES][STG_BUFS]
    const uint32_t bar_cfree = bar_cfull + 8 * SLICES * STG_BUFS;
    const uint32_t bar_rfull = bar_cfree + 8 * SLICES * STG_BUFS, bar_rfree = bar_rfull + 8;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + G::SMEM_MISC);
    int* fin_flag = reinterpret_cast<int*>(smem + G::SMEM_MISC + 4);

    if (G::HAS_TAP && P.c4) {
        uint32_t* tap_w = reinterpret_cast<uint32_t*>(smem + G::SMEM_TAP);
        const int ng = (int)(P.Kp / 4);
        for (int g = tid; g < ng; g += NT) {
            uint32_t e = ~0u;
            if (4 * (int64_t)g < p.K) {
                const int k = 4 * g, rs = k / p.C, c = k - rs * p.C, r = rs / p.S, s_ = rs - r * p.S;
                e = (uint32_t)(r * p.dh) | ((uint32_t)(s_ * p.dw) << 8) | ((uint32_t)c << 16);
            }
            tap_w[g] = e;
        }
    }
    if (KS == 16)   // K chunk 2 of the weight buffers is zero (the MMA's K is 32)
        for (int i = tid; i < STAGES * 64; i += NT)
            reinterpret_cast<uint32_t*>(smem + G::SMEM_W + (i >> 6) * W_STAGE + 256)[i & 63] = 0u;
    if (TCE && tid < 128) {
        // SEL in the K-major canonical layout of the weight stages ((j / 16) * 256 + (n / 8) * 128 +
        // (n % 8) * 16 + j % 16): row n holds a 1 at byte n of both 16-byte K chunks
        const int o = tid * 4, kc = o >> 8, n = ((o >> 7) & 1) * 8 + ((o >> 4) & 7), j0 = o & 15;
        (void)kc;
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) v |= (j0 + b == n ? 1u : 0u) << (8 * b);
        reinterpret_cast<uint32_t*>(smem + G::SMEM_SEL)[tid] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(bar_full + 8 * s, PT + 1);     // the producers' cp.async arrivals + expect_tx
            mbar_init(bar_empty + 8 * s, CW);
            mbar_init(bar_mma + 8 * s, SLICES);      // every slice issuer's commit
        }
        for (int s = 0; s < 2 * SLICES; ++s) {
            mbar_init(bar_tfull + 8 * s, 1);         // the slice issuer's commit
            mbar_init(bar_tfree + 8 * s, 4);         // the slice's 4 consumer warps
        }
        for (int s = 0; s < SLICES * STG_BUFS; ++s) {
            mbar_init(bar_cfull + 8 * s, 4);         // the slice's 4 consumer warps
            mbar_init(bar_cfree + 8 * s, 1);         // the E MMAs' commit
        }
        mbar_init(bar_rfull, 1);                     // the residual copies (expect_tx)
        mbar_init(bar_rfree, CW);                    // every consumer warp read its rows
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // programmatic dependent launch: let the next layer's CTAs start their prologue on SMs this
    // grid frees, and wait here (prologue done) until the previous layer's outputs are complete
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");

    // ---- work decomposition (shared by all roles) ----
    const int64_t m_tiles = (p.M + BM - 1) / BM, n_blocks = (p.N + TN - 1) / TN;
    const int splits = P.splits > 0 ? P.splits : 1;
    const int64_t n_work = m_tiles * n_blocks * splits;
    const int nst_all = (int)(P.Kp / KS);
    const int sps = P.stages_per_split > 0 ? P.stages_per_split : nst_all;
    const bool sk = P.streamk != 0;
    const int64_t G_ = gridDim.x;
    const int64_t t_all = m_tiles * n_blocks;
    // streamk 1: whole waves round-robin, then the tail cut; 2: every (tile, stage) iteration cut
    // into one contiguous slice per CTA (no wave quantisation at a few waves)
    const int64_t t_dp = sk ? (P.streamk == 2 ? 0 : (t_all / G_) * G_) : 0;
    const int64_t it_sk = (t_all - t_dp) * (int64_t)nst_all;
    // the tail is cut among the first G_sk CTAs only (pieces of >= a few stages; the host
    // picks sk_ctas), the rest get empty ranges
    const int64_t G_sk = (P.sk_ctas > 0 && P.sk_ctas < G_) ? P.sk_ctas : G_;
    auto sk_begin = [&](int64_t c) { return t_dp * nst_all + ((c < G_sk ? c : G_sk) * it_sk) / G_sk; };
    struct Gen { int64_t cur, end; bool dp; };
    auto gen_init = [&](Gen& g) {
        g.dp = !sk || t_dp > 0;
        g.cur = blockIdx.x;
        g.end = sk ? t_dp : n_work;
        if (!g.dp) { g.cur = sk_begin(blockIdx.x); g.end = sk_begin(blockIdx.x + 1); }
    };
    auto gen_next = [&](Gen& g, int64_t& t, int& s_b, int& s_e) -> bool {
        if (g.dp) {
            if (g.cur < g.end) {
                const int ks = (int)(g.cur % splits);
                t = g.cur / splits;
                s_b = ks * sps;
                s_e = min(nst_all, s_b + sps);
                g.cur += G_;
                return true;
            }
            if (!sk) return false;
            g.dp = false;
            g.cur = sk_begin(blockIdx.x);
            g.end = sk_begin(blockIdx.x + 1);
        }
        if (g.cur >= g.end) return false;
        t = g.cur / nst_all;
        s_b = (int)(g.cur - t * nst_all);
        const int64_t rem = s_b + (g.end - g.cur);
        s_e = (int)(rem < (int64_t)nst_all ? rem : (int64_t)nst_all);
        g.cur += s_e - s_b;
        return true;
    };
    auto tile_mn = [&](int64_t t, int64_t& nb, int64_t& m0) {
        int64_t mt;
        if (P.nb_fast) { nb = t % n_blocks; mt = t / n_blocks; }
        else { mt = t % m_tiles; nb = t / m_tiles; }
        m0 = mt * BM;
    };

    if (warp >= CW) {
        // =============================== producer warps ===============================
        const int pt = tid - BM;
        const uint32_t* tap_s = reinterpret_cast<const uint32_t*>(smem + G::SMEM_TAP);
        int4* rowinfo = reinterpret_cast<int4*>(smem + G::SMEM_ROW);   // {roff lo, roff hi, hb, wb | valid}
        Gen g;
        gen_init(g);
        int64_t t;
        int s_b, s_e;
        uint32_t item = 0;
        const int64_t pix = p.cs ? p.cs : p.C;    // NHWC pixel stride (grouped conv: all channels)
        while (gen_next(g, t, s_b, s_e)) {
            int64_t nb, m0;
            tile_mn(t, nb, m0);
            // grouped conv: this column tile's group selects its input channels
            const int64_t goff = P.grp_cout ? (nb * TN / P.grp_cout) * P.grp_cin : 0;
#pragma unroll 1
            for (int r = pt; r < ((P4W_TMA_ON && P.tma_a) ? 0 : BM); r += PT) {
                const RowInfo ri = P.is_conv ? make_row<LOAD_CONV>(p, m0 + r) : make_row<LOAD_GEMM>(p, m0 + r);
                const int64_t ro = ri.base + goff + (P.is_conv ? ((int64_t)ri.hb * p.Wd + ri.wb) * pix : 0);
                rowinfo[r] = make_int4((int)(ro & 0xffffffff), (int)(ro >> 32), ri.hb,
                                       ri.valid ? ri.wb : (int)0x80000000);
            }
            // im2col mode: each slice's first output pixel as its window corner (w, h, n), kept
            // in the (otherwise unused) row-info slots, not in registers
            int4* im_crd = rowinfo;
            if (P.tma_a == 2 && pt == 0) {
                const uint32_t hw = (uint32_t)p.Ho * (uint32_t)p.Wo;
#pragma unroll
                for (int j = 0; j < SLICES; ++j) {
                    const int64_t m = m0 + j * 128;
                    const uint32_t mm = (uint32_t)(m < p.M ? m : p.M);   // rows past M: image N (zeros)
                    const uint32_t img = mm / hw, rem = mm - img * hw, ho = rem / (uint32_t)p.Wo,
                                   wo = rem - ho * (uint32_t)p.Wo;
                    im_crd[j] = make_int4((int)wo * p.sw - p.pw, (int)ho * p.sh - p.ph, (int)img, 0);
                }
            }
            int t_r = 0, t_s = 0, t_c = 0;
            if (P.is_conv && !P.c4) {
                const int k0 = s_b * KS, rs = k0 / p.C;
                t_c = k0 - rs * p.C;
                t_r = rs / p.S;
                t_s = rs - t_r * p.S;
            }
            for (int st = s_b; st < s_e; ++st, ++item) {
                const int buf = (int)(item % STAGES);
                if (item >= (uint32_t)STAGES) {
                    const uint32_t ph = ((item / STAGES) - 1) & 1u;
                    mbar_wait(bar_empty + 8 * buf, ph);
                    mbar_wait(bar_mma + 8 * buf, ph);
                }
#pragma unroll
                for (int pl = 0; pl < NPL; ++pl) {
                    const int64_t k0 = (int64_t)st * KS + 16 * pl;
                    const uint32_t dst0 = s_base + G::SMEM_A + buf * A_STAGE + pl * (BM * 16);
                    if (P4W_TMA_ON && P.tma_a) {
                        // one 16 k x 128 row box per MMA slice, issued with the table copies
                    } else if (P.c4) {
                        uint32_t tv[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) tv[j] = tap_s[(int)(k0 >> 2) + j];
#pragma unroll 1
                        for (int r = pt; r < BM; r += PT) {
                            const int4 ri = rowinfo[r];
                            const int64_t ro = (int64_t)(uint32_t)ri.x | ((int64_t)ri.y << 32);
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const int rdh = (int)(tv[j] & 0xffu), sdw = (int)((tv[j] >> 8) & 0xffu);
                                const bool ok = ri.w != (int)0x80000000 && tv[j] != ~0u &&
                                                (unsigned)(ri.z + rdh) < (unsigned)p.H &&
                                                (unsigned)(ri.w + sdw) < (unsigned)p.Wd;
                                const int64_t toff = ((int64_t)rdh * p.Wd + sdw) * pix + (int)(tv[j] >> 16);
                                cp_async4_p(dst0 + r * 16 + 4 * j, ok ? p.A + ro + toff : p.A, ok);
                            }
                        }
                    } else if (P.is_conv) {
                        const int rdh = t_r * p.dh, sdw = t_s * p.dw;
                        // the tap's source base, formed once per plane (pinned in a register: left
                        // to itself the compiler re-derives it per row inside the row's branch)
                        const int8_t* a_tap = p.A + (((int64_t)rdh * p.Wd + sdw) * pix + t_c);
                        asm volatile("" : "+l"(a_tap));
                        const bool kin = k0 < p.K;
                        const unsigned H = (unsigned)p.H, Wd = (unsigned)p.Wd;
#pragma unroll 1
                        for (int r = pt; r < BM; r += PT) {
                            const int4 ri = rowinfo[r];
                            const int64_t ro = (int64_t)(uint32_t)ri.x | ((int64_t)ri.y << 32);
                            const bool ok = kin && ri.w != (int)0x80000000 && (unsigned)(ri.z + rdh) < H &&
                                            (unsigned)(ri.w + sdw) < Wd;
                            cp_async16_p(dst0 + r * 16, ok ? a_tap + ro : p.A, ok);
                        }
                        t_c += 16;
                        if (t_c >= p.C) {
                            t_c = 0;
                            if (++t_s == p.S) { t_s = 0; ++t_r; }
                        }
                    } else {
                        const int64_t rem = p.K - k0;
                        const uint32_t nbytes = rem >= 16 ? 16u : (rem > 0 ? (uint32_t)rem : 0u);
#pragma unroll 1
                        for (int r = pt; r < BM; r += PT) {
                            const int4 ri = rowinfo[r];
                            const int64_t ro = (int64_t)(uint32_t)ri.x | ((int64_t)ri.y << 32);
                            const bool ok = ri.w != (int)0x80000000 && nbytes > 0;
                            if (nbytes == 16u) cp_async16_p(dst0 + r * 16, ok ? p.A + ro + k0 : p.A, ok);
                            else cp_async16(dst0 + r * 16, ok ? p.A + ro + k0 : p.A, ok ? nbytes : 0u);
                        }
                    }
                }
                cp_async_mbar_arrive(bar_full + 8 * buf);
                if (pt == 0) {
                    const uint32_t bar = bar_full + 8 * buf;
                    const uint32_t* tbl_g = P.tables + ((size_t)nb * P.Kp + (size_t)st * KS) * G::NQ * G::TROWS;
                    const int8_t* w_g = P.wpk + ((size_t)nb * (P.Kp / 16) + (size_t)st * NPL) * p4::W_STAGE;
                    mbar_expect_tx(bar, TBL_STAGE + NPL * p4::W_STAGE + ((P4W_TMA_ON && P.tma_a) ? NPL * BM * 16 : 0));
#if P4W_TMA_ON
                    if (P.tma_a == 1) {
#pragma unroll
                        for (int pl = 0; pl < NPL; ++pl)
#pragma unroll 1
                            for (int j = 0; j < SLICES; ++j)
                                tma_load_2d(s_base + G::SMEM_A + buf * A_STAGE + pl * (BM * 16) + j * 128 * 16,
                                            &P.tmap_a, st * KS + 16 * pl, (int)(m0 + j * 128), bar);
                    } else if (P.tma_a == 2) {
#pragma unroll
                        for (int pl = 0; pl < NPL; ++pl) {
                            // plane k0 = (r * S + s) * C + c: tap (r, s), channels c .. c + 15;
                            // planes past K read channel C (out of range: zeros)
                            const int k0 = st * KS + 16 * pl;
                            const int rs = k0 / p.C, c = k0 < p.K ? k0 - rs * p.C : (p.cs ? p.cs : p.C);
                            const int r = rs / p.S, s_ = rs - r * p.S;
#pragma unroll 1
                            for (int j = 0; j < SLICES; ++j) {
                                const int4 cj = im_crd[j];
                                tma_load_im2col(s_base + G::SMEM_A + buf * A_STAGE + pl * (BM * 16) + j * 128 * 16,
                                                &P.tmap_a, c, cj.x, cj.y, cj.z, (uint16_t)(s_ * p.dw),
                                                (uint16_t)(r * p.dh), bar);
                            }
                        }
                    }
#endif
                    bulk_g2s(s_base + G::SMEM_TBL + buf * TBL_STAGE, tbl_g, TBL_STAGE, bar);
                    bulk_g2s(s_base + G::SMEM_W + buf * W_STAGE, w_g, NPL * p4::W_STAGE, bar);
                }
            }
        }
    } else {
        // =============================== consumer warps ===============================
        const uint32_t t_lane = (uint32_t)((warp & 3) * 32) << 16;
        const int slice = warp >> 2;
        const uint32_t slice_col = (uint32_t)slice * TN;
        const uint32_t t_e = tmem + t_lane + 256u + slice_col;                                   // E16 sums
        const uint32_t t_stg = tmem + t_lane + STG_BASE + (uint32_t)(slice * STG_BUFS) * STG_COLS;   // E8 staging
        const uint32_t c_full = bar_cfull + 8 * slice * STG_BUFS, c_free = bar_cfree + 8 * slice * STG_BUFS;
        const uint32_t t_full = bar_tfull + 16 * slice, t_free = bar_tfree + 16 * slice;
        // the slice issuer (lane 0 of one of its 4 warps, spread over the 4 SM sub-partitions)
        // issues every MMA into the slice's accumulators -- exact part and E sums -- so they
        // execute in its issue order
        const bool iss_warp = (warp & 3) == (slice & 3);
        const bool issuer = iss_warp && lane == 0;
        constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TN >> 3) << 17) | ((128u >> 4) << 24);
        constexpr uint32_t IDESC_E = (2u << 4) | ((uint32_t)(TN >> 3) << 17) | ((128u >> 4) << 24);   // u8 x u8
        // per-launch epilogue scalars: loaded once into shared memory (not held in registers
        // across the lookup loop)
        EpiConst& kconst = *reinterpret_cast<EpiConst*>(smem + G::SMEM_KC);
        if (tid == 0) kconst = p4t_epi_const(P);
        consumer_sync<BM>();
        Gen g;
        gen_init(g);
        int64_t tile;
        int s_b, s_e;
        uint32_t item = 0, tcount = 0, chunk = 0, rcount = 0;
        bool pend = false;   // the issuer's staged chunk chunk - 1 is not summed yet
        while (gen_next(g, tile, s_b, s_e)) {
            int64_t nb, m0;
            tile_mn(tile, nb, m0);
            const int64_t n0 = nb * TN;
            // accumulator sets: E8 one (the slice's warps meet at each tile boundary anyway: the
            // next tile's E MMAs need all 4 warps' staged words), E16 two
            constexpr uint32_t NSET = TCE ? 1u : 2u;
            // DP4: iacc[q][j] = sum of column 4q + j's biased bytes, 32-bit, for the whole tile
            uint32_t iacc[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) iacc[q][0] = iacc[q][1] = iacc[q][2] = iacc[q][3] = 0u;
            const uint32_t tb = tcount % NSET, tph = (tcount / NSET) & 1u;
            const bool wlive = m0 + warp * 32 < p.M;
            // E16: per column pair q, pacc[q][0] = sum v (mod 2^32) and pacc[q][1] = sum (v >> 16);
            // the low column's sum is pacc[q][0] - 2^16 pacc[q][1] (mod 2^32, exact: both sums < 2^32)
            uint32_t pacc[8][2];
#pragma unroll
            for (int q = 0; q < 8; ++q) pacc[q][0] = pacc[q][1] = 0u;
            bool e_first = true;
            const uint32_t d_acc = tmem + tb * 128u + slice_col;   // the slice's accumulator (set tb)
            // E MMAs of staged chunk c: D += G * SEL, G = the slice's 128 rows x 64 staged bytes
            auto issue_e = [&](uint32_t c) {
                const uint32_t b = c % STG_BUFS;
                mbar_wait(c_full + 8 * b, (c / STG_BUFS) & 1u);
                tc_fence_after();
                const uint32_t a_t = tmem + STG_BASE + (uint32_t)(slice * STG_BUFS + b) * STG_COLS;
                const uint64_t sel = umma_desc_kmajor(s_base + G::SMEM_SEL, 256u, 128u);
                umma_i8_ts(d_acc, a_t, sel, IDESC_E, 1u);
                umma_i8_ts(d_acc, a_t + 8u, sel, IDESC_E, 1u);
                umma_commit(c_free + 8 * b);
            };
            for (int st = s_b; st < s_e; ++st, ++item) {
                const int buf = (int)(item % STAGES);
                mbar_wait(bar_full + 8 * buf, (item / STAGES) & 1u);
                if (iss_warp) {
                    if (issuer) {
                        if (st == s_b && tcount >= NSET) mbar_wait(t_free + 8 * tb, tph ^ 1u);
                        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // cp.async data -> MMA
                        tc_fence_after();
                        const uint32_t a0 = s_base + G::SMEM_A + buf * A_STAGE + slice * 128 * 16;
                        umma_i8(d_acc, umma_desc_kmajor(a0, KS == 32 ? (uint32_t)(BM * 16) : 0u, 128u),
                                umma_desc_kmajor(s_base + G::SMEM_W + buf * W_STAGE, 256u, 128u), IDESC,
                                st == s_b ? 0u : 1u);
                        umma_commit(bar_mma + 8 * buf);
                    }
                    __syncwarp();
                }
                if (G::RESBUF && P.tma_res && tid == 0 && st == (s_e - P4W_RES_LEAD > s_b ? s_e - P4W_RES_LEAD : s_b)) {
                    // the tile's residual rows: one 16-column x 128-row fp32 box per slice, once
                    // every warp has read the previous piece's (res_free)
                    if (rcount > 0) mbar_wait(bar_rfree, (rcount - 1) & 1u);
                    mbar_expect_tx(bar_rfull, BM * 64);
#pragma unroll 1
                    for (int j = 0; j < SLICES; ++j)
                        tma_load_2d(s_base + G::SMEM_RES + j * 128 * 64, &P.tmap_res, (int)n0, (int)(m0 + j * 128),
                                    bar_rfull);
                }
                // shared-window address of this stage's tables: one IMAD per code forms the row
                // address, the (k, quad) offsets are immediates of the loads
                const uint32_t tb_addr = s_base + G::SMEM_TBL + (uint32_t)(buf * TBL_STAGE);
                const uint8_t* at = smem + G::SMEM_A + buf * A_STAGE;
#pragma unroll
                for (int pl = 0; pl < NPL; ++pl) {
                    uint4 av = make_uint4(0u, 0u, 0u, 0u);
                    if (wlive) av = *reinterpret_cast<const uint4*>(at + pl * (BM * 16) + tid * 16);
                    const uint32_t aw[4] = {av.x, av.y, av.z, av.w};
                    if constexpr (TCE) {
                        // one chunk = 4 k: the 16 words (k, quad) of the row go to staging column
                        // 4 k + quad; the slice's E MMA sums column bytes j with j mod 16 == n
#pragma unroll
                        for (int kk = 0; kk < 16; kk += 4) {
                            const uint32_t b = chunk % STG_BUFS;
                            if (chunk >= (uint32_t)STG_BUFS) {
                                mbar_wait(c_free + 8 * b, ((chunk / STG_BUFS) - 1) & 1u);
                                tc_fence_after();
                            }
                            if (wlive) {
                                uint32_t ra[4], v[16];
#pragma unroll
                                for (int i = 0; i < 4; ++i)
                                    ra[i] = tb_addr + __byte_perm(aw[kk >> 2], 0u, 0x4440u + i) * 4u;
#pragma unroll
                                for (int i = 0; i < 4; ++i)
#pragma unroll
                                    for (int q = 0; q < 4; ++q)
                                        asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v[4 * i + q])
                                                     : "r"(ra[i] + (uint32_t)(((pl * 16 + kk + i) * G::NQ + q) * TQ)));
                                tmem_st16(t_stg + b * STG_COLS, v);
                                tmem_wait_st();
                            }
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(c_full + 8 * b);
                            // the issuer sums the PREVIOUS chunk (its 4 warps have most likely
                            // staged it by now), so it rarely waits on its slice
                            if (iss_warp) {
                                if (issuer && pend) issue_e(chunk - 1u);
                                __syncwarp();
                            }
                            pend = true;
                            ++chunk;
                        }
                    } else if (DP4 && wlive) {
                        // 4 k at a time: per quad the 4 words (k .. k+3) are transposed into one
                        // word per column (6 PRMT) and summed by one dp4a each
#pragma unroll
                        for (int kk = 0; kk < 16; kk += 4) {
                            uint32_t ra[4];
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                ra[i] = tb_addr + __byte_perm(aw[kk >> 2], 0u, 0x4440u + i) * 4u;
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                uint32_t v[4];
#pragma unroll
                                for (int i = 0; i < 4; ++i)
                                    asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v[i])
                                                 : "r"(ra[i] + (uint32_t)(((pl * 16 + kk + i) * G::NQ + q) * TQ)));
                                const uint32_t t0 = __byte_perm(v[0], v[1], 0x5140u);   // c0 k0, c0 k1, c1 k0, c1 k1
                                const uint32_t t1 = __byte_perm(v[2], v[3], 0x5140u);   // c0 k2, c0 k3, c1 k2, c1 k3
                                const uint32_t t2 = __byte_perm(v[0], v[1], 0x7362u);   // c2 ..., c3 ...
                                const uint32_t t3 = __byte_perm(v[2], v[3], 0x7362u);
                                iacc[q][0] = __dp4a(__byte_perm(t0, t1, 0x5410u), 0x01010101u, iacc[q][0]);
                                iacc[q][1] = __dp4a(__byte_perm(t0, t1, 0x7632u), 0x01010101u, iacc[q][1]);
                                iacc[q][2] = __dp4a(__byte_perm(t2, t3, 0x5410u), 0x01010101u, iacc[q][2]);
                                iacc[q][3] = __dp4a(__byte_perm(t2, t3, 0x7632u), 0x01010101u, iacc[q][3]);
                            }
                        }
                    } else if (E16 && wlive) {
#pragma unroll
                        for (int kk = 0; kk < 16; kk += 2) {
                            const uint32_t ua0 = __byte_perm(aw[kk >> 2], 0u, 0x4440u + (kk & 3));
                            const uint32_t ua1 = __byte_perm(aw[kk >> 2], 0u, 0x4440u + ((kk + 1) & 3));
                            const uint32_t r0 = tb_addr + ua0 * 4u, r1 = tb_addr + ua1 * 4u;
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                uint32_t v0, v1;
                                asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v0)
                                             : "r"(r0 + (uint32_t)(((pl * 16 + kk) * G::NQ + q) * TQ)));
                                asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v1)
                                             : "r"(r1 + (uint32_t)(((pl * 16 + kk + 1) * G::NQ + q) * TQ)));
                                pacc[q][0] += v0 + v1;
                                pacc[q][1] += __byte_perm(v0, 0u, 0x4432u) + __byte_perm(v1, 0u, 0x4432u);
                            }
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_empty + 8 * buf);
                if (E16 && ((st - s_b + 1) % G::FLUSH_STAGES == 0 || st + 1 == s_e)) {
                    // E16: the 16-bit lane sums, decoded, are added into TMEM every 256 k
                    uint32_t ev[16];
                    if (!e_first) {
                        tmem_ld16(t_e, ev);
                        tmem_wait_ld();
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j) ev[j] = 0u;
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        ev[2 * q + 0] += pacc[q][0] - (pacc[q][1] << 16);
                        ev[2 * q + 1] += pacc[q][1];
                        pacc[q][0] = pacc[q][1] = 0u;
                    }
                    tmem_st16(t_e, ev);
                    tmem_wait_st();
                    e_first = false;
                }
            }
            if (iss_warp) {
                if (issuer) {
                    if (pend) issue_e(chunk - 1u);
                    umma_commit(t_full + 8 * tb);
                }
                __syncwarp();
            }
            pend = false;
            int corr = (E16 ? 32768 : p4::E_BIAS) * KS * (s_e - s_b);
            if (s_e == nst_all) corr += (int)(((P.Kp - p.K) + p.pad_lookups) * (int64_t)p.t00);
            // the row's residual groups: issued before the wait on the tile's MMAs, so their
            // latency overlaps it (the K loop's registers are free here)
            const int64_t m_row = m0 + tid;
            const bool pre = RES && m_row < p.M &&
                             (kconst.mode == EPI_RES_RELU_Y_Q ? n0 + TN <= p.N
                                                               : p.ep.residual != nullptr && p4t_vec_ok(P, n0));
            float4 res[TN / 4];
            // residual rows staged by TMA: row tid, 16-byte chunk j at j ^ ((tid >> 1) & 3) (the
            // tensor maps' 64-byte swizzle: conflict-free row reads); with P.tma_y the block's y
            // goes back into the same rows and out through a TMA store per slice
            const int swz = (tid >> 1) & 3;
            float4* rrow = reinterpret_cast<float4*>(smem + G::SMEM_RES + tid * 64);
            const bool tres = G::RESBUF && P.tma_res;
            if (tres) {
                mbar_wait(bar_rfull, rcount & 1u);
                if (pre) {
#pragma unroll
                    for (int j = 0; j < TN / 4; ++j) res[j] = rrow[j ^ swz];
                }
                if (!P.tma_y) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar_rfree);
                }
                ++rcount;
            } else if (pre) {
                const float4* rp = reinterpret_cast<const float4*>(p.ep.residual + m_row * p.ep.ldr + n0);
#pragma unroll
                for (int j = 0; j < TN / 4; ++j) res[j] = __ldg(rp + j);
            }
            // this tile's sums: TMEM set tb (exact part + E sums for TCE), complete once tile_full[tb] flips
            mbar_wait(t_full + 8 * tb, tph);
            tc_fence_after();
            uint32_t ex[16], es[16];
            tmem_ld16(d_acc + t_lane, ex);
            if constexpr (TCE) {
#pragma unroll
                for (int j = 0; j < 16; ++j) es[j] = 0u;
            } else if constexpr (DP4) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int j = 0; j < 4; ++j) es[4 * q + j] = iacc[q][j];
            } else {
                tmem_ld16(t_e, es);
            }
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(t_free + 8 * tb);   // set tb may be overwritten
            ++tcount;
            int eacc[16];
#pragma unroll
            for (int n = 0; n < 16; ++n) eacc[n] = (int)(ex[n] + es[n]) - corr;
            const int64_t m = m0 + tid;
            // y by TMA store (residual-mode fast epilogue, whole column tile): each slice's 4 warps
            // write their rows, then the slice issuer stores the 16 x 128 box; the residual
            // buffer is released once every slice's store has read it
            const bool ystore = tres && P.tma_y && kconst.mode == EPI_RES_RELU_Y_Q && n0 + TN <= p.N &&
                                (splits == 1 || sk);
            float4* ys = (ystore) ? rrow : nullptr;
            auto ystore_done = [&](bool wrote) {
                if (wrote) {
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    asm volatile("bar.sync %0, 128;\n" ::"r"(2 + slice) : "memory");
                    if (issuer) {
                        tma_store_2d(&P.tmap_y, (int)n0, (int)(m0 + slice * 128),
                                     s_base + G::SMEM_RES + slice * 128 * 64);
                        bulk_commit_wait_read();
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_rfree);
            };
            if (tres && P.tma_y && !ystore) {     // residual read, y not staged: release now
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_rfree);
            }
            if (sk && !(s_b == 0 && s_e == nst_all)) {
                // a stream-K piece: park it in this CTA's partial slot (0: the first piece of its
                // range, 1: the last); the contributor completing the tile's stage count sums
                // the other contributors' slots (exact int32) and runs the epilogue
                const int64_t x0 = t_dp * nst_all + (tile - t_dp) * nst_all;   // tile's first iteration
                const int64_t my_b = sk_begin(blockIdx.x);
                const int slot = my_b >= x0 ? 0 : 1;
                int4* part = reinterpret_cast<int4*>(P.ws + (((int64_t)blockIdx.x * 2 + slot) * BM + tid) * TN);
#pragma unroll
                for (int j = 0; j < TN / 4; ++j)
                    __stcg(part + j, make_int4(eacc[4 * j], eacc[4 * j + 1], eacc[4 * j + 2], eacc[4 * j + 3]));
                __threadfence();
                consumer_sync<BM>();
                int64_t c_first = ((x0 - t_dp * nst_all) * G_sk) / it_sk;
                while (c_first + 1 < G_sk && sk_begin(c_first + 1) <= x0) ++c_first;
                if (tid == 0) {
                    const int old = atomicAdd(P.cnt + c_first, s_e - s_b);
                    const int fin = (old + (s_e - s_b) == nst_all) ? 1 : 0;
                    if (fin) P.cnt[c_first] = 0;
                    *fin_flag = fin;
                }
                consumer_sync<BM>();
                const int fin = *fin_flag;
                consumer_sync<BM>();   // fin_flag is reused by the next piece
                if (fin) {
                    __threadfence();
                    const int64_t x1 = x0 + nst_all;   // one past the tile's last iteration
                    for (int64_t c = c_first; c < G_sk && sk_begin(c) < x1; ++c) {
                        const int64_t cb = sk_begin(c);
                        if (c == blockIdx.x || cb == sk_begin(c + 1)) continue;   // self / empty range
                        const int4* op = reinterpret_cast<const int4*>(
                            P.ws + (((int64_t)c * 2 + (cb >= x0 ? 0 : 1)) * BM + tid) * TN);
#pragma unroll
                        for (int j = 0; j < TN / 4; ++j) {
                            const int4 v = __ldcg(op + j);
                            eacc[4 * j] += v.x; eacc[4 * j + 1] += v.y; eacc[4 * j + 2] += v.z; eacc[4 * j + 3] += v.w;
                        }
                    }
                    if (m < p.M) p4t_store_row<RES>(P, m, n0, eacc, 1, kconst, pre ? res : nullptr, ys, swz);
                }
                if (ystore && !fin) ystore_done(false);
                else if (ystore) ystore_done(true);
            } else {
                if (m < p.M) p4t_store_row<RES>(P, m, n0, eacc, splits, kconst, pre ? res : nullptr, ys, swz);
                if (ystore) ystore_done(true);
            }
        }
    }
    if (G::RESBUF && P.tma_y) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");   // y stores done
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS)
                     : "memory");
    }
}

}  // namespace axq

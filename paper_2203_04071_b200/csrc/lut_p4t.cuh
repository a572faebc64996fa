// lut_p4t.cuh -- "P4T": the P4 LUT-GEMM / implicit-im2col LUT-conv (lut_p4.cuh) with the
// exact part of the delta8 split on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// Same result as lut_p4.cuh / lut_mm.cuh: acc[m][n] = sum_k LUT[a[m][k]][w[n][k]] in int32,
// exact, computed as  sum_k a*w  +  sum_k E[a][w]  with E = LUT - a*w (int8, delta8).
//
//  * sum_k a*w (a dense int8 contraction): one elected thread issues, per 16-k stage,
//    tcgen05.mma.cta_group::1.kind::i8 (M = 128, N = 16, K = 32) for each 128-row slice of the
//    CTA tile, operands read from the staged shared-memory tiles through SWIZZLE_NONE K-major
//    descriptors.  K = 32 is the instruction's fixed depth; the stage holds 16 k, so the B
//    descriptor's second 16-byte K chunk points at 256 zero bytes (the A descriptor's second
//    chunk re-reads the first, multiplied by those zeros).  Accumulators live in TMEM
//    (columns [0, 128)), not registers.
//  * sum_k E: as in P4, one 32-bit LDS of the weight-specialised packed table serves 4
//    lookups; packed 16-bit sums are flushed every 256 k into TMEM columns [128, 256)
//    (tcgen05.ld / add / tcgen05.st by the owning warp).
//  * With no register accumulators for the exact part, the CTA runs 32 warps (1024 threads,
//    one output row per lane, 1024 x 16 CTA tile): twice the warps per scheduler of P4, so
//    the lookup stream's latency is hidden by occupancy.  Row 32*w + lane of the tile is
//    TMEM lane 32*(w % 4) + lane of MMA slice w / 4: each warp reads exactly the TMEM lane
//    quarter it may access.
//  * Staging, tile order, implicit im2col loaders, split-K and the fused epilogue are P4's.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lut_p4.cuh"

namespace axq {

namespace p4t {
constexpr int WARPS = 32;
constexpr int NT = WARPS * 32;             // 1024 threads
constexpr int BM = NT;                     // 1024 rows per CTA tile, one per lane
constexpr int TN = p4::TN;                 // 16 columns
constexpr int W_STAGE = 512;               // [2 K chunks][16 n][16 k] (KS = 16: chunk 2 zero)
constexpr int TMEM_COLS = 256;             // [0,128): exact part, [128,256): E sums

// KS = k per stage: 32 for half-range tables (64 KiB per stage), 16 for full-range ones.
template <bool HALF, int KS>
struct Geo {
    static constexpr int TROWS = HALF ? 128 : 256;
    static constexpr int TQ = TROWS * 4;
    static constexpr int TBL_STAGE = KS * (TN / 4) * TQ;   // 64 KiB (32 KiB for HALF, KS 16)
    static constexpr int A_STAGE = BM * KS;                // KS / 16 planes of [BM][16 B]
    static constexpr int STAGES = (HALF && KS == 16) ? 4 : 2;
    static constexpr int FLUSH_STAGES = 256 / KS;          // 16-bit packed sums: every 256 k
    static constexpr int SMEM_TBL = 0;
    static constexpr int SMEM_A = SMEM_TBL + STAGES * TBL_STAGE;
    static constexpr int SMEM_W = SMEM_A + STAGES * A_STAGE;
    static constexpr int SMEM_BAR = SMEM_W + STAGES * W_STAGE;   // full[S], mma[S], tile, tmem addr
    static constexpr int SMEM_TAP = SMEM_BAR + 8 * (2 * STAGES + 2);
    static constexpr int SMEM_BYTES = SMEM_TAP + p4::TAP_BYTES;
};
template <bool HALF>
__host__ __device__ constexpr int ks_of() { return HALF ? 32 : 16; }
}  // namespace p4t

// ---- tcgen05 helpers ----
__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // SWIZZLE_NONE K-major canonical layout: core matrices of 8 rows x 16 B (rows 16 B apart);
    // LBO = byte distance between the two K chunks, SBO = between 8-row groups; version 1.
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | ((uint64_t)1 << 46);
}

__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// Output of one lane's row (16 columns, int32 totals in v): raw / atomic int32 or the fused
// epilogue (P4's, one row per lane).
// Per-launch epilogue constants (loaded once per CTA, not per tile).
struct EpiConst {
    float sc, s_out, qm, r_out;   // r_out = RN(1 / s_out) for epi_quant_r
};
__device__ __forceinline__ EpiConst p4t_epi_const(const P4Args& P) {
    const EpiArgs& e = P.mm.ep;
    EpiConst k{0.f, 1.f, 127.f, 1.f};
    if (P.mm.C_out == nullptr) {
        k.sc = __fmul_rn(*e.sa, *e.sw);
        k.s_out = e.q ? *e.s_out : 1.f;
        k.qm = (float)((1 << ((e.q ? e.bits_out : 8) - 1)) - 1);
        k.r_out = __frcp_rn(k.s_out);
    }
    return k;
}

// the row-layout vector epilogue applies (16-byte aligned fp32 rows, 4-byte aligned codes)
__device__ __forceinline__ bool p4t_vec_ok(const P4Args& P, int64_t n0) {
    const MMArgs& p = P.mm;
    const EpiArgs& e = p.ep;
    return !P.transposed && p.C_out == nullptr && (n0 + p4::TN <= p.N) && !e.y_nchw &&
           (!e.y || (((e.ldy & 3) == 0) && ((reinterpret_cast<uintptr_t>(e.y) & 15) == 0))) &&
           (!e.residual || (((e.ldr & 3) == 0) && ((reinterpret_cast<uintptr_t>(e.residual) & 15) == 0))) &&
           (!e.bias || ((reinterpret_cast<uintptr_t>(e.bias) & 15) == 0)) &&
           (!e.q || (((e.ldq & 3) == 0) && ((reinterpret_cast<uintptr_t>(e.q) & 3) == 0)));
}

template <bool FASTQ = false>
__device__ __forceinline__ void p4t_store_row(const P4Args& P, int64_t m, int64_t n0, const int (&eacc)[16],
                                              int splits, const EpiConst& kc, const float4* res_pre);

__device__ __forceinline__ void p4t_store_row(const P4Args& P, int64_t m, int64_t n0, const int (&eacc)[16],
                                              int splits) {
    p4t_store_row<false>(P, m, n0, eacc, splits, p4t_epi_const(P), nullptr);
}

// res_pre: the row's 4 residual float4 groups already loaded (vector path only), or null.
// FASTQ: requantize through the reciprocal (epi_quant_r) -- used by the residual-layer
// instantiation only (elsewhere its registers cost more than the division it saves)
template <bool FASTQ>
__device__ __forceinline__ void p4t_store_row(const P4Args& P, int64_t m, int64_t n0, const int (&eacc)[16],
                                              int splits, const EpiConst& kc, const float4* res_pre) {
    using namespace p4;
    const MMArgs& p = P.mm;
    const EpiArgs& e = p.ep;
    if (P.transposed) {
        // axq_lut_gemm_xs: rows are weight rows (bias / per-channel scale index), columns are
        // activation rows; lanes = consecutive weight rows -> coalesced along the output row
        if (p.C_out != nullptr) {
#pragma unroll
            for (int n = 0; n < TN; ++n)
                if (n0 + n < p.N) p.C_out[(n0 + n) * p.ldc + m] = eacc[n];
            return;
        }
        const float sc_r = e.sw_ch ? __fmul_rn(*e.sa, e.sw_ch[m]) : __fmul_rn(*e.sa, *e.sw);
        const float b = e.bias ? e.bias[m] : 0.f;
        const float s_out = e.q ? *e.s_out : 1.f;
        const float qm = (float)((1 << ((e.q ? e.bits_out : 8) - 1)) - 1);
#pragma unroll
        for (int n = 0; n < TN; ++n) {
            const int64_t nn = n0 + n;
            if (nn >= p.N) continue;
            float v = __fmul_rn(__int2float_rn(eacc[n]), sc_r);
            if (e.bias) v = __fadd_rn(v, b);
            if (e.residual) v = __fadd_rn(v, e.residual[nn * e.ldr + m]);
            if (e.relu) v = v > 0.f ? v : 0.f;
            if (e.y) e.y[nn * e.ldy + m] = v;
            if (e.q) e.q[nn * e.ldq + m] = epi_quant(v, s_out, qm);
        }
        return;
    }
    if (p.C_out != nullptr) {
        int32_t* c = p.C_out + m * p.ldc + n0;
        if (splits > 1) {
#pragma unroll
            for (int n = 0; n < TN; ++n)
                if (n0 + n < p.N) atomicAdd(c + n, eacc[n]);
        } else {
#pragma unroll
            for (int n = 0; n < TN; ++n)
                if (n0 + n < p.N) c[n] = eacc[n];
        }
        return;
    }
    const float sc = kc.sc, s_out = kc.s_out, qm = kc.qm;
    const bool vec = p4t_vec_ok(P, n0);
    if (vec) {
        const bool q16 = e.q && ((e.ldq & 15) == 0) && ((reinterpret_cast<uintptr_t>(e.q) & 15) == 0);
        // residual groups are loaded one ahead (8 live registers, not 16: the P4W consumer
        // runs at 64 registers per thread)
        const float4* rp = (e.residual && !res_pre) ? reinterpret_cast<const float4*>(e.residual + m * e.ldr + n0)
                                                    : nullptr;
        float4 rnext = res_pre ? res_pre[0] : (rp ? __ldg(rp) : make_float4(0.f, 0.f, 0.f, 0.f));
        uint32_t qw[TN / 4];
#pragma unroll
        for (int n = 0; n < TN; n += 4) {
            const float4 rcur = rnext;
            if (n + 4 < TN) {
                if (res_pre) rnext = res_pre[(n + 4) / 4];
                else if (rp) rnext = __ldg(rp + (n + 4) / 4);
            }
            const int64_t nn = n0 + n;
            float v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = __fmul_rn(__int2float_rn(eacc[n + j]), epi_sc(e, sc, nn + j));
            if (e.bias) {
                const float4 b = *reinterpret_cast<const float4*>(e.bias + nn);
                v[0] = __fadd_rn(v[0], b.x); v[1] = __fadd_rn(v[1], b.y);
                v[2] = __fadd_rn(v[2], b.z); v[3] = __fadd_rn(v[3], b.w);
            }
            if (e.residual) {
                const float4 rr = rcur;
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
                for (int j = 0; j < 4; ++j)
                    w |= (uint32_t)(uint8_t)(FASTQ ? epi_quant_r(v[j], s_out, kc.r_out, qm) : epi_quant(v[j], s_out, qm))
                         << (8 * j);
                qw[n / 4] = w;
                if (!q16) *reinterpret_cast<uint32_t*>(e.q + m * e.ldq + nn) = w;
            }
        }
        if (e.q && q16) *reinterpret_cast<uint4*>(e.q + m * e.ldq + n0) = make_uint4(qw[0], qw[1], qw[2], qw[3]);
    } else if (e.y_nchw) {
        // NCHW fp32 output: lanes are consecutive pixels (coalesced per column)
        const int64_t img = m / e.hw, pix = m - img * e.hw;
        float* yb = e.y ? e.y + (img * p.N + n0) * e.hw + pix : nullptr;
#pragma unroll
        for (int n = 0; n < TN; ++n) {
            const int64_t nn = n0 + n;
            if (nn < p.N) {
                const float v = epi_value(eacc[n], m, nn, sc, e);
                if (yb) __stcs(yb + n * e.hw, v);
                if (e.q) e.q[m * e.ldq + nn] = epi_quant(v, s_out, qm);
            }
        }
    } else {
#pragma unroll
        for (int n = 0; n < TN; ++n) {
            const int64_t nn = n0 + n;
            if (nn < p.N) epi_store(epi_value(eacc[n], m, nn, sc, e), m, nn, p.N, e, s_out, qm);
        }
    }
}

template <bool HALF>
__global__ void __launch_bounds__(p4t::NT, 1) lut_p4t_kernel(const __grid_constant__ P4Args P) {
    using namespace p4t;
    constexpr int KS = ks_of<HALF>();
    using G = p4t::Geo<HALF, KS>;
    constexpr int STAGES = G::STAGES, TBL_STAGE = G::TBL_STAGE, TQ = G::TQ, A_STAGE = G::A_STAGE;
    constexpr int NPL = KS / 16;               // activation planes per stage
    constexpr int SMEM_TBL = G::SMEM_TBL, SMEM_A = G::SMEM_A, SMEM_W = G::SMEM_W;
    extern __shared__ __align__(1024) uint8_t p4t_smem[];
    uint8_t* smem = p4t_smem;
    const MMArgs& p = P.mm;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t s_base = smem_u32(smem);
    const uint32_t bar_full = s_base + G::SMEM_BAR;              // [STAGES] tables + weights landed
    const uint32_t bar_mma = bar_full + 8 * STAGES;              // [STAGES] MMA done reading buffer
    const uint32_t bar_tile = bar_mma + 8 * STAGES;              // tile's MMAs done
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + G::SMEM_BAR + 8 * (2 * STAGES + 1));

    if (P.c4) {
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
    // KS = 16: zero K chunk 2 of every weight buffer (read by the MMA through the async proxy)
    if (KS == 16)
        for (int i = tid; i < STAGES * 64; i += NT)
            reinterpret_cast<uint32_t*>(smem + SMEM_W + (i >> 6) * W_STAGE + 256)[i & 63] = 0u;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    if (tid == 0) {
        for (int s = 0; s < 2 * STAGES + 1; ++s) mbar_init(bar_full + 8 * s, 1);
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
    // this warp's TMEM rows: lane quarter warp % 4, MMA slice warp / 4
    const uint32_t t_row = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t t_exact = t_row + (uint32_t)(warp >> 2) * TN;
    const uint32_t t_e = t_row + 128u + (uint32_t)(warp >> 2) * TN;
    // i8 MMA instruction descriptor: s32 accumulate, s8 x s8, K-major A and B, N = 16, M = 128
    constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TN >> 3) << 17) | ((128u >> 4) << 24);

    const int64_t m_tiles = (p.M + BM - 1) / BM, n_blocks = (p.N + TN - 1) / TN;
    const int splits = P.splits > 0 ? P.splits : 1;
    const int64_t n_work = m_tiles * n_blocks * splits;
    const int nst_all = (int)(P.Kp / KS);
    const int sps = P.stages_per_split > 0 ? P.stages_per_split : nst_all;
    // Stream-K (fused epilogue with a workspace), data-parallel + stream-K hybrid: the whole
    // waves of tiles run round-robin (concurrent CTAs share one table stream); the T % grid
    // tail tiles' (tile, stage) iterations are cut into gridDim.x equal contiguous ranges.  A
    // tail tile cut by a range boundary is summed exactly in the int32 workspace and finished
    // by whichever contributor completes its stage count.
    const bool sk = P.streamk != 0;
    const int64_t G_ = gridDim.x;
    const int64_t t_all = m_tiles * n_blocks;
    const int64_t t_dp = sk ? (t_all / G_) * G_ : 0;
    const int64_t it_sk = (t_all - t_dp) * (int64_t)nst_all;
    auto sk_begin = [&](int64_t c) { return t_dp * nst_all + (c * it_sk) / G_; };

    // segments: (tile, stage range) in this CTA's order; cur < 0 encodes the round-robin phase
    struct Gen { int64_t cur, end; bool dp; };
    auto gen_init = [&](Gen& g) {
        if (sk) { g.dp = t_dp > 0; g.cur = blockIdx.x; g.end = t_dp; if (!g.dp) { g.cur = sk_begin(blockIdx.x); g.end = sk_begin(blockIdx.x + 1); } }
        else { g.dp = true; g.cur = blockIdx.x; g.end = n_work; }
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

    // ---- producer: a flat per-CTA stream of (tile, stage) items over STAGES buffers ----
    Gen pg;
    gen_init(pg);
    int64_t i_t = 0, i_nb = 0, i_m0 = 0;
    int i_st = 0, i_se = 0;
    bool i_done = false;
    int t_r = 0, t_s = 0, t_c = 0;
    RowInfo irow;
    int64_t roff = 0;
    auto set_issue_tile = [&]() {
        if (!gen_next(pg, i_t, i_st, i_se)) { i_done = true; return; }
        tile_mn(i_t, i_nb, i_m0);
        irow = P.is_conv ? make_row<LOAD_CONV>(p, i_m0 + tid) : make_row<LOAD_GEMM>(p, i_m0 + tid);
        roff = irow.base + (P.is_conv ? ((int64_t)irow.hb * p.Wd + irow.wb) * p.C : 0);
        if (P.is_conv && !P.c4) {
            const int k0 = i_st * KS, rs = k0 / p.C;
            t_c = k0 - rs * p.C;
            t_r = rs / p.S;
            t_s = rs - t_r * p.S;
        }
    };
    const uint32_t* tap_s = reinterpret_cast<const uint32_t*>(smem + G::SMEM_TAP);
    uint32_t issued = 0;
    auto issue_next = [&]() {
        if (i_done) return;
        const int buf = (int)(issued % STAGES);
        if (issued >= (uint32_t)STAGES)   // the MMA of this buffer's previous item must be done
            mbar_wait(bar_mma + 8 * buf, ((issued / STAGES) - 1) & 1u);
        const uint32_t a_dst = s_base + SMEM_A + buf * A_STAGE + tid * 16;
#pragma unroll
        for (int pl = 0; pl < NPL; ++pl) {
            const int64_t k0 = (int64_t)i_st * KS + 16 * pl;
            const uint32_t dst = a_dst + pl * (BM * 16);
            if (P.c4) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t tv = tap_s[(int)(k0 >> 2) + j];
                    const int rdh = (int)(tv & 0xffu), sdw = (int)((tv >> 8) & 0xffu);
                    const int64_t toff = ((int64_t)rdh * p.Wd + sdw) * p.C + (int)(tv >> 16);
                    const bool ok = irow.valid && tv != ~0u && (unsigned)(irow.hb + rdh) < (unsigned)p.H &&
                                    (unsigned)(irow.wb + sdw) < (unsigned)p.Wd;
                    cp_async4(dst + 4 * j, ok ? p.A + roff + toff : p.A, ok ? 4u : 0u);
                }
            } else if (P.is_conv) {
                const int rdh = t_r * p.dh, sdw = t_s * p.dw;
                const int64_t toff = ((int64_t)rdh * p.Wd + sdw) * p.C + t_c;
                const bool ok = irow.valid && k0 < p.K && (unsigned)(irow.hb + rdh) < (unsigned)p.H &&
                                (unsigned)(irow.wb + sdw) < (unsigned)p.Wd;
                cp_async16(dst, ok ? p.A + roff + toff : p.A, ok ? 16u : 0u);
                t_c += 16;
                if (t_c >= p.C) {
                    t_c = 0;
                    if (++t_s == p.S) { t_s = 0; ++t_r; }
                }
            } else {
                const int64_t rem = p.K - k0;
                const uint32_t nb = rem >= 16 ? 16u : (rem > 0 ? (uint32_t)rem : 0u);
                const bool ok = irow.valid && nb > 0;
                cp_async16(dst, ok ? p.A + roff + k0 : p.A, ok ? nb : 0u);
            }
        }
        cp_async_commit();
        if (tid == 0) {
            const uint32_t bar = bar_full + 8 * buf;
            const uint32_t* tbl_g = P.tables + ((size_t)i_nb * P.Kp + (size_t)i_st * KS) * 4 * G::TROWS;
            const int8_t* w_g = P.wpk + ((size_t)i_nb * (P.Kp / 16) + (size_t)i_st * NPL) * p4::W_STAGE;
            mbar_expect_tx(bar, TBL_STAGE + NPL * p4::W_STAGE);
            bulk_g2s(s_base + SMEM_TBL + buf * TBL_STAGE, tbl_g, TBL_STAGE, bar);
            bulk_g2s(s_base + SMEM_W + buf * W_STAGE, w_g, NPL * p4::W_STAGE, bar);
        }
        ++issued;
        if (++i_st >= i_se) set_issue_tile();
    };
    set_issue_tile();
#pragma unroll
    for (int i = 0; i < STAGES; ++i) issue_next();

    uint32_t consumed = 0, tiles_done = 0;
    int* fin_flag = reinterpret_cast<int*>(smem + G::SMEM_BAR + 8 * (2 * STAGES + 1) + 4);
    Gen cg;
    int64_t tile;
    int s_b, s_e;
    gen_init(cg);
    while (gen_next(cg, tile, s_b, s_e)) {
        int64_t nb, m0;
        tile_mn(tile, nb, m0);
        const int64_t n0 = nb * TN;
        const bool wlive = m0 + warp * 32 < p.M;   // rows past M: no lookups (ragged last tile)
        if (p.C_out == nullptr && p.ep.residual && n0 + TN <= p.N && m0 + tid < p.M)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p.ep.residual + (m0 + tid) * p.ep.ldr + n0),
                         "r"(TN * 4)
                         : "memory");

        uint32_t pacc[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q) pacc[q][0] = pacc[q][1] = 0u;
        bool e_first = true;

        // packed 16-bit lane sums -> TMEM E accumulators (first flush of the tile overwrites)
        auto flush = [&]() {
            uint32_t ev[16];
            if (!e_first) {
                tmem_ld16(t_e, ev);
                tmem_wait_ld();
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) ev[j] = 0u;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                ev[4 * q + 0] += pacc[q][0] & 0xffffu;
                ev[4 * q + 2] += pacc[q][0] >> 16;
                ev[4 * q + 1] += pacc[q][1] & 0xffffu;
                ev[4 * q + 3] += pacc[q][1] >> 16;
                pacc[q][0] = pacc[q][1] = 0u;
            }
            tmem_st16(t_e, ev);
            tmem_wait_st();
            e_first = false;
        };

        for (int st = s_b; st < s_e; ++st) {
            const int buf = (int)(consumed % STAGES);
            const uint32_t later = issued - consumed - 1;
            if (later >= 3) cp_async_wait<3>(); else if (later == 2) cp_async_wait<2>();
            else if (later == 1) cp_async_wait<1>(); else cp_async_wait<0>();
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // cp.async data -> MMA
            mbar_wait(bar_full + 8 * buf, (consumed / STAGES) & 1u);
            ++consumed;
            tc_fence_before();
            __syncthreads();                 // item visible to all; previous buffer consumed
            tc_fence_after();
            if (tid == 0) {
                // exact part: 8 MMAs (128-row slices) into TMEM columns [16 j, 16 j + 16)
                const uint32_t a0 = s_base + SMEM_A + buf * A_STAGE;
                const uint64_t bdesc = umma_desc_kmajor(s_base + SMEM_W + buf * W_STAGE, 256u, 128u);
#pragma unroll
                for (int j = 0; j < BM / 128; ++j)
                    umma_i8(tmem + (uint32_t)j * TN,
                            umma_desc_kmajor(a0 + j * 128 * 16, KS == 32 ? (uint32_t)(BM * 16) : 0u, 128u), bdesc, IDESC,
                            st == s_b ? 0u : 1u);
                umma_commit(bar_mma + 8 * buf);
                if (st + 1 == s_e) umma_commit(bar_tile);
            }
            if (consumed >= 2) issue_next();   // refill the buffer the previous item used
            const uint8_t* tb = smem + SMEM_TBL + buf * TBL_STAGE;
            const uint8_t* at = smem + SMEM_A + buf * A_STAGE;

            // ---- E lookups: 4 per 32-bit shared load, packed 16-bit accumulation; the loads
            //      of two consecutive k are summed by one 3-input add per accumulator ----
#pragma unroll
            for (int pl = 0; pl < NPL; ++pl) {
                if (!wlive) break;
                const uint4 av = *reinterpret_cast<const uint4*>(at + pl * (BM * 16) + tid * 16);
                const uint32_t aw[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
                for (int kk = 0; kk < 16; kk += 2) {
                    const uint32_t ua0 = __byte_perm(aw[kk >> 2], 0u, 0x4440u + (kk & 3));
                    const uint32_t ua1 = __byte_perm(aw[kk >> 2], 0u, 0x4440u + ((kk + 1) & 3));
                    const uint8_t* r0 = tb + (pl * 16 + kk) * 4 * TQ + ua0 * 4u;
                    const uint8_t* r1 = tb + (pl * 16 + kk + 1) * 4 * TQ + ua1 * 4u;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t v0 = *reinterpret_cast<const uint32_t*>(r0 + q * TQ);
                        const uint32_t v1 = *reinterpret_cast<const uint32_t*>(r1 + q * TQ);
                        pacc[q][0] += __byte_perm(v0, 0u, 0x4240u) + __byte_perm(v1, 0u, 0x4240u);
                        pacc[q][1] += __byte_perm(v0, 0u, 0x4341u) + __byte_perm(v1, 0u, 0x4341u);
                    }
                }
            }
            if ((st - s_b + 1) % G::FLUSH_STAGES == 0 || st + 1 == s_e) flush();
        }
        int corr = p4::E_BIAS * KS * (s_e - s_b);
        if (s_e == nst_all) corr += (int)(((P.Kp - p.K) + p.pad_lookups) * (int64_t)p.t00);

        // the tile's MMAs are complete once bar_tile flips
        mbar_wait(bar_tile, tiles_done & 1u);
        ++tiles_done;
        tc_fence_after();
        uint32_t ex[16], es[16];
        tmem_ld16(t_exact, ex);
        tmem_ld16(t_e, es);
        tmem_wait_ld();
        int eacc[16];
#pragma unroll
        for (int n = 0; n < 16; ++n) eacc[n] = (int)(ex[n] + es[n]) - corr;
        const int64_t m = m0 + tid;
        if (sk && !(s_b == 0 && s_e == nst_all)) {
            // a stream-K piece: add it to the workspace; the contributor that completes the
            // tile's stage count reads the exact total back (and re-zeroes the workspace)
            int* wrow = P.ws + m * p.N + n0;
            if (m < p.M) {
#pragma unroll
                for (int n = 0; n < TN; ++n)
                    if (n0 + n < p.N) atomicAdd(wrow + n, eacc[n]);
            }
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                const int64_t x = (tile - t_dp) * nst_all;   // the tile's first tail iteration
                int64_t c = (x * G_) / it_sk;
                while (c + 1 < G_ && sk_begin(c + 1) - t_dp * nst_all <= x) ++c;
                const int old = atomicAdd(P.cnt + c, s_e - s_b);
                const int fin = (old + (s_e - s_b) == nst_all) ? 1 : 0;
                if (fin) P.cnt[c] = 0;
                *fin_flag = fin;
            }
            __syncthreads();
            if (*fin_flag) {
                __threadfence();
                if (m < p.M) {
#pragma unroll
                    for (int n = 0; n < TN; ++n) {
                        eacc[n] = (n0 + n < p.N) ? __ldcg(wrow + n) : 0;
                        if (n0 + n < p.N) wrow[n] = 0;
                    }
                    p4t_store_row(P, m, n0, eacc, 1);
                }
            }
        } else if (m < p.M) {
            p4t_store_row(P, m, n0, eacc, splits);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS)
                     : "memory");
    }
}

}  // namespace axq

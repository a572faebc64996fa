// lut_p4.cuh -- "P4" LUT-GEMM / implicit-im2col LUT-conv for delta8 tables (sm_100a).
//
// Same result as lut_mm.cuh (acc[m][n] = sum_k LUT[a[m][k]][w[n][k]], int32, exact), built so
// that one shared-memory load serves FOUR lookups instead of one:
//
//  * The table is split exactly as LUT = a*w + E (E fits int8, the delta8 representation).
//  * Weight-specialised tables (prepared once per layer, axq_wpack_create): for every k and
//    every quad of 4 output columns q, T[k][q][ua] = (E[ua][w(4q,k)], E[ua][w(4q+1,k)],
//    E[ua][w(4q+2,k)], E[ua][w(4q+3,k)]) as 4 int8 in one 32-bit word (1 KiB per (k, q)).
//    A lane that owns output row m fetches T[k][q][a[m][k]] with ONE 32-bit LDS and gets the
//    E terms of 4 outputs.  Bank = ua mod 32: lanes only conflict when two of them hold
//    different activation codes congruent mod 32 (measured ~1.8-way for ReLU'd data).
//  * The exact part sum_k a*w is a dense int8 contraction: it runs on the tensor cores
//    (mma.sync m16n8k16 s8, fragments by ldmatrix from the staged operand tiles).
//  * Per 16-k stage the CTA stages, double-buffered: the E tables of its 16 columns (64 KiB,
//    one cp.async.bulk, mbarrier complete_tx), the packed weight tile (256 B, bulk) and the
//    activation tile (1024 rows x 16 B, cp.async with zero-fill = implicit im2col, semantic
//    padding taps read as a = 0 and are looked up, A11).
//  * CTA tile 1024 rows x 16 columns, 16 warps.  A lane owns 2 rows x 16 columns of E sums,
//    kept as biased (E + 128) bytes added in pairs of 16-bit lanes: per shared load 2 PRMT
//    split the even / odd bytes and 2 IMAD (FMA pipe, multiplier 1 passed as a parameter) add
//    them, so the ALU and FMA pipes share the work.  Every 256 k the packed sums are flushed
//    through a per-warp shared scratch into the mma accumulators (exact part); the bias
//    128*Kp is removed at the end and the fused epilogue of lut_mm.cuh runs on the result.
//  * Persistent grid (one CTA per SM), tiles walked m-major within an n-column block.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lut_mm.cuh"
#include "lut_p4_args.h"

namespace axq {

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}

// whole 16 bytes or zeros (ignore-src predicate): keeps the fixed-size LDGSTS form -- a
// variable src-size operand can compile to the ZFILL form, measured at ~16x the shared-memory
// wavefronts per copy
__device__ __forceinline__ void cp_async16_p(uint32_t dst, const void* src, bool ok) {
    asm volatile("{\n.reg .pred p;\nsetp.eq.u32 p, %2, 0;\ncp.async.cg.shared.global [%0], [%1], 16, p;\n}\n" ::"r"(dst),
                 "l"(src), "r"((uint32_t)ok)
                 : "memory");
}

__device__ __forceinline__ void cp_async4_p(uint32_t dst, const void* src, bool ok) {
    asm volatile("{\n.reg .pred p;\nsetp.eq.u32 p, %2, 0;\ncp.async.ca.shared.global [%0], [%1], 4, p;\n}\n" ::"r"(dst),
                 "l"(src), "r"((uint32_t)ok)
                 : "memory");
}

__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                            uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

__device__ __forceinline__ void ldmatrix_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n"
                 : "=r"(r0), "=r"(r1)
                 : "r"(addr));
}

// Sign-extend byte j of v with PTX prmt's sign-replicate selectors (the CUDA __byte_perm
// intrinsic only honours the low 3 bits of each selector nibble).
template <uint32_t SEL>
__device__ __forceinline__ int prmt_sext(uint32_t v) {
    int r;
    asm("prmt.b32 %0, %1, 0, %2;\n" : "=r"(r) : "r"(v), "n"(SEL));
    return r;
}

__device__ __forceinline__ void mma_s8_16816(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(b0));
}

// Per-tile output of one warp (rows mw .. mw + 32*RPL - 1, columns n0 .. n0+TN-1): the int32
// totals wait in the warp's shared scratch.  Not inlined, so the register allocation of the
// lookup loop does not depend on which epilogue features exist.
template <int RPL>
__device__ __noinline__ void p4_epilogue(const P4Args& P, const int* scr, int64_t mw, int64_t n0, int corr,
                                         int splits, int lane) {
    using namespace p4;
    const MMArgs& p = P.mm;
    auto sidx = [](int row, int col) { return row * TN + (col ^ (row & 15)); };
    const EpiArgs& e = p.ep;
    const bool raw = p.C_out != nullptr;
    const bool vec = !raw && (n0 + TN <= p.N) && !e.y_nchw &&
                     (!e.y || (((e.ldy & 3) == 0) && ((reinterpret_cast<uintptr_t>(e.y) & 15) == 0))) &&
                     (!e.residual || (((e.ldr & 3) == 0) && ((reinterpret_cast<uintptr_t>(e.residual) & 15) == 0))) &&
                     (!e.bias || ((reinterpret_cast<uintptr_t>(e.bias) & 15) == 0)) &&
                     (!e.q || (((e.ldq & 3) == 0) && ((reinterpret_cast<uintptr_t>(e.q) & 3) == 0)));
    const bool q16 = vec && e.q && ((e.ldq & 15) == 0) && ((reinterpret_cast<uintptr_t>(e.q) & 15) == 0);

    // ---- output: atomic int32 (split K), raw int32, or the fused epilogue ----
    const float sc = raw ? 0.f : __fmul_rn(*e.sa, *e.sw);
    const float s_out = (!raw && e.q) ? *e.s_out : 1.f;
    const float qm = (float)((1 << ((!raw && e.q ? e.bits_out : 8) - 1)) - 1);
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
        const int64_t m = mw + r * 32 + lane;
        if (m >= p.M) continue;
        int eacc[TN];
#pragma unroll
        for (int n = 0; n < TN; ++n) eacc[n] = scr[sidx(r * 32 + lane, n)] - corr;
        if (raw) {
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
            continue;
        }
        if (vec) {
            // all of the row's residual loads first: one latency per row, not per 4 columns
            float4 res[TN / 4];
            if (e.residual) {
                const float4* rp = reinterpret_cast<const float4*>(e.residual + m * e.ldr + n0);
#pragma unroll
                for (int j = 0; j < TN / 4; ++j) res[j] = __ldg(rp + j);
            }
            uint32_t qw[TN / 4];
#pragma unroll
            for (int n = 0; n < TN; n += 4) {
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
                    const float4 rr = res[n / 4];
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
                    qw[n / 4] = w;
                    if (!q16) *reinterpret_cast<uint32_t*>(e.q + m * e.ldq + nn) = w;
                }
            }
            if (q16) *reinterpret_cast<uint4*>(e.q + m * e.ldq + n0) = make_uint4(qw[0], qw[1], qw[2], qw[3]);
        } else if (e.y_nchw) {
            // NCHW fp32 output: lanes are consecutive pixels, so each column's stores are
            // coalesced; the (image, pixel) split is computed once per row
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
    __syncwarp();
}

template <int RPL, bool HALF>
__global__ void __launch_bounds__(p4::NT, 1) lut_p4_kernel(const __grid_constant__ P4Args P) {
    using namespace p4;
    using G = Geo<HALF>;
    constexpr int STAGES = G::STAGES, TBL_STAGE = G::TBL_STAGE, TQ = G::TQ;
    constexpr int SMEM_TBL = G::SMEM_TBL, SMEM_A = G::SMEM_A, SMEM_W = G::SMEM_W;
    constexpr int SMEM_BAR = G::SMEM_BAR, SMEM_SCR = G::SMEM_SCR;
    constexpr int BMR = WARPS * 32 * RPL;    // rows per CTA tile (1024 or 512)
    constexpr int MT = 2 * RPL;              // m16 tiles per warp
    constexpr int WROWS = 32 * RPL;          // rows per warp
    extern __shared__ __align__(1024) uint8_t p4_smem[];
    uint8_t* smem = p4_smem;
    const MMArgs& p = P.mm;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t s_base = smem_u32(smem);
    const uint32_t bar0 = s_base + SMEM_BAR;

    if (P.c4) {
        // tap table of the 4-byte loader: entry g covers k = 4g .. 4g+3 (one tap, C % 4 == 0)
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
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    const int64_t m_tiles = (p.M + BMR - 1) / BMR, n_blocks = (p.N + TN - 1) / TN;
    const int splits = P.splits > 0 ? P.splits : 1;
    const int64_t n_work = m_tiles * n_blocks * splits;
    const int nst_all = (int)(P.Kp / KS);
    const int sps = P.stages_per_split > 0 ? P.stages_per_split : nst_all;

    // ---- work decomposition: tile -> (n block, m tile, k split) -> stage range ----
    auto decode = [&](int64_t tile, int64_t& nb, int64_t& m0, int& s_b, int& s_e) {
        const int ks = (int)(tile % splits);
        const int64_t rest = tile / splits;
        int64_t mt;
        if (P.nb_fast) {
            nb = rest % n_blocks;
            mt = rest / n_blocks;
        } else {
            mt = rest % m_tiles;
            nb = rest / m_tiles;
        }
        m0 = mt * BMR;
        s_b = ks * sps;
        s_e = min(nst_all, s_b + sps);
    };

    // ---- producer state: a flat per-CTA stream of (tile, stage) items, STAGES buffers ----
    // Per row: the offset of its receptive-field origin (conv) or row start (GEMM), computed
    // once per tile.  Per item: the filter tap (r, s) and channel c0 of k0, advanced
    // incrementally (no divisions on the per-stage path).
    int64_t i_tile = blockIdx.x, i_nb = 0, i_m0 = 0;
    int i_st = 0, i_se = 0;
    int t_r = 0, t_s = 0, t_c = 0;
    RowInfo irow[RPL];
    int64_t roff[RPL];
    auto set_issue_tile = [&]() {
        if (i_tile >= n_work) return;
        decode(i_tile, i_nb, i_m0, i_st, i_se);
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
            irow[i] = P.is_conv ? make_row<LOAD_CONV>(p, i_m0 + tid + i * NT)
                                : make_row<LOAD_GEMM>(p, i_m0 + tid + i * NT);
            roff[i] = irow[i].base + (P.is_conv ? ((int64_t)irow[i].hb * p.Wd + irow[i].wb) * p.C : 0);
        }
        if (P.is_conv && !P.c4) {
            const int k0 = i_st * KS, rs = k0 / p.C;
            t_c = k0 - rs * p.C;
            t_r = rs / p.S;
            t_s = rs - t_r * p.S;
        }
    };
    const uint32_t* tap_s = reinterpret_cast<const uint32_t*>(smem + G::SMEM_TAP);
    uint32_t issued = 0;   // items issued by this CTA (buffer = index % STAGES)
    auto issue_next = [&]() {
        if (i_tile >= n_work) return;
        const int buf = (int)(issued % STAGES);
        const int64_t k0 = (int64_t)i_st * KS;
        const uint32_t a_dst = s_base + SMEM_A + buf * A_STAGE + tid * KS;
        if (P.c4) {
            // C % 4 == 0 (small C, e.g. the padded network input): 4 taps of 4 bytes per 16 k,
            // tap geometry from the shared tap table (r*dh | s*dw << 8 | c << 16; ~0u past K)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t tv = tap_s[i_st * 4 + j];
                const int rdh = (int)(tv & 0xffu), sdw = (int)((tv >> 8) & 0xffu);
                const int64_t toff = ((int64_t)rdh * p.Wd + sdw) * p.C + (int)(tv >> 16);
#pragma unroll
                for (int i = 0; i < RPL; ++i) {
                    const RowInfo& ri = irow[i];
                    const bool ok = ri.valid && tv != ~0u && (unsigned)(ri.hb + rdh) < (unsigned)p.H &&
                                    (unsigned)(ri.wb + sdw) < (unsigned)p.Wd;
                    cp_async4(a_dst + i * NT * KS + 4 * j, ok ? p.A + roff[i] + toff : p.A, ok ? 4u : 0u);
                }
            }
        } else if (P.is_conv) {
            // C % 16 == 0: the 16 k of the item lie inside one filter tap
            const int rdh = t_r * p.dh, sdw = t_s * p.dw;
            const int64_t toff = ((int64_t)rdh * p.Wd + sdw) * p.C + t_c;
#pragma unroll
            for (int i = 0; i < RPL; ++i) {
                const RowInfo& ri = irow[i];
                const bool ok = ri.valid && k0 < p.K && (unsigned)(ri.hb + rdh) < (unsigned)p.H &&
                                (unsigned)(ri.wb + sdw) < (unsigned)p.Wd;
                cp_async16(a_dst + i * NT * KS, ok ? p.A + roff[i] + toff : p.A, ok ? 16u : 0u);
            }
            t_c += KS;
            if (t_c >= p.C) {
                t_c = 0;
                if (++t_s == p.S) { t_s = 0; ++t_r; }
            }
        } else {
            const int64_t rem = p.K - k0;
            const uint32_t nb = rem >= 16 ? 16u : (rem > 0 ? (uint32_t)rem : 0u);
#pragma unroll
            for (int i = 0; i < RPL; ++i) {
                const bool ok = irow[i].valid && nb > 0;
                cp_async16(a_dst + i * NT * KS, ok ? p.A + roff[i] + k0 : p.A, ok ? nb : 0u);
            }
        }
        cp_async_commit();
        if (tid == 0) {
            const uint32_t bar = bar0 + 8 * buf;
            const uint32_t* tbl_g = P.tables + ((size_t)i_nb * P.Kp + (size_t)i_st * KS) * 4 * G::TROWS;
            const int8_t* w_g = P.wpk + ((size_t)i_nb * (P.Kp / KS) + i_st) * W_STAGE;
            mbar_expect_tx(bar, TBL_STAGE + W_STAGE);
            bulk_g2s(s_base + SMEM_TBL + buf * TBL_STAGE, tbl_g, TBL_STAGE, bar);
            bulk_g2s(s_base + SMEM_W + buf * W_STAGE, w_g, W_STAGE, bar);
        }
        ++issued;
        if (++i_st >= i_se) {
            i_tile += gridDim.x;
            set_issue_tile();
        }
    };
    set_issue_tile();
#pragma unroll
    for (int i = 0; i < STAGES; ++i) issue_next();

    int* scr = reinterpret_cast<int*>(smem + SMEM_SCR + warp * SCR_WARP);
    const int g = lane >> 2, t4 = lane & 3;
    // element (row, col) of the warp scratch, XOR-swizzled so that a lane reading its row
    // and a thread writing its mma fragment are (nearly) conflict free
    auto sidx = [](int row, int col) { return row * TN + (col ^ (row & 15)); };
    const uint32_t one = P.one;
    uint32_t consumed = 0;   // items consumed (buffer = index % STAGES, phase = index / STAGES)

    for (int64_t tile = blockIdx.x; tile < n_work; tile += gridDim.x) {
        int64_t nb, m0;
        int s_b, s_e;
        decode(tile, nb, m0, s_b, s_e);
        const int64_t n0 = nb * TN;
        if (p.C_out == nullptr && p.ep.residual && n0 + TN <= p.N) {
            // the epilogue's residual rows (TN fp32 each): pull them into L2 while the
            // lookups run, so the epilogue does not stall on HBM latency
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
                const int64_t m = m0 + warp * WROWS + r * 32 + lane;
                if (m < p.M)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p.ep.residual + m * p.ep.ldr + n0),
                                 "r"(TN * 4) : "memory");
            }
        }

        uint32_t pacc[RPL][4][2];   // packed 16-bit E sums: [row][quad][even (c0,c2) / odd (c1,c3)]
#pragma unroll
        for (int r = 0; r < RPL; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) pacc[r][q][0] = pacc[r][q][1] = 0u;
        int cacc[MT][2][4];         // exact part: m16 tiles x 2 n8 tiles x mma C fragment
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int c = 0; c < 4; ++c) cacc[i][j][c] = 0;

        // packed lane sums -> scratch (lane layout) -> added into the mma fragments
        auto flush = [&]() {
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
                const int row = r * 32 + lane;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    scr[sidx(row, 4 * q + 0)] = (int)(pacc[r][q][0] & 0xffffu);
                    scr[sidx(row, 4 * q + 2)] = (int)(pacc[r][q][0] >> 16);
                    scr[sidx(row, 4 * q + 1)] = (int)(pacc[r][q][1] & 0xffffu);
                    scr[sidx(row, 4 * q + 3)] = (int)(pacc[r][q][1] >> 16);
                    pacc[r][q][0] = pacc[r][q][1] = 0u;
                }
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int row = i * 16 + g, col = j * 8 + 2 * t4;
                    cacc[i][j][0] += scr[sidx(row, col)];
                    cacc[i][j][1] += scr[sidx(row, col + 1)];
                    cacc[i][j][2] += scr[sidx(row + 8, col)];
                    cacc[i][j][3] += scr[sidx(row + 8, col + 1)];
                }
            __syncwarp();
        };

        for (int st = s_b; st < s_e; ++st) {
            const int buf = (int)(consumed % STAGES);
            // this item's cp.async group is complete once at most (later items in flight)
            // groups remain outstanding
            const uint32_t later = issued - consumed - 1;
            if (later >= 2) cp_async_wait<2>(); else if (later == 1) cp_async_wait<1>(); else cp_async_wait<0>();
            mbar_wait(bar0 + 8 * buf, (consumed / STAGES) & 1u);
            ++consumed;
            __syncthreads();                 // item visible to all; the previous buffer is free
            if (consumed >= 2) issue_next(); // refill the buffer the previous item used
            const uint8_t* tb = smem + SMEM_TBL + buf * TBL_STAGE;
            const uint8_t* at = smem + SMEM_A + buf * A_STAGE;

            // ---- exact part on the tensor cores: MT m16 x 2 n8 tiles, k = 16 ----
            {
                uint32_t b0, b1;
                ldmatrix_x2(s_base + SMEM_W + buf * W_STAGE + (lane & 15) * KS, b0, b1);
#pragma unroll
                for (int h = 0; h < RPL; ++h) {
                    uint32_t a0, a1, a2, a3;
                    ldmatrix_x4(s_base + SMEM_A + buf * A_STAGE + (warp * WROWS + h * 32 + lane) * KS, a0, a1, a2, a3);
                    mma_s8_16816(cacc[2 * h][0], a0, a1, b0);
                    mma_s8_16816(cacc[2 * h][1], a0, a1, b1);
                    mma_s8_16816(cacc[2 * h + 1][0], a2, a3, b0);
                    mma_s8_16816(cacc[2 * h + 1][1], a2, a3, b1);
                }
            }
            // ---- E lookups: 4 per 32-bit shared load, packed 16-bit accumulation ----
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
                const uint4 av = *reinterpret_cast<const uint4*>(at + (warp * WROWS + r * 32 + lane) * KS);
                const uint32_t aw[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
                for (int kk = 0; kk < KS; ++kk) {
                    const uint32_t ua = __byte_perm(aw[kk >> 2], 0u, 0x4440u + (kk & 3));
                    const uint8_t* row_t = tb + kk * 4 * TQ + ua * 4u;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t v = *reinterpret_cast<const uint32_t*>(row_t + q * TQ);
                        const uint32_t ev = __byte_perm(v, 0u, 0x4240u);   // [b0, 0, b2, 0]
                        const uint32_t od = __byte_perm(v, 0u, 0x4341u);   // [b1, 0, b3, 0]
                        asm("mad.lo.u32 %0, %1, %2, %0;\n" : "+r"(pacc[r][q][0]) : "r"(ev), "r"(one));
                        asm("mad.lo.u32 %0, %1, %2, %0;\n" : "+r"(pacc[r][q][1]) : "r"(od), "r"(one));
                    }
                }
            }
            if ((st - s_b + 1) % FLUSH_STAGES == 0 || st + 1 == s_e) flush();
        }
        // bias of the packed sums and the storage-padding lookups (counted by the split that
        // holds the end of K)
        int corr = E_BIAS * KS * (s_e - s_b);
        if (s_e == nst_all) corr += (int)(((P.Kp - p.K) + p.pad_lookups) * (int64_t)p.t00);
        // the int32 total of every output: write the mma fragments to the scratch, read rows
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int row = i * 16 + g, col = j * 8 + 2 * t4;
                scr[sidx(row, col)] = cacc[i][j][0];
                scr[sidx(row, col + 1)] = cacc[i][j][1];
                scr[sidx(row + 8, col)] = cacc[i][j][2];
                scr[sidx(row + 8, col + 1)] = cacc[i][j][3];
            }
        __syncwarp();
        p4_epilogue<RPL>(P, scr, m0 + warp * WROWS, n0, corr, splits, lane);
    }
}

// ---- weight preparation: E tables and the packed weight tile (once per layer) ----
// tables[((nb*Kp + k)*4 + q)*rows + u] = bytes j=0..3: E[u][w(16nb+4q+j, k)] + 128 (E = delta8
// table); rows = 256, or 128 when only non-negative codes u will be looked up.
// swap = 1 specialises the tables on the FIRST (activation) operand instead: the packed codes
// are activations x and the looked-up row code u is a weight, so the byte is E[x][u] + 128
// (used to build tables from a small activation matrix per call, axq_lut_gemm_xs); the
// caller then passes the transposed table ([ua][uw]) so the reads stay row-contiguous.
// Persistent blocks with the 64 KiB packing table staged in shared memory.  Work items are
// (nb, 64-k chunk): the chunk's 16 x 64 packed codes are read once (coalesced), then per k each
// thread writes 4 consecutive words of one quad: the 4 codes' table rows are read 4 bytes at a
// time (u .. u+3), biased (E + 128 == E ^ 0x80 for an int8 E) and byte-transposed with 8
// PRMTs, one 16-byte store.  (A [k][u][quad] layout -- one 16-byte lookup load per k in the
// GEMM kernels -- measured slower there: more bank-conflict wavefronts per lookup.)
constexpr int PACK_THREADS = 256;
constexpr int PACK_KC = 64;
__global__ void __launch_bounds__(PACK_THREADS) p4_pack_tables_kernel(
        const int8_t* __restrict__ W, int64_t N, int64_t K, int64_t ldw, int64_t Kp,
        const int8_t* __restrict__ dtab, uint32_t* __restrict__ tables, int rows, int swap) {
    extern __shared__ __align__(16) uint8_t pk_tab[];   // [256 codes][256 u]
    __shared__ uint8_t codes[p4::TN][PACK_KC];
    {   // all 16 loads of a thread in flight at once (not 16 dependent L2 round trips)
        uint4 v[65536 / 16 / PACK_THREADS];
#pragma unroll
        for (int i = 0; i < 65536 / 16 / PACK_THREADS; ++i)
            v[i] = __ldg(reinterpret_cast<const uint4*>(dtab) + threadIdx.x + i * PACK_THREADS);
#pragma unroll
        for (int i = 0; i < 65536 / 16 / PACK_THREADS; ++i)
            reinterpret_cast<uint4*>(pk_tab)[threadIdx.x + i * PACK_THREADS] = v[i];
    }
    const int64_t n_blocks = (N + p4::TN - 1) / p4::TN;
    const int64_t k_chunks = (Kp + PACK_KC - 1) / PACK_KC;
    const int per_q = rows / 4;                          // uint4 groups per quad
    const int q = threadIdx.x / per_q, u4 = (threadIdx.x - q * per_q) * 4;
    const bool active = threadIdx.x < 4 * per_q;
    for (int64_t item = blockIdx.x; item < n_blocks * k_chunks; item += gridDim.x) {
        const int64_t nb = item / k_chunks, k0 = (item - nb * k_chunks) * PACK_KC;
        const int kn = (int)min((int64_t)PACK_KC, Kp - k0);
        __syncthreads();
        for (int i = threadIdx.x; i < p4::TN * PACK_KC; i += PACK_THREADS) {
            const int j = i / PACK_KC, kk = i - j * PACK_KC;
            const int64_t n = nb * p4::TN + j, k = k0 + kk;
            codes[j][kk] = (n < N && k < K) ? (uint8_t)W[n * ldw + k] : 0;
        }
        __syncthreads();
        if (!active) continue;
        uint32_t* dst = tables + (nb * Kp + k0) * 4 * rows + q * rows + u4;
#pragma unroll 2
        for (int kk = 0; kk < kn; ++kk) {
            uint32_t w[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                w[j] = *reinterpret_cast<const uint32_t*>(pk_tab + ((int)codes[4 * q + j][kk] << 8) + u4) ^ 0x80808080u;
            const uint32_t lo01 = __byte_perm(w[0], w[1], 0x5140), hi01 = __byte_perm(w[0], w[1], 0x7362);
            const uint32_t lo23 = __byte_perm(w[2], w[3], 0x5140), hi23 = __byte_perm(w[2], w[3], 0x7362);
            uint4 o;
            o.x = __byte_perm(lo01, lo23, 0x5410);
            o.y = __byte_perm(lo01, lo23, 0x7632);
            o.z = __byte_perm(hi01, hi23, 0x5410);
            o.w = __byte_perm(hi01, hi23, 0x7632);
            *reinterpret_cast<uint4*>(dst + (int64_t)kk * 4 * rows) = o;
        }
    }
}

// P4W16 tables (E = LUT - a*w beyond int8 but within int16; half range, codes 0..127):
//   tables[nb][k][p][u] = (E[u][w(16nb+2p, k)] + 32768) | (E[u][w(16nb+2p+1, k)] + 32768) << 16
// from the int16 E table e16 [uw][ua] (128 KiB, staged in shared memory).
__global__ void __launch_bounds__(PACK_THREADS) p4_pack16_tables_kernel(
        const int8_t* __restrict__ W, int64_t N, int64_t K, int64_t ldw, int64_t Kp,
        const int16_t* __restrict__ e16, uint32_t* __restrict__ tables) {
    extern __shared__ __align__(16) uint8_t pk16_tab[];   // [256 uw][256 ua] int16
    __shared__ uint8_t codes[p4::TN][PACK_KC];
    for (int i = threadIdx.x; i < 131072 / 16; i += PACK_THREADS)
        reinterpret_cast<uint4*>(pk16_tab)[i] = __ldg(reinterpret_cast<const uint4*>(e16) + i);
    const int16_t* et = reinterpret_cast<const int16_t*>(pk16_tab);
    const int64_t n_blocks = (N + p4::TN - 1) / p4::TN;
    const int64_t k_chunks = (Kp + PACK_KC - 1) / PACK_KC;
    const int pr = threadIdx.x >> 5, u4 = (threadIdx.x & 31) * 4;   // pair 0..7, codes u4..u4+3
    for (int64_t item = blockIdx.x; item < n_blocks * k_chunks; item += gridDim.x) {
        const int64_t nb = item / k_chunks, k0 = (item - nb * k_chunks) * PACK_KC;
        const int kn = (int)min((int64_t)PACK_KC, Kp - k0);
        __syncthreads();
        for (int i = threadIdx.x; i < p4::TN * PACK_KC; i += PACK_THREADS) {
            const int j = i / PACK_KC, kk = i - j * PACK_KC;
            const int64_t n = nb * p4::TN + j, k = k0 + kk;
            codes[j][kk] = (n < N && k < K) ? (uint8_t)W[n * ldw + k] : 0;
        }
        __syncthreads();
        uint32_t* dst = tables + ((nb * Kp + k0) * 8 + pr) * 128 + u4;
        for (int kk = 0; kk < kn; ++kk) {
            const int16_t* r0 = et + ((int)codes[2 * pr][kk] << 8) + u4;
            const int16_t* r1 = et + ((int)codes[2 * pr + 1][kk] << 8) + u4;
            uint32_t o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                o[j] = (uint32_t)(uint16_t)(r0[j] + 32768) | ((uint32_t)(uint16_t)(r1[j] + 32768) << 16);
            *reinterpret_cast<uint4*>(dst + (int64_t)kk * 8 * 128) = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
}

// wpk[((nb*(Kp/16) + kc)*16 + nl)*16 + kk] = W[16nb+nl][16kc+kk] (0 outside)
__global__ void p4_pack_w_kernel(const int8_t* __restrict__ W, int64_t N, int64_t K, int64_t ldw, int64_t Kp,
                                 int8_t* __restrict__ wpk) {
    const int64_t n_blocks = (N + p4::TN - 1) / p4::TN;
    const int64_t total = n_blocks * Kp * p4::TN;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += gs) {
        const int kk = (int)(i & 15);
        const int nl = (int)((i >> 4) & 15);
        const int64_t t = i >> 8;
        const int64_t kc = t % (Kp / 16), nb = t / (Kp / 16);
        const int64_t n = nb * p4::TN + nl, k = kc * 16 + kk;
        wpk[i] = (n < N && k < K) ? W[n * ldw + k] : (int8_t)0;
    }
}

}  // namespace axq

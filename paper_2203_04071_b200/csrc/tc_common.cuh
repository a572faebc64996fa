// tc_common.cuh -- shared pieces of the packed-table kernels with a tcgen05 exact part (P4W,
// lut_p4w.cuh): the SWIZZLE_NONE K-major UMMA descriptor, tcgen05.mma kind::i8 issue / commit,
// TMEM loads and stores, and the fused per-row epilogue (dequantize, bias, residual, ReLU,
// fp32 / requantized stores; A13/A14/A17).
//
// The packed-table split: LUT[a][w] = a*w + E[a][w] with E int8, so
//   acc[m][n] = sum_k a*w (a dense int8 contraction: tensor cores, TMEM accumulators)
//             + sum_k E[a][w] (the lookups: packed weight-specialised tables in shared memory).
#include <cstdint>
#include <cuda_runtime.h>

#include "lut_p4.cuh"

namespace axq {


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

// A from TMEM (row i = lane i, 4 int8 elements per 32-bit column, K = 32 -> 8 columns), B from
// shared memory
__device__ __forceinline__ void umma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
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
// Specialised epilogue modes (decided once per launch; the ResNet forward's three layer kinds),
// all: row layout, per-tensor scale, no bias, 16-byte aligned rows and code rows.
enum : int {
    EPI_GENERIC = 0,
    EPI_RELU_Q = 1,          // ReLU + requantize (bottleneck c1 / c2)
    EPI_RES_RELU_Y_Q = 2,    // + fp32 residual, ReLU, fp32 y and requantize (block output c3)
    EPI_Y = 3,               // fp32 y only (projection shortcut)
};
struct EpiConst {
    float sc, s_out, qm, r_out;   // r_out = RN(1 / s_out) for epi_quant_r
    int mode, pad0, pad1, pad2;
};
__device__ __forceinline__ EpiConst p4t_epi_const(const P4Args& P) {
    const EpiArgs& e = P.mm.ep;
    EpiConst k{0.f, 1.f, 127.f, 1.f, EPI_GENERIC, 0, 0, 0};
    if (P.mm.C_out == nullptr) {
        k.sc = __fmul_rn(*e.sa, *e.sw);
        k.s_out = e.q ? *e.s_out : 1.f;
        k.qm = (float)((1 << ((e.q ? e.bits_out : 8) - 1)) - 1);
        k.r_out = __frcp_rn(k.s_out);
        const auto a16 = [](const void* ptr, int64_t ld) {
            return ((reinterpret_cast<uintptr_t>(ptr) & 15) == 0) && ((ld & 3) == 0);
        };
        const bool plain = !P.transposed && !e.bias && !e.sw_ch && !e.y_nchw;
        const bool q16 = e.q && ((e.ldq & 15) == 0) && ((reinterpret_cast<uintptr_t>(e.q) & 15) == 0);
        if (plain && e.relu && q16 && !e.residual && !e.y) k.mode = EPI_RELU_Q;
        else if (plain && e.relu && q16 && e.residual && a16(e.residual, e.ldr) && e.y && a16(e.y, e.ldy))
            k.mode = EPI_RES_RELU_Y_Q;
        else if (plain && !e.relu && !e.q && !e.residual && e.y && a16(e.y, e.ldy)) k.mode = EPI_Y;
    }
    return k;
}

// the specialised row epilogue (kc.mode != EPI_GENERIC, whole 16-column tile, no split): the
// generic path's arithmetic without its per-element flag tests; ReLU outputs requantize through
// the sign-free reciprocal test (epi_quant_r_nn, bit-identical to epi_quant)
// ys (residual mode only): the row's fp32 y goes to this shared-memory row instead (16-byte
// chunk j at ys[j ^ swz], the 64-byte swizzle of the TMA store that writes it out)
__device__ __forceinline__ void p4t_store_row_fast(const P4Args& P, int64_t m, int64_t n0, const int (&eacc)[16],
                                                   const EpiConst& kc, const float4* res_pre,
                                                   float4* ys = nullptr, int swz = 0) {
    const EpiArgs& e = P.mm.ep;
    const float sc = kc.sc;
    if (kc.mode == EPI_Y) {
        float4* yp = reinterpret_cast<float4*>(e.y + m * e.ldy + n0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            yp[j] = make_float4(__fmul_rn(__int2float_rn(eacc[4 * j]), sc), __fmul_rn(__int2float_rn(eacc[4 * j + 1]), sc),
                                __fmul_rn(__int2float_rn(eacc[4 * j + 2]), sc), __fmul_rn(__int2float_rn(eacc[4 * j + 3]), sc));
        return;
    }
    const bool res = kc.mode == EPI_RES_RELU_Y_Q;
    const float4* rp = res ? reinterpret_cast<const float4*>(e.residual + m * e.ldr + n0) : nullptr;
    float4* yp = res ? reinterpret_cast<float4*>(e.y + m * e.ldy + n0) : nullptr;
    uint32_t qw[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __fmul_rn(__int2float_rn(eacc[4 * j + u]), sc);
        if (res) {
            const float4 r = res_pre ? res_pre[j] : __ldg(rp + j);
            v[0] = __fadd_rn(v[0], r.x); v[1] = __fadd_rn(v[1], r.y);
            v[2] = __fadd_rn(v[2], r.z); v[3] = __fadd_rn(v[3], r.w);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = v[u] > 0.f ? v[u] : 0.f;
        if (res) {
            if (ys) ys[j ^ swz] = make_float4(v[0], v[1], v[2], v[3]);
            else yp[j] = make_float4(v[0], v[1], v[2], v[3]);
        }
        uint32_t w = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) w |= epi_quant_r_nn(v[u], kc.s_out, kc.r_out, kc.qm) << (8 * u);
        qw[j] = w;
    }
    *reinterpret_cast<uint4*>(e.q + m * e.ldq + n0) = make_uint4(qw[0], qw[1], qw[2], qw[3]);
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
                                              int splits, const EpiConst& kc, const float4* res_pre,
                                              float4* ys = nullptr, int swz = 0);

__device__ __forceinline__ void p4t_store_row(const P4Args& P, int64_t m, int64_t n0, const int (&eacc)[16],
                                              int splits) {
    p4t_store_row<false>(P, m, n0, eacc, splits, p4t_epi_const(P), nullptr);
}

// res_pre: the row's 4 residual float4 groups already loaded (vector path only), or null.
// FASTQ: requantize through the reciprocal (epi_quant_r) -- used by the residual-layer
// instantiation only (elsewhere its registers cost more than the division it saves)
template <bool FASTQ>
__device__ __forceinline__ void p4t_store_row(const P4Args& P, int64_t m, int64_t n0, const int (&eacc)[16],
                                              int splits, const EpiConst& kc, const float4* res_pre,
                                              float4* ys, int swz) {
    using namespace p4;
    const MMArgs& p = P.mm;
    const EpiArgs& e = p.ep;
    if (kc.mode != EPI_GENERIC && splits == 1 && n0 + TN <= p.N) {
        p4t_store_row_fast(P, m, n0, eacc, kc, res_pre, ys, swz);
        return;
    }
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
}  // namespace axq

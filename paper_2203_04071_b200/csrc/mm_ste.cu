// mm_ste.cu -- NEXT-4: the straight-through-estimator (STE) backward of an approximate linear
// layer (§III.A.2 "Retraining": QAT "based on Straight Through Estimator
// (STE) derivative approximation ... fake quantization modules which work with quantized
// floating point values").  Under the STE the quantizer and the ACU are the identity in the
// backward pass, so the layer's gradients are plain dense products of the upstream gradient with
// the fake-quantized operands (fl32(s * q)), masked where the input lies outside the calibrated
// clip range (A36):
//   gx[m][k] = [|x[m][k]| <= clip_a] * sum_n gy[m][n] * fl(s_w * qw[n][k])
//   gw[n][k] = [|w[n][k]| <= clip_w] * sum_m gy[m][n] * fl(s_a * qa[m][k])
//   gb[n]    = sum_m gy[m][n]
// Both products run on the tensor cores (ste_tc_kernel: tcgen05.mma kind::f16, the fp32 operand
// split exactly into three bf16 terms, the int8 codes exact in bf16, fp32 accumulators in TMEM);
// the STE mask is applied in the epilogue.  The result is compared with the fp64 oracle under
// the fp32 dot-product error bound (tests/test_gpu_ste.py).  ste_gemm_kernel, the former fp32
// SIMT version, is kept as the A/B reference (AXQ_STE_SIMT=1).
#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "axq.h"
#include <climits>
#include "async_copy.cuh"

namespace axq {
axq_status cuda_fail_ext(int e);   // axq_api.cu: records the code for axq_last_cuda_error()
namespace ste {
constexpr int BM = 128, BN = 128, BK = 16, NT = 256;
}

// C[i][j] = mask(i, j) * sum_p A(i, p) * fl(s_b * B[p][j]),  A(i, p) = TA ? A[p*lda + i] : A[i*lda + p]
// Split K (blockIdx.z of gridDim.z, chunks of kc): each split writes its raw partial sums to
// C + z * M * ldc (a workspace slice); ste_reduce_kernel adds the slices in a fixed order and
// applies the mask.  One split: the mask is applied here.
template <bool TA>
__global__ void __launch_bounds__(ste::NT) ste_gemm_kernel(int64_t M, int64_t N, int64_t K, const float* __restrict__ A,
                                                       int64_t lda, const int8_t* __restrict__ B, int64_t ldb,
                                                       const float* __restrict__ s_b, float* __restrict__ C, int64_t ldc,
                                                       const float* __restrict__ R, int64_t ldr,
                                                       const float* __restrict__ clip, int64_t kc) {
    using namespace ste;
    const int64_t kb = (int64_t)blockIdx.z * kc, ke = min(K, kb + kc);
    C += (int64_t)blockIdx.z * M * ldc;
    if (gridDim.z > 1) R = nullptr;
    // double-buffered shared tiles; the next k-tile is fetched into registers while the
    // current one is multiplied (one barrier per k-tile)
    __shared__ __align__(16) float As[2][BK][BM + 4];
    __shared__ __align__(16) float Bs[2][BK][BN + 4];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    const float sb = *s_b;
    constexpr int LA = BM * BK / NT, LB = BN * BK / NT;
    float ra[LA];
    int rb[LB];   // raw codes: converted in stash(), after the current tile's FMAs (not stalling on the load)
    auto fetch = [&](int64_t k0) {
#pragma unroll
        for (int i = 0; i < LA; ++i) {
            const int idx = tid + i * NT;
            int r, c;
            if (TA) { c = idx / BM; r = idx - c * BM; }     // consecutive threads: consecutive rows
            else { r = idx / BK; c = idx - r * BK; }        // consecutive threads: consecutive k
            const int64_t m = m0 + r, k = k0 + c;
            ra[i] = (m < M && k < ke) ? (TA ? A[k * lda + m] : A[m * lda + k]) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < LB; ++i) {
            const int idx = tid + i * NT;
            const int kk = idx / BN, c = idx - kk * BN;
            const int64_t k = k0 + kk, n = n0 + c;
            rb[i] = (k < ke && n < N) ? (int)B[k * ldb + n] : 0;
        }
    };
    auto stash = [&](int buf) {
#pragma unroll
        for (int i = 0; i < LA; ++i) {
            const int idx = tid + i * NT;
            int r, c;
            if (TA) { c = idx / BM; r = idx - c * BM; }
            else { r = idx / BK; c = idx - r * BK; }
            As[buf][c][r] = ra[i];
        }
#pragma unroll
        for (int i = 0; i < LB; ++i) {
            const int idx = tid + i * NT;
            const int kk = idx / BN, c = idx - kk * BN;
            Bs[buf][kk][c] = __fmul_rn(sb, (float)rb[i]);   // fake-quant value fl(s * q)
        }
    };
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    int buf = 0;
    if (kb < ke) {
        fetch(kb);
        stash(0);
    }
    __syncthreads();
    for (int64_t k0 = kb; k0 < ke; k0 += BK) {
        const bool more = k0 + BK < ke;
        if (more) fetch(k0 + BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 8]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 8 + 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 8]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 8 + 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
        }
        if (more) stash(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
    const float cl = R ? *clip : 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t m = m0 + ty * 8 + i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t n = n0 + tx * 8 + j;
            if (n >= N) continue;
            float v = acc[i][j];
            if (R && !(fabsf(R[m * ldr + n]) <= cl)) v = 0.f;   // STE: outside the clip range
            C[m * ldc + n] = v;
        }
    }
}

// ---------------------------------------------------------------------------------------
// The same product on the 5th-generation tensor cores (tcgen05.mma kind::f16, fp32 accumulators
// in TMEM).  The int8 codes are exact in bf16; the fp32 operand A is split exactly into three
// bf16 terms hi + mid + lo (each the round-to-nearest bf16 of the remainder, so |A - hi - mid -
// lo| <= 2^-27 |A|, below fp32's own unit roundoff), and the three products accumulate into one
// TMEM accumulator: C = sum_p (hi + mid + lo)(i, p) * q(p, j), times the per-tensor scale s_b in
// the epilogue, or with a per-p scale s_b[p] folded into A first (fl(A * s_b[p])).
// CTA tile 128 (i) x 128 (j), 32 p per stage (2 MMAs of K = 16 per term), double-buffered; the
// 4 warps convert the operands of stage s+1 while the tensor cores run stage s; each thread owns
// one TMEM lane (row i) in the epilogue.
// ---------------------------------------------------------------------------------------
namespace stetc {
constexpr int BM = 128, BN = 128, BK = 32, NT = 256;
constexpr int A_TERM = BM * BK * 2;               // one bf16 term of the A tile: 8 KiB
constexpr int A_STAGE = 3 * A_TERM;               // hi, mid, lo
constexpr int B_STAGE = BN * BK * 2;              // 8 KiB
constexpr int STAGE = A_STAGE + B_STAGE;          // 32 KiB
constexpr int SMEM = 2 * STAGE + 64;              // + mbarriers / TMEM address
// instruction descriptor: D f32 (bits 4-5 = 1), A / B bf16 (7-9, 10-12 = 1), K-major, N >> 3,
// M >> 4
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
}  // namespace stetc

__device__ __forceinline__ uint64_t ste_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // SWIZZLE_NONE K-major: core matrices 8 rows x 16 B; LBO between K chunks, SBO between 8-row
    // groups; descriptor version 1 (sm_100)
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | ((uint64_t)1 << 46);
}

__device__ __forceinline__ uint16_t bf16_rn_bits(float x) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

// chunk layout of a [rows][32 k] bf16 tile: k chunk c (8 k = 16 B) at c * rows * 16, row r at r * 16
template <bool TA, bool PCS>
__global__ void __launch_bounds__(stetc::NT) ste_tc_kernel(int64_t M, int64_t N, int64_t K, const float* __restrict__ A,
                                                          int64_t lda, const int8_t* __restrict__ B, int64_t ldb,
                                                          const float* __restrict__ s_b, float* __restrict__ C,
                                                          int64_t ldc, const float* __restrict__ R, int64_t ldr,
                                                          const float* __restrict__ clip, int clip_vec, int64_t kc) {
    using namespace stetc;
    extern __shared__ __align__(1024) uint8_t st_smem[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const int64_t kb = (int64_t)blockIdx.z * kc, ke = min(K, kb + kc);
    C += (int64_t)blockIdx.z * M * ldc;
    const bool split = gridDim.z > 1;
    // row tiles on grid.x (up to 2^31 - 1: a conv's N*Ho*Wo positions), column tiles on grid.y
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(st_smem);
    const uint32_t bar = s_base + 2 * STAGE;                   // mma-done barriers [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(st_smem + 2 * STAGE + 16);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar + 8));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(tmem_slot)), "n"(BN) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const float sb = PCS ? 1.f : *s_b;

    // operand staging of the p-range [k0, k0 + 32) into stage buffer `buf`: thread t converts
    // row t of A (3 bf16 terms) and column t of B, 4 chunks of 8 p each
    // two threads per row / column: thread (row, half) converts the K chunks 2 half, 2 half + 1
    const int row = tid & (BM - 1), half = tid >> 7;
    const bool avec = !TA && ((lda & 3) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
    auto stage = [&](int buf, int64_t k0) {
        uint8_t* sa = st_smem + buf * STAGE;
        uint8_t* sbuf = sa + A_STAGE;
        const int64_t i = m0 + row, j = n0 + row;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            const int c = half * 2 + cc;
            const int64_t p0 = k0 + c * 8;
            float a[8];
            int8_t q[8];
            if (avec && i < M && p0 + 8 <= ke) {
                const float4 f0 = __ldg(reinterpret_cast<const float4*>(A + i * lda + p0));
                const float4 f1 = __ldg(reinterpret_cast<const float4*>(A + i * lda + p0) + 1);
                a[0] = f0.x; a[1] = f0.y; a[2] = f0.z; a[3] = f0.w;
                a[4] = f1.x; a[5] = f1.y; a[6] = f1.z; a[7] = f1.w;
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int64_t p = p0 + e;
                    a[e] = (p < ke && i < M) ? (TA ? __ldg(A + p * lda + i) : __ldg(A + i * lda + p)) : 0.f;
                }
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int64_t p = p0 + e;
                if (PCS && p < ke) a[e] = __fmul_rn(a[e], __ldg(s_b + p));   // per-channel scale of the summed index
                q[e] = (p < ke && j < N) ? B[p * ldb + j] : (int8_t)0;
            }
            uint32_t hw[4], mw[4], lw[4], bw[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
                uint16_t h[2], md[2], l[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const float x = a[e + u];
                    h[u] = bf16_rn_bits(x);
                    const float r1 = __fsub_rn(x, __bfloat162float(__ushort_as_bfloat16(h[u])));
                    md[u] = bf16_rn_bits(r1);
                    const float r2 = __fsub_rn(r1, __bfloat162float(__ushort_as_bfloat16(md[u])));
                    l[u] = bf16_rn_bits(r2);
                }
                hw[e / 2] = (uint32_t)h[0] | ((uint32_t)h[1] << 16);
                mw[e / 2] = (uint32_t)md[0] | ((uint32_t)md[1] << 16);
                lw[e / 2] = (uint32_t)l[0] | ((uint32_t)l[1] << 16);
                bw[e / 2] = (uint32_t)bf16_rn_bits((float)q[e]) | ((uint32_t)bf16_rn_bits((float)q[e + 1]) << 16);
            }
            const int off = c * BM * 16 + row * 16;
            *reinterpret_cast<uint4*>(sa + 0 * A_TERM + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(sa + 1 * A_TERM + off) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
            *reinterpret_cast<uint4*>(sa + 2 * A_TERM + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            *reinterpret_cast<uint4*>(sbuf + c * BN * 16 + row * 16) = make_uint4(bw[0], bw[1], bw[2], bw[3]);
        }
    };

    const int nst = (int)((ke - kb + BK - 1) / BK);
    uint32_t mma_phase[2] = {0u, 0u};
    if (nst > 0) stage(0, kb);
    for (int s = 0; s < nst; ++s) {
        const int buf = s & 1;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic stores -> MMA
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint32_t sa = s_base + buf * STAGE, sbb = sa + A_STAGE;
#pragma unroll
            for (int t = 0; t < 3; ++t)
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk) {
                    // K step of 16 = chunks 2kk, 2kk+1: LBO = one chunk (rows x 16 B), SBO = 128 B
                    const uint64_t ad = ste_desc(sa + t * A_TERM + kk * 2 * BM * 16, BM * 16, 128);
                    const uint64_t bd = ste_desc(sbb + kk * 2 * BN * 16, BN * 16, 128);
                    const uint32_t acc = (s > 0 || t > 0 || kk > 0) ? 1u : 0u;
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                                 "l"(ad), "l"(bd), "r"(IDESC), "r"(acc)
                                 : "memory");
                }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             bar + 8 * buf) : "memory");
        }
        if (s + 1 < nst) {
            if (s >= 1) {   // buffer buf ^ 1 was read by the MMAs of stage s - 1
                asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                             "@!p bra W_%=;\n}\n" ::"r"(bar + 8 * (buf ^ 1)), "r"(mma_phase[buf ^ 1]) : "memory");
                mma_phase[buf ^ 1] ^= 1u;
            }
            stage(buf ^ 1, kb + (int64_t)(s + 1) * BK);
        }
    }
    // wait for the last MMAs (and the one before it, if its barrier phase is still pending)
    if (nst >= 2) {
        const int b2 = (nst - 2) & 1;
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                     "@!p bra W_%=;\n}\n" ::"r"(bar + 8 * b2), "r"(mma_phase[b2]) : "memory");
        mma_phase[b2] ^= 1u;
    }
    if (nst >= 1) {
        const int b1 = (nst - 1) & 1;
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                     "@!p bra W_%=;\n}\n" ::"r"(bar + 8 * b1), "r"(mma_phase[b1]) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // ---- epilogue: warp w reads TMEM lane quarter w % 4 (rows), column half w / 4 ----
    const int erow = (warp & 3) * 32 + (tid & 31);
    const int64_t i = m0 + erow;
    const float cl = (R && !split) ? (clip_vec ? (i < M ? clip[i] : 0.f) : *clip) : 0.f;
#pragma unroll 1
    for (int c0 = (warp >> 2) * (BN / 2); c0 < (warp >> 2) * (BN / 2) + BN / 2; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (i >= M) continue;
        if (nst == 0) {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = 0u;
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int64_t j = n0 + c0 + e;
            if (j >= N) continue;
            float x = __uint_as_float(v[e]);
            if (!PCS) x = __fmul_rn(x, sb);
            if (R && !split && !(fabsf(R[i * ldr + j]) <= cl)) x = 0.f;   // STE: outside the clip range
            C[i * ldc + j] = x;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(BN) : "memory");
}

// C[i] = mask(i) * sum_{z < S} part[z][i], the splits added in order (deterministic); clip_vec:
// the clip is per row (clip[i / N], a per-channel weight clip), else one scalar
__global__ void ste_reduce_kernel(int S, int64_t MN, int64_t N, const float* __restrict__ part,
                                  float* __restrict__ C, const float* __restrict__ R,
                                  const float* __restrict__ clip, int clip_vec) {
    const float cl0 = (R && !clip_vec) ? *clip : 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < MN; i += (int64_t)gridDim.x * blockDim.x) {
        float v = part[i];
        for (int z = 1; z < S; ++z) v = __fadd_rn(v, part[(int64_t)z * MN + i]);
        if (R && !(fabsf(R[i]) <= (clip_vec ? clip[i / N] : cl0))) v = 0.f;
        C[i] = v;
    }
}

// Column sums over many rows, deterministic: block (column group of 32, row block rb) sums its
// rows per warp (rows w, w + 8, ...), the 8 warps in order, into part[rb][n]; run again over
// part with one row block it adds the row blocks in order.
__global__ void __launch_bounds__(256) ste_colsum_part_kernel(int64_t M, int64_t N, const float* __restrict__ gy,
                                                              int64_t ldg, float* __restrict__ part) {
    __shared__ float red[8][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n = (int64_t)blockIdx.x * 32 + lane;
    const int64_t rows = (M + gridDim.y - 1) / gridDim.y, r0 = (int64_t)blockIdx.y * rows, r1 = min(M, r0 + rows);
    float s = 0.f;
    if (n < N) {
#pragma unroll 8
        for (int64_t m = r0 + warp; m < r1; m += 8) s = __fadd_rn(s, __ldg(gy + m * ldg + n));
    }
    red[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && n < N) {
        float t = red[0][lane];
        for (int w = 1; w < 8; ++w) t = __fadd_rn(t, red[w][lane]);
        part[(int64_t)blockIdx.y * N + n] = t;
    }
}


}  // namespace axq

#include "ste_pp.cuh"

namespace axq {
// The pre-converted path of one product on its own (prep launch + GEMM launch [+ reduce]):
// the workspace holds the partial slots (slots > 1 only), A' and B'.  Returns false (nothing
// launched) when the workspace cannot hold A' and B' -- the caller then runs ste_tc_kernel.
static bool ste_prep_product(bool ta, int64_t Mg, int64_t Ng, int64_t Kg, const float* A, int64_t lda,
                             const int8_t* B, int64_t ldb, const float* sB, bool sB_vec, float* C, int64_t ldc,
                             const float* R, const float* clip, bool clip_vec, float* workspace,
                             int64_t workspace_elems, int sms, cudaStream_t st,
                             const stepp::ConvGeo* conv_b = nullptr) {
    PrepPlan pl;
    if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return false;
    if (!pp_plan(Mg, Ng, Kg, ldc, sms, 0, pl)) return false;
    const int64_t ab = pp_ab_elems(pl);
    if (workspace_elems < ab) return false;
    if (!pp_plan(Mg, Ng, Kg, ldc, sms, workspace_elems - ab, pl)) return false;
    uint4* Ap = reinterpret_cast<uint4*>(workspace + pl.part);
    uint4* Bp = reinterpret_cast<uint4*>(workspace + pl.part + round32(pl.a_elems));
    stepp::PrepArgs pa{};
    pa.job[0] = pp_job_a(ta, Mg, Kg, A, lda, sB, sB_vec, pl.KT, Ap, sms);
    pa.job[1] = conv_b ? pp_job_b_conv(Ng, Kg, B, *conv_b, pl.KT, Bp, sms) : pp_job_b(Ng, Kg, B, ldb, pl.KT, Bp, sms);
    pa.njobs = 2;
    pp_launch_prep(pa, st);
    stepp::GemmArgs ga{};
    ga.job[0] = pp_job_gemm(pl, Mg, Ng, ldc, Ap, Bp, sB, sB_vec, pl.slots > 1 ? workspace : C, R, clip, clip_vec, 0);
    ga.njobs = 1;
    pp_launch_gemm(ga, pl.CZ, pp_ctas(pl, pl.CZ), st);
    if (pl.slots > 1)
        ste_reduce_kernel<<<(unsigned)std::min<int64_t>((Mg * ldc + 255) / 256, 8 * sms), 256, 0, st>>>(
            (int)pl.slots, Mg * ldc, Ng, workspace, C, R, clip, clip_vec ? 1 : 0);
    return true;
}

// One STE product C[Mg][Ng] = mask * A(Mg x Kg) . fq(B[Kg][ldb]) (R: mask operand [Mg][Ng] or null)
// on the tensor cores (ste_tc_kernel); sB_vec: the scale is per summed index p (per-channel
// weight scales of gx), else one scalar; clip_vec: the clip is per output row i (per-channel
// weight clip of gw).  Split K (deterministic, through the workspace) until ~2 CTAs per SM.
static void ste_product(bool ta, int64_t Mg, int64_t Ng, int64_t Kg, const float* A, int64_t lda,
                        const int8_t* B, int64_t ldb, const float* sB, bool sB_vec, float* C, int64_t ldc,
                        const float* R, const float* clip, bool clip_vec, float* workspace, int64_t workspace_elems,
                        cudaStream_t st) {
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static unsigned configured = 0;
    if (!(configured & (1u << (dev & 31)))) {
        cudaFuncSetAttribute(ste_tc_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, stetc::SMEM);
        cudaFuncSetAttribute(ste_tc_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, stetc::SMEM);
        cudaFuncSetAttribute(ste_tc_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, stetc::SMEM);
        cudaFuncSetAttribute(ste_tc_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, stetc::SMEM);
        configured |= 1u << (dev & 31);
    }
    static const bool simt = std::getenv("AXQ_STE_SIMT") != nullptr;   // A/B: the fp32 SIMT GEMM
    if (simt && !sB_vec && !clip_vec && (Mg + ste::BM - 1) / ste::BM <= 65535) {
        const int64_t t2 = ((Ng + ste::BN - 1) / ste::BN) * ((Mg + ste::BM - 1) / ste::BM);
        int64_t S2 = std::min<int64_t>({(2 * (int64_t)sms + t2 - 1) / t2, 128, std::max<int64_t>(1, Kg / 64)});
        S2 = workspace ? std::min<int64_t>(S2, workspace_elems / std::max<int64_t>(1, Mg * ldc)) : 1;
        if (S2 < 2) S2 = 1;
        const int64_t kc2 = ((Kg + S2 - 1) / S2 + ste::BK - 1) / ste::BK * ste::BK;
        S2 = (Kg + kc2 - 1) / kc2;
        dim3 g2((unsigned)((Ng + ste::BN - 1) / ste::BN), (unsigned)((Mg + ste::BM - 1) / ste::BM), (unsigned)S2);
        float* o2 = S2 > 1 ? workspace : C;
        if (ta) ste_gemm_kernel<true><<<g2, ste::NT, 0, st>>>(Mg, Ng, Kg, A, lda, B, ldb, sB, o2, ldc, R, ldc, clip, kc2);
        else ste_gemm_kernel<false><<<g2, ste::NT, 0, st>>>(Mg, Ng, Kg, A, lda, B, ldb, sB, o2, ldc, R, ldc, clip, kc2);
        if (S2 > 1)
            ste_reduce_kernel<<<(unsigned)std::min<int64_t>((Mg * ldc + 255) / 256, 8 * sms), 256, 0, st>>>(
                (int)S2, Mg * ldc, Ng, workspace, C, R, clip, 0);
        return;
    }
    const int64_t tiles = ((Ng + stetc::BN - 1) / stetc::BN) * ((Mg + stetc::BM - 1) / stetc::BM);
    static const bool noprep = std::getenv("AXQ_STE_NOPREP") != nullptr;   // A/B: the in-kernel conversion
    if (!noprep && workspace && ste_prep_product(ta, Mg, Ng, Kg, A, lda, B, ldb, sB, sB_vec, C, ldc, R, clip, clip_vec,
                                                 workspace, workspace_elems, sms, st))
        return;
    // (a conv's weight gradient sums over all N*Ho*Wo positions into a few tiles: up to 128 slices)
    int64_t S = std::min<int64_t>({(2 * (int64_t)sms + tiles - 1) / tiles, 128, std::max<int64_t>(1, Kg / 128)});
    S = workspace ? std::min<int64_t>(S, workspace_elems / std::max<int64_t>(1, Mg * ldc)) : 1;
    if (S < 2) S = 1;
    const int64_t kc = ((Kg + S - 1) / S + stetc::BK - 1) / stetc::BK * stetc::BK;
    S = (Kg + kc - 1) / kc;
    dim3 grid((unsigned)((Mg + stetc::BM - 1) / stetc::BM), (unsigned)((Ng + stetc::BN - 1) / stetc::BN), (unsigned)S);
    float* out = S > 1 ? workspace : C;
    const int cv = clip_vec ? 1 : 0;
    if (ta) {
        if (sB_vec) ste_tc_kernel<true, true><<<grid, stetc::NT, stetc::SMEM, st>>>(Mg, Ng, Kg, A, lda, B, ldb, sB, out, ldc, R, ldc, clip, cv, kc);
        else ste_tc_kernel<true, false><<<grid, stetc::NT, stetc::SMEM, st>>>(Mg, Ng, Kg, A, lda, B, ldb, sB, out, ldc, R, ldc, clip, cv, kc);
    } else {
        if (sB_vec) ste_tc_kernel<false, true><<<grid, stetc::NT, stetc::SMEM, st>>>(Mg, Ng, Kg, A, lda, B, ldb, sB, out, ldc, R, ldc, clip, cv, kc);
        else ste_tc_kernel<false, false><<<grid, stetc::NT, stetc::SMEM, st>>>(Mg, Ng, Kg, A, lda, B, ldb, sB, out, ldc, R, ldc, clip, cv, kc);
    }
    if (S > 1)
        ste_reduce_kernel<<<(unsigned)std::min<int64_t>((Mg * ldc + 255) / 256, 8 * sms), 256, 0, st>>>(
            (int)S, Mg * ldc, Ng, workspace, C, R, clip, cv);
}

// gb = column sums of gy [M][N], deterministic: RB = ceil(M / 128) row blocks (a function of M
// only, <= 1024; ~16 rows per warp) summed by ste_colsum_part_kernel into RB x N partials, which
// the same kernel then adds in order (one row block); RB < 4 (or no workspace for the
// partials): one pass straight into gb.
static int64_t ste_colsum_rb(int64_t M) {
    const int64_t RB = std::min<int64_t>(1024, (M + 127) / 128);
    return RB >= 4 ? RB : 1;
}
static void ste_colsum(int64_t M, int64_t N, const float* gy, float* gb, float* workspace, int64_t workspace_elems,
                       cudaStream_t st) {
    const int64_t cg = (N + 31) / 32;
    int64_t RB = ste_colsum_rb(M);
    if (!workspace || workspace_elems < RB * N) RB = 1;
    if (RB > 1) {
        ste_colsum_part_kernel<<<dim3((unsigned)cg, (unsigned)RB), 256, 0, st>>>(M, N, gy, N, workspace);
        ste_colsum_part_kernel<<<dim3((unsigned)cg, 1), 256, 0, st>>>(RB, N, workspace, N, gb);
    } else {
        ste_colsum_part_kernel<<<dim3((unsigned)cg, 1), 256, 0, st>>>(M, N, gy, N, gb);
    }
}

// gx[n][h][w][c] = mask * sum_{r, s} gcols[(n, ho, wo)][(r, s, c)] over the output positions whose
// window covers (h, w) (the adjoint of im2col; r, s in ascending order: deterministic)
__global__ void ste_col2im_kernel(int64_t total, int H, int W, int C, int R, int S, int sh, int sw, int ph,
                                  int pw, int Ho, int Wo, const float* __restrict__ gcols, int64_t ldg,
                                  const float* __restrict__ x, const float* __restrict__ clip,
                                  float* __restrict__ gx) {
    const float cl = x ? *clip : 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % C);
        int64_t t = i / C;
        const int w_ = (int)(t % W);
        t /= W;
        const int h = (int)(t % H);
        const int64_t n = t / H;
        float acc = 0.f;
        for (int r = 0; r < R; ++r) {
            const int hh = h + ph - r;
            if (hh < 0 || hh % sh) continue;
            const int ho = hh / sh;
            if (ho >= Ho) continue;
            for (int s_ = 0; s_ < S; ++s_) {
                const int ww = w_ + pw - s_;
                if (ww < 0 || ww % sw) continue;
                const int wo = ww / sw;
                if (wo >= Wo) continue;
                acc = __fadd_rn(acc, gcols[((n * Ho + ho) * Wo + wo) * ldg + ((int64_t)r * S + s_) * C + c]);
            }
        }
        if (x && !(fabsf(x[i]) <= cl)) acc = 0.f;
        gx[i] = acc;
    }
}

// col2im for C % 4 == 0 and 32-bit indices: one thread per 4 channels of one input pixel (float4
// gathers of gcols, the same (r, s) order as ste_col2im_kernel)
__global__ void __launch_bounds__(256) ste_col2im4_kernel(int total4, int H, int W, int C4, int R, int S, int sh,
                                                          int sw, int ph, int pw, int Ho, int Wo,
                                                          const float4* __restrict__ gcols, int ldg4,
                                                          const float4* __restrict__ x,
                                                          const float* __restrict__ clip, float4* __restrict__ gx) {
    const float cl = x ? *clip : 0.f;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total4; i += gridDim.x * blockDim.x) {
        const int c4 = i % C4;
        int t = i / C4;
        const int w_ = t % W;
        t /= W;
        const int h = t % H;
        const int n = t / H;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = 0; r < R; ++r) {
            const int hh = h + ph - r;
            if (hh < 0 || hh % sh) continue;
            const int ho = hh / sh;
            if (ho >= Ho) continue;
            for (int s_ = 0; s_ < S; ++s_) {
                const int ww = w_ + pw - s_;
                if (ww < 0 || ww % sw) continue;
                const int wo = ww / sw;
                if (wo >= Wo) continue;
                const float4 g = __ldg(gcols + ((int64_t)(n * Ho + ho) * Wo + wo) * ldg4 + (r * S + s_) * C4 + c4);
                acc.x = __fadd_rn(acc.x, g.x); acc.y = __fadd_rn(acc.y, g.y);
                acc.z = __fadd_rn(acc.z, g.z); acc.w = __fadd_rn(acc.w, g.w);
            }
        }
        if (x) {
            const float4 xv = __ldg(x + i);
            if (!(fabsf(xv.x) <= cl)) acc.x = 0.f;
            if (!(fabsf(xv.y) <= cl)) acc.y = 0.f;
            if (!(fabsf(xv.z) <= cl)) acc.z = 0.f;
            if (!(fabsf(xv.w) <= cl)) acc.w = 0.f;
        }
        gx[i] = acc;
    }
}
}  // namespace axq

namespace axq {
static int ste_sms() {
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        sms = 148;
    }
    return sms > 0 ? sms : 148;
}
static int64_t ste_colsum_need(int64_t M, int64_t N) {
    if (M <= 0 || N <= 0) return 0;
    const int64_t RB = ste_colsum_rb(M);
    return RB > 1 ? RB * N : 0;
}
static int64_t ste_product_need(int64_t Mg, int64_t Ng, int64_t Kg, int64_t ldc, int sms) {
    PrepPlan pl;
    if (Mg <= 0 || Ng <= 0 || Kg <= 0) return 0;
    if (!pp_plan(Mg, Ng, Kg, ldc, sms, INT64_MAX / 4, pl)) return 0;
    return pl.part + pp_ab_elems(pl);
}

// The fused linear backward (one prep launch, one GEMM launch for gx and gw): both products
// with at most 8 K slices, sharing the larger cluster size.  Workspace: A'x B'x A'w B'w, then the
// column-sum partials.
struct FusedPlan {
    bool ok;
    PrepPlan px, pw;
    int64_t cz, rb, need;
};
static FusedPlan ste_fused_plan(int64_t M, int64_t N, int64_t K, bool hx, bool hw, bool hb, int sms) {
    FusedPlan f{};
    if (K <= 0 || (!hx && !hw)) return f;
    // room 0: a product wanting more than one cluster of slices gets exactly one (S = CZ); one
    // wanting more than 8 (a long summed dimension) runs alone with partial slots instead
    if (hx && (!pp_plan(M, K, N, K, sms, 0, f.px) || f.px.S0 > 8)) return f;
    if (hw && (!pp_plan(N, K, M, K, sms, 0, f.pw) || f.pw.S0 > 8)) return f;
    // slices for the launch as a whole: ~2 CTAs per SM over both products' tiles (a power of two
    // <= the cluster cap), each product capped at >= 4 k tiles per slice
    const int64_t tiles = (hx ? f.px.Mt * f.px.Nt : 0) + (hw ? f.pw.Mt * f.pw.Nt : 0);
    int64_t S = 1;
    while (S < pp_max_cz() && S * tiles < 2 * (int64_t)sms) S *= 2;
    auto cap = [](const PrepPlan& p, int64_t s) {
        while (s > 1 && s * 4 > p.KT) s /= 2;
        return s;
    };
    if (hx) pp_set_s(f.px, cap(f.px, S));
    if (hw) pp_set_s(f.pw, cap(f.pw, S));
    f.cz = std::max<int64_t>(hx ? f.px.CZ : 1, hw ? f.pw.CZ : 1);   // each keeps its own S <= cz
    f.rb = hb ? ste_colsum_rb(M) : 1;
    f.need = (hx ? pp_ab_elems(f.px) : 0) + (hw ? pp_ab_elems(f.pw) : 0) + (f.rb > 1 ? round32(f.rb * N) : 0);
    f.ok = true;
    return f;
}
}  // namespace axq

extern "C" int64_t axq_ste_linear_workspace_elems(int64_t M, int64_t N, int64_t K) {
    using namespace axq;
    if (M < 0 || N < 0 || K < 0 || M >= ((int64_t)1 << 40) || N >= ((int64_t)1 << 40) || K >= ((int64_t)1 << 40))
        return -1;
    const int sms = ste_sms();
    const FusedPlan f = ste_fused_plan(M, N, K, true, true, true, sms);
    return std::max<int64_t>({f.ok ? f.need : 0, ste_product_need(M, K, N, K, sms), ste_product_need(N, K, M, K, sms),
                              ste_colsum_need(M, N), 0});
}

extern "C" int64_t axq_ste_conv2d_workspace_elems(const axq_conv_desc* d) {
    using namespace axq;
    if (!d || d->N < 0 || d->H <= 0 || d->W <= 0 || d->C <= 0 || d->K <= 0 || d->R <= 0 || d->S <= 0 ||
        d->stride_h <= 0 || d->stride_w <= 0 || d->pad_h < 0 || d->pad_w < 0)
        return -1;
    const int64_t Ho = (d->H + 2 * d->pad_h - d->R) / d->stride_h + 1, Wo = (d->W + 2 * d->pad_w - d->S) / d->stride_w + 1;
    if (Ho <= 0 || Wo <= 0) return -1;
    const int64_t M = d->N * Ho * Wo, Kc = d->R * d->S * d->C, No = d->K;
    const int sms = ste_sms();
    return std::max<int64_t>({ste_product_need(No, Kc, M, Kc, sms), ste_product_need(M, Kc, No, Kc, sms),
                              ste_colsum_need(M, No), 0});
}

extern "C" axq_status axq_ste_linear_backward_pc(int64_t M, int64_t N, int64_t K, const float* gy,
                                                 const int8_t* qa, const float* d_scale_a, const float* x,
                                                 const float* d_clip_a, const int8_t* qw,
                                                 const float* d_scale_w, const float* d_scale_w_ch,
                                                 const float* w, const float* d_clip_w,
                                                 const float* d_clip_w_ch, float* gx, float* gw, float* gb,
                                                 float* workspace, int64_t workspace_elems, void* stream) {
    using namespace axq;
    if (M < 0 || N < 0 || K < 0) return AXQ_ERR_INVALID;
    if (M >= ((int64_t)1 << 40) || N >= ((int64_t)1 << 40) || K >= ((int64_t)1 << 40)) return AXQ_ERR_INVALID;
    if (M == 0 || N == 0) {   // empty sums: every gradient that exists is zero
        cudaStream_t st = (cudaStream_t)stream;
        cudaError_t e = cudaSuccess;
        if (gx && M * K > 0) e = cudaMemsetAsync(gx, 0, M * K * sizeof(float), st);
        if (e == cudaSuccess && gw && N * K > 0) e = cudaMemsetAsync(gw, 0, N * K * sizeof(float), st);
        if (e == cudaSuccess && gb && N > 0) e = cudaMemsetAsync(gb, 0, N * sizeof(float), st);
        return e == cudaSuccess ? AXQ_OK : cuda_fail_ext((int)e);
    }
    if (!gy) return AXQ_ERR_INVALID;
    const float* sw = d_scale_w_ch ? d_scale_w_ch : d_scale_w;
    const float* cw = d_clip_w_ch ? d_clip_w_ch : d_clip_w;
    if (gx && (!qw || !sw || (x && !d_clip_a))) return AXQ_ERR_INVALID;
    if (gw && (!qa || !d_scale_a || (w && !cw))) return AXQ_ERR_INVALID;
    if ((K + 127) / 128 > 65535 || (N + 127) / 128 > 65535) return AXQ_ERR_UNSUPPORTED;   // column tiles: grid.y
    cudaStream_t st = (cudaStream_t)stream;
    static const bool noprep = std::getenv("AXQ_STE_NOPREP") != nullptr;   // A/B: the in-kernel conversion
    const int sms = ste_sms();
    const FusedPlan f = ste_fused_plan(M, N, K, gx != nullptr, gw != nullptr, gb != nullptr, sms);
    if (!noprep && f.ok && workspace && (reinterpret_cast<uintptr_t>(workspace) & 15) == 0 &&
        workspace_elems >= f.need) {
        // one prep launch (A', B' of both products + the first column-sum pass), one GEMM launch
        float* wp = workspace;
        stepp::PrepArgs pa{};
        stepp::GemmArgs ga{};
        int64_t ctas = 0;
        if (gx) {   // gx[m][k] = mask * sum_n gy[m][n] * fq(qw)[n][k]
            uint4* Ap = reinterpret_cast<uint4*>(wp);
            uint4* Bp = reinterpret_cast<uint4*>(wp + round32(f.px.a_elems));
            wp += pp_ab_elems(f.px);
            pa.job[pa.njobs++] = pp_job_a(false, M, N, gy, N, sw, d_scale_w_ch != nullptr, f.px.KT, Ap, sms);
            pa.job[pa.njobs++] = pp_job_b(K, N, qw, K, f.px.KT, Bp, sms);
            ga.job[ga.njobs++] = pp_job_gemm(f.px, M, K, K, Ap, Bp, sw, d_scale_w_ch != nullptr, gx, x, d_clip_a,
                                             false, ctas);
            ctas += pp_ctas(f.px, f.cz);
        }
        if (gw) {   // gw[n][k] = mask * sum_m gy[m][n] * fq(qa)[m][k]
            uint4* Ap = reinterpret_cast<uint4*>(wp);
            uint4* Bp = reinterpret_cast<uint4*>(wp + round32(f.pw.a_elems));
            wp += pp_ab_elems(f.pw);
            pa.job[pa.njobs++] = pp_job_a(true, N, M, gy, N, d_scale_a, false, f.pw.KT, Ap, sms);
            pa.job[pa.njobs++] = pp_job_b(K, M, qa, K, f.pw.KT, Bp, sms);
            ga.job[ga.njobs++] = pp_job_gemm(f.pw, N, K, K, Ap, Bp, d_scale_a, false, gw, w, cw,
                                             d_clip_w_ch != nullptr, ctas);
            ctas += pp_ctas(f.pw, f.cz);
        }
        if (gb) pa.job[pa.njobs++] = pp_job_colsum(M, N, gy, f.rb, f.rb > 1 ? wp : gb, sms);
        pp_launch_prep(pa, st);
        pp_launch_gemm(ga, f.cz, ctas, st);
        if (gb && f.rb > 1)
            ste_colsum_part_kernel<<<dim3((unsigned)((N + 31) / 32), 1), 256, 0, st>>>(f.rb, N, wp, N, gb);
        const cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? AXQ_OK : cuda_fail_ext((int)e);
    }
    if (gx && K > 0)
        ste_product(false, M, K, N, gy, N, qw, K, sw, d_scale_w_ch != nullptr, gx, K, x, d_clip_a, false, workspace,
                    workspace_elems, st);
    if (gw && K > 0)
        ste_product(true, N, K, M, gy, N, qa, K, d_scale_a, false, gw, K, w, cw, d_clip_w_ch != nullptr, workspace,
                    workspace_elems, st);
    if (gb) ste_colsum(M, N, gy, gb, workspace, workspace_elems, st);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? AXQ_OK : cuda_fail_ext((int)e);
}

extern "C" axq_status axq_ste_linear_backward(int64_t M, int64_t N, int64_t K, const float* gy,
                                              const int8_t* qa, const float* d_scale_a, const float* x,
                                              const float* d_clip_a, const int8_t* qw,
                                              const float* d_scale_w, const float* w,
                                              const float* d_clip_w, float* gx, float* gw, float* gb,
                                              float* workspace, int64_t workspace_elems, void* stream) {
    return axq_ste_linear_backward_pc(M, N, K, gy, qa, d_scale_a, x, d_clip_a, qw, d_scale_w, nullptr, w, d_clip_w,
                                      nullptr, gx, gw, gb, workspace, workspace_elems, stream);
}

// NEXT-4 for convolution (groups = 1, dilation 1): the STE backward through the explicit im2col
// of the forward's codes (the conv is the GEMM of its im2col matrix), see include/axq.h.
extern "C" axq_status axq_ste_conv2d_backward_pc(const axq_conv_desc* d, const float* gy, const int8_t* qx,
                                                 const float* d_scale_a, const float* x, const float* d_clip_a,
                                                 const int8_t* qw, const float* d_scale_w,
                                                 const float* d_scale_w_ch, const float* w,
                                                 const float* d_clip_w, const float* d_clip_w_ch, float* gx,
                                                 float* gw, float* gb, int8_t* cols, int64_t ldcols,
                                                 float* gcols, float* workspace, int64_t workspace_elems,
                                                 void* stream) {
    using namespace axq;
    const float* sw = d_scale_w_ch ? d_scale_w_ch : d_scale_w;
    const float* cw = d_clip_w_ch ? d_clip_w_ch : d_clip_w;
    if (!d || d->groups != 1 || d->dil_h != 1 || d->dil_w != 1 || (d->c_valid && d->c_valid != d->C) ||
        d->N < 0 || d->H <= 0 || d->W <= 0 || d->C <= 0 || d->K <= 0 || d->R <= 0 || d->S <= 0 ||
        d->stride_h <= 0 || d->stride_w <= 0 || d->pad_h < 0 || d->pad_w < 0)
        return AXQ_ERR_INVALID;
    const int64_t Ho = (d->H + 2 * d->pad_h - d->R) / d->stride_h + 1, Wo = (d->W + 2 * d->pad_w - d->S) / d->stride_w + 1;
    if (Ho <= 0 || Wo <= 0) return AXQ_ERR_INVALID;
    const int64_t M = d->N * Ho * Wo, Kc = d->R * d->S * d->C, No = d->K;
    if (M >= ((int64_t)1 << 31) || d->N * d->H * d->W * d->C >= ((int64_t)1 << 40)) return AXQ_ERR_INVALID;
    if (!gy && M > 0) return AXQ_ERR_INVALID;
    if (gw && (!qx || !d_scale_a || !cols || ldcols < Kc || (ldcols & 15) || (w && !cw))) return AXQ_ERR_INVALID;
    if (gx && (!qw || !sw || !gcols || (x && !d_clip_a))) return AXQ_ERR_INVALID;
    if ((Kc + 127) / 128 > 65535 || (No + 127) / 128 > 65535) return AXQ_ERR_UNSUPPORTED;   // column tiles
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (M == 0) {   // empty sums
        if (gx) e = cudaMemsetAsync(gx, 0, d->N * d->H * d->W * d->C * sizeof(float), st);
        if (e == cudaSuccess && gw) e = cudaMemsetAsync(gw, 0, No * Kc * sizeof(float), st);
        if (e == cudaSuccess && gb) e = cudaMemsetAsync(gb, 0, No * sizeof(float), st);
        return e == cudaSuccess ? AXQ_OK : cuda_fail_ext((int)e);
    }
    static const bool noprep = std::getenv("AXQ_STE_NOPREP") != nullptr;
    if (gw) {   // gw[k][(r, s, c)] = mask * sum_m gy[m][k] * fq(im2col(qx)[m][(r, s, c)])
        // pre-converted path: B' gathered straight from qx (implicit im2col, cols unused);
        // otherwise the explicit im2col into cols
        const stepp::ConvGeo cg{(int)d->H, (int)d->W, (int)d->C, (int)Ho, (int)Wo, (int)d->stride_h,
                                (int)d->stride_w, (int)d->pad_h, (int)d->pad_w, (int)d->S};
        const bool small = d->H * d->W * d->C < ((int64_t)1 << 31);
        if (noprep || !small ||
            !ste_prep_product(true, No, Kc, M, gy, No, qx, 0, d_scale_a, false, gw, Kc, w, cw, d_clip_w_ch != nullptr,
                              workspace, workspace_elems, ste_sms(), st, &cg)) {
            const axq_status r = axq_im2col_nhwc_i8(qx, d->N, d->H, d->W, d->C, 0, d->R, d->S, d->stride_h,
                                                    d->stride_w, d->pad_h, d->pad_w, cols, ldcols, stream);
            if (r != AXQ_OK) return r;
            ste_product(true, No, Kc, M, gy, No, cols, ldcols, d_scale_a, false, gw, Kc, w, cw, d_clip_w_ch != nullptr,
                        workspace, workspace_elems, st);
        }
    }
    if (gx) {   // gcols = gy . fq(W) [M][(r, s, c)], then the adjoint of im2col, masked
        ste_product(false, M, Kc, No, gy, No, qw, Kc, sw, d_scale_w_ch != nullptr, gcols, Kc, nullptr, nullptr, false,
                    workspace, workspace_elems, st);
        const int64_t total = d->N * d->H * d->W * d->C;
        int sms = 148, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const bool al = ((reinterpret_cast<uintptr_t>(gcols) | reinterpret_cast<uintptr_t>(gx) |
                          reinterpret_cast<uintptr_t>(x)) & 15) == 0;
        if ((d->C & 3) == 0 && al && total < ((int64_t)1 << 31) && M * Kc < ((int64_t)1 << 33))
            ste_col2im4_kernel<<<(unsigned)std::min<int64_t>((total / 4 + 255) / 256, 16 * sms), 256, 0, st>>>(
                (int)(total / 4), (int)d->H, (int)d->W, (int)(d->C / 4), (int)d->R, (int)d->S, (int)d->stride_h,
                (int)d->stride_w, (int)d->pad_h, (int)d->pad_w, (int)Ho, (int)Wo,
                reinterpret_cast<const float4*>(gcols), (int)(Kc / 4), reinterpret_cast<const float4*>(x), d_clip_a,
                reinterpret_cast<float4*>(gx));
        else
            ste_col2im_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 16 * sms), 256, 0, st>>>(
                total, (int)d->H, (int)d->W, (int)d->C, (int)d->R, (int)d->S, (int)d->stride_h, (int)d->stride_w,
                (int)d->pad_h, (int)d->pad_w, (int)Ho, (int)Wo, gcols, Kc, x, d_clip_a, gx);
    }
    if (gb) ste_colsum(M, No, gy, gb, workspace, workspace_elems, st);
    e = cudaGetLastError();
    return e == cudaSuccess ? AXQ_OK : cuda_fail_ext((int)e);
}

extern "C" axq_status axq_ste_conv2d_backward(const axq_conv_desc* d, const float* gy, const int8_t* qx,
                                              const float* d_scale_a, const float* x, const float* d_clip_a,
                                              const int8_t* qw, const float* d_scale_w, const float* w,
                                              const float* d_clip_w, float* gx, float* gw, float* gb,
                                              int8_t* cols, int64_t ldcols, float* gcols, float* workspace,
                                              int64_t workspace_elems, void* stream) {
    return axq_ste_conv2d_backward_pc(d, gy, qx, d_scale_a, x, d_clip_a, qw, d_scale_w, nullptr, w, d_clip_w, nullptr,
                                      gx, gw, gb, cols, ldcols, gcols, workspace, workspace_elems, stream);
}

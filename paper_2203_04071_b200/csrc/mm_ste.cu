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

// ---------------------------------------------------------------------------------------
// Pre-converted operands ("prep" path): each operand is converted ONCE per product into the
// tiled canonical K-major layout the MMA reads, so a stage of the GEMM is a handful of bulk
// copies and the tensor cores are not starved by the per-tile fp32 -> bf16 conversion.
//   A' = [m tile][k tile][term hi / mid / lo][chunk 0..3][128 rows][8 bf16]   (3 x 8 KiB per tile pair)
//   B' = [n tile][k tile][chunk 0..3][128 rows][8 bf16]                      (8 KiB)
// (row = the GEMM's M resp. N index, chunk = 8 consecutive summed indices p.)
// ---------------------------------------------------------------------------------------
namespace stepp {
constexpr int BM = 128, BN = 128, BK = 32;
constexpr int TILE_A = 3 * BM * BK * 2;        // 24 KiB
constexpr int TILE_B = BN * BK * 2;            // 8 KiB
constexpr int STAGES = 3;
constexpr int STAGE = TILE_A + TILE_B;         // 32 KiB
constexpr int TS = BN + 4;                     // epilogue tile row stride (floats): conflict-free float4 rows
constexpr int SMEM = STAGES * STAGE + 128;     // 2 CTAs per SM
static_assert(BM * TS * 4 <= STAGES * STAGE, "epilogue tile must fit the stage buffers");
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
}  // namespace stepp

// thread -> (row, chunk) of one (m tile, k tile): 8 consecutive p of row i, split into 3 terms.
// TA (A[p][i]): row fastest, a warp reads 32 consecutive i per p; else chunk fastest, 4 threads
// read one row's 32 consecutive p (two float4 each when aligned).
template <bool TA, bool PCS>
__global__ void __launch_bounds__(256) ste_prep_a_kernel(int64_t M, int64_t K, const float* __restrict__ A,
                                                         int64_t lda, const float* __restrict__ s_b,
                                                         int64_t KT, int avec, uint4* __restrict__ out) {
    const int64_t total = ((M + 127) / 128) * KT * 4 * 128;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int row = TA ? (int)(g & 127) : (int)((g >> 2) & 127);
        const int c = TA ? (int)((g >> 7) & 3) : (int)(g & 3);
        const int64_t tk = g >> 9;                       // (m tile, k tile)
        const int64_t kt = tk % KT, mt = tk / KT;
        const int64_t i = mt * 128 + row, p0 = kt * 32 + c * 8;
        float a[8];
        if (!TA && avec && i < M && p0 + 8 <= K) {
            const float4 f0 = __ldg(reinterpret_cast<const float4*>(A + i * lda + p0));
            const float4 f1 = __ldg(reinterpret_cast<const float4*>(A + i * lda + p0) + 1);
            a[0] = f0.x; a[1] = f0.y; a[2] = f0.z; a[3] = f0.w;
            a[4] = f1.x; a[5] = f1.y; a[6] = f1.z; a[7] = f1.w;
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int64_t p = p0 + e;
                a[e] = (i < M && p < K) ? (TA ? __ldg(A + p * lda + i) : __ldg(A + i * lda + p)) : 0.f;
            }
        }
        if (PCS) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (p0 + e < K) a[e] = __fmul_rn(a[e], __ldg(s_b + p0 + e));   // per-channel scale of p
        }
        uint32_t hw[4], mw[4], lw[4];
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
        }
        uint4* base = out + tk * (3 * 4 * 128) + c * 128 + row;      // in 16-byte units
        base[0] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        base[4 * 128] = make_uint4(mw[0], mw[1], mw[2], mw[3]);
        base[8 * 128] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

// thread -> (4 columns j .. j + 3, chunk) of one (n tile, k tile): the int8 codes B[p][j] of 8
// consecutive p, one 4-byte load per p when aligned, as bf16 (exact) into 4 rows of the tile
__global__ void __launch_bounds__(256) ste_prep_b_kernel(int64_t N, int64_t K, const int8_t* __restrict__ B,
                                                         int64_t ldb, int64_t KT, int bvec, uint4* __restrict__ out) {
    const int64_t total = ((N + 127) / 128) * KT * 4 * 32;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int rq = (int)(g & 31), c = (int)((g >> 5) & 3);
        const int64_t tk = g >> 7;
        const int64_t kt = tk % KT, nt = tk / KT;
        const int64_t j0 = nt * 128 + rq * 4, p0 = kt * 32 + c * 8;
        uint32_t q[8];     // q[e] = bytes of B[p0 + e][j0 .. j0 + 3]
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int64_t p = p0 + e;
            uint32_t v = 0u;
            if (p < K) {
                if (bvec && j0 + 4 <= N) {
                    v = __ldg(reinterpret_cast<const unsigned int*>(B + p * ldb + j0));
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (j0 + u < N) v |= (uint32_t)(uint8_t)B[p * ldb + j0 + u] << (8 * u);
                }
            }
            q[e] = v;
        }
        uint4* base = out + tk * (4 * 128) + c * 128 + rq * 4;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
                const float f0 = (float)(int8_t)(q[e] >> (8 * u)), f1 = (float)(int8_t)(q[e + 1] >> (8 * u));
                w[e / 2] = (uint32_t)bf16_rn_bits(f0) | ((uint32_t)bf16_rn_bits(f1) << 16);
            }
            base[u] = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

// C tile (128 x 128) of split z from the pre-converted operands: thread 0 streams the stages
// (one bulk copy per operand), thread 32 issues the MMAs.  Epilogue: the 4 warps move the TMEM
// accumulator into a padded shared-memory tile; the CZ CTAs of a cluster (the split-K slices
// z = CZ * c .. CZ * c + CZ - 1 of one output tile) then reduce their tiles through distributed
// shared memory, CTA rank q owning rows [q * 128 / CZ, (q + 1) * 128 / CZ), adding the slices
// in rank order (deterministic), and write those rows with coalesced 512-byte row stores --
// to C (scaled, masked) when the cluster covers every slice, else (scaled) to partial slot c of
// the workspace for ste_reduce_kernel.
template <bool PCS>
__global__ void __launch_bounds__(128) ste_pp_kernel(int64_t M, int64_t N, int64_t KT, const uint4* __restrict__ Ap,
                                                     const uint4* __restrict__ Bp, const float* __restrict__ s_b,
                                                     float* __restrict__ C, int64_t ldc, const float* __restrict__ R,
                                                     int64_t ldr, const float* __restrict__ clip, int clip_vec,
                                                     int64_t kts_per_split, int CZ) {
    using namespace stepp;
    extern __shared__ __align__(1024) uint8_t pp_smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t mt = blockIdx.x, nt = blockIdx.y;
    const int64_t kt0 = (int64_t)blockIdx.z * kts_per_split, kt1 = min(KT, kt0 + kts_per_split);
    const int nkt = (int)max((int64_t)0, kt1 - kt0);
    const bool final_out = (int)gridDim.z == CZ;           // the cluster holds every K slice
    if (!final_out) C += (int64_t)(blockIdx.z / CZ) * M * ldc;
    const uint32_t s_base = smem_u32(pp_smem);
    const uint32_t bar_full = s_base + STAGES * STAGE, bar_mma = bar_full + 8 * STAGES;
    const uint32_t bar_done = bar_mma + 8 * STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pp_smem + STAGES * STAGE + 16 * STAGES + 8);
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_mma + 8 * s, 1);
        }
        mbar_init(bar_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(BN) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    if (tid == 0) {
        // producer: stage s <- k tile kt0 + s (A' 24 KiB + B' 8 KiB, two bulk copies)
        for (int s = 0; s < nkt; ++s) {
            const int buf = s % STAGES;
            if (s >= STAGES) mbar_wait(bar_mma + 8 * buf, ((s / STAGES) - 1) & 1u);
            const uint32_t bar = bar_full + 8 * buf;
            mbar_expect_tx(bar, STAGE);
            const int64_t kt = kt0 + s;
            bulk_g2s(s_base + buf * STAGE, Ap + (mt * KT + kt) * (3 * 4 * 128), TILE_A, bar);
            bulk_g2s(s_base + buf * STAGE + TILE_A, Bp + (nt * KT + kt) * (4 * 128), TILE_B, bar);
        }
    } else if (tid == 32) {
        // MMA issuer: 3 terms x 2 K steps of 16 per stage into one TMEM accumulator
        for (int s = 0; s < nkt; ++s) {
            const int buf = s % STAGES;
            mbar_wait(bar_full + 8 * buf, (s / STAGES) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint32_t sa = s_base + buf * STAGE, sbb = sa + TILE_A;
#pragma unroll
            for (int t = 0; t < 3; ++t)
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk) {
                    const uint64_t ad = ste_desc(sa + t * (TILE_A / 3) + kk * 2 * BM * 16, BM * 16, 128);
                    const uint64_t bd = ste_desc(sbb + kk * 2 * BN * 16, BN * 16, 128);
                    const uint32_t acc = (s > 0 || t > 0 || kk > 0) ? 1u : 0u;
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                                 "l"(ad), "l"(bd), "r"(IDESC), "r"(acc)
                                 : "memory");
                }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             bar_mma + 8 * buf) : "memory");
        }
        if (nkt > 0)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             bar_done) : "memory");
    }
    // everyone waits for all MMAs: one more commit onto bar_done (single phase; a per-stage
    // barrier's parity would alias with its phase STAGES stages earlier)
    if (nkt > 0) mbar_wait(bar_done, 0u);
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // TMEM -> shared tile T[128][TS] (row = TMEM lane; the stage buffers are idle now)
    float* T = reinterpret_cast<float*>(pp_smem);
    {
        const int r = warp * 32 + lane;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
            uint32_t v[16];
            const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            if (nkt == 0) {
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = 0u;
            }
            float4* dst = reinterpret_cast<float4*>(T + r * TS + c0);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                dst[e] = make_float4(__uint_as_float(v[4 * e]), __uint_as_float(v[4 * e + 1]),
                                     __uint_as_float(v[4 * e + 2]), __uint_as_float(v[4 * e + 3]));
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    uint32_t q = 0;
    if (CZ > 1) {
        asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(q));
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else {
        __syncthreads();
    }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(BN) : "memory");
    // rows [r0, r1) of the tile: lane l owns columns 4l .. 4l + 3, a warp one row at a time
    const int r0 = (int)(q * BM / CZ), r1 = (int)((q + 1) * BM / CZ);
    const float sb = PCS ? 1.f : *s_b;
    const bool apply_mask = R && final_out;
    const int64_t j = nt * BN + 4 * lane;
    const bool vec = j + 4 <= N && (ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
    const uint32_t t_base = smem_u32(T);
    for (int r = r0 + warp; r < r1; r += 4) {
        const int64_t i = mt * BM + r;
        if (i >= M) break;
        const uint32_t a = t_base + (uint32_t)(r * TS + 4 * lane) * 4u;
        float4 x;
        if (CZ == 1) {
            x = *reinterpret_cast<const float4*>(T + r * TS + 4 * lane);
        } else {
            x = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int z = 0; z < CZ; ++z) {
                uint32_t ra;
                float4 y;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(a), "r"(z));
                asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                             : "=f"(y.x), "=f"(y.y), "=f"(y.z), "=f"(y.w) : "r"(ra) : "memory");
                if (z == 0) {
                    x = y;
                } else {
                    x.x = __fadd_rn(x.x, y.x); x.y = __fadd_rn(x.y, y.y);
                    x.z = __fadd_rn(x.z, y.z); x.w = __fadd_rn(x.w, y.w);
                }
            }
        }
        if (!PCS) {
            x.x = __fmul_rn(x.x, sb); x.y = __fmul_rn(x.y, sb);
            x.z = __fmul_rn(x.z, sb); x.w = __fmul_rn(x.w, sb);
        }
        if (apply_mask) {
            const float cl = clip_vec ? clip[i] : *clip;
            const float* rr = R + i * ldr + j;
            if (j + 0 < N && !(fabsf(rr[0]) <= cl)) x.x = 0.f;
            if (j + 1 < N && !(fabsf(rr[1]) <= cl)) x.y = 0.f;
            if (j + 2 < N && !(fabsf(rr[2]) <= cl)) x.z = 0.f;
            if (j + 3 < N && !(fabsf(rr[3]) <= cl)) x.w = 0.f;
        }
        float* crow = C + i * ldc + j;
        if (vec) {
            *reinterpret_cast<float4*>(crow) = x;
        } else {
            if (j + 0 < N) crow[0] = x.x;
            if (j + 1 < N) crow[1] = x.y;
            if (j + 2 < N) crow[2] = x.z;
            if (j + 3 < N) crow[3] = x.w;
        }
    }
    if (CZ > 1)   // keep this CTA's tile alive until every rank of the cluster has read it
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
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
// rows per warp (rows w, w + 8, ...), the 8 warps in order, into part[rb][n]; ste_colsum_kernel
// then adds the row blocks in order.
constexpr int COLSUM_RB = 128;
__global__ void __launch_bounds__(256) ste_colsum_part_kernel(int64_t M, int64_t N, const float* __restrict__ gy,
                                                              int64_t ldg, float* __restrict__ part) {
    __shared__ float red[8][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n = (int64_t)blockIdx.x * 32 + lane;
    const int64_t rows = (M + gridDim.y - 1) / gridDim.y, r0 = (int64_t)blockIdx.y * rows, r1 = min(M, r0 + rows);
    float s = 0.f;
    if (n < N)
        for (int64_t m = r0 + warp; m < r1; m += 8) s = __fadd_rn(s, gy[m * ldg + n]);
    red[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && n < N) {
        float t = red[0][lane];
        for (int w = 1; w < 8; ++w) t = __fadd_rn(t, red[w][lane]);
        part[(int64_t)blockIdx.y * N + n] = t;
    }
}

// gb[n] = sum_m gy[m][n], sequential in m (one thread per column, coalesced rows)
__global__ void ste_colsum_kernel(int64_t M, int64_t N, const float* __restrict__ gy, int64_t ldg,
                                  float* __restrict__ gb) {
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    float s = 0.f;
    for (int64_t m = 0; m < M; ++m) s = __fadd_rn(s, gy[m * ldg + n]);
    gb[n] = s;
}

}  // namespace axq


namespace axq {
// Plan of the pre-converted path of one STE product (see stepp): the workspace holds, in order,
// the split-K partial slots (slots x Mg x ldc fp32, slots > 1 only), A' and B'.  K slices: ~2
// CTAs per SM, >= 4 k tiles each; up to 8 slices reduce inside a cluster (distributed shared
// memory), beyond that clusters of 8 write partial slots that ste_reduce_kernel adds in order.
struct PrepPlan {
    int64_t Mt, Nt, KT, a_elems, b_elems, S, CZ, slots, kps, part, need;
};
static int64_t round32(int64_t e) { return (e + 31) / 32 * 32; }
static bool ste_prep_plan(int64_t Mg, int64_t Ng, int64_t Kg, int64_t ldc, int sms, int64_t workspace_elems,
                          PrepPlan& pl) {
    using namespace stepp;
    pl.Mt = (Mg + BM - 1) / BM;
    pl.Nt = (Ng + BN - 1) / BN;
    pl.KT = (Kg + BK - 1) / BK;
    if (pl.Nt > 65535 || pl.Mt > 0x7fffffff || pl.KT == 0) return false;
    pl.a_elems = pl.Mt * pl.KT * (TILE_A / 4);
    pl.b_elems = pl.Nt * pl.KT * (TILE_B / 4);
    const int64_t ab = round32(pl.a_elems) + round32(pl.b_elems);
    if (workspace_elems < ab) return false;
    const int64_t tiles = pl.Mt * pl.Nt;
    int64_t S = std::min<int64_t>({(2 * (int64_t)sms + tiles - 1) / tiles, 128, std::max<int64_t>(1, pl.KT / 4)});
    pl.CZ = std::min<int64_t>(S, 8);
    if (S > 8) {
        const int64_t room = (workspace_elems - ab) / std::max<int64_t>(1, round32(Mg * ldc));
        const int64_t slots = std::min<int64_t>((S + 7) / 8, room);
        S = slots >= 2 ? slots * 8 : 8;
    }
    pl.kps = (pl.KT + S - 1) / S;
    if (S > 8) {   // drop whole clusters that would hold no k tile
        S = (pl.KT + pl.kps - 1) / pl.kps;
        S = std::max<int64_t>(8, (S + 7) / 8 * 8);
    }
    pl.S = S;
    pl.slots = S / pl.CZ;
    pl.part = pl.slots > 1 ? round32(pl.slots * Mg * ldc) : 0;
    pl.need = pl.part + ab;
    return pl.need <= workspace_elems;
}

static bool ste_prep_product(bool ta, int64_t Mg, int64_t Ng, int64_t Kg, const float* A, int64_t lda,
                             const int8_t* B, int64_t ldb, const float* sB, bool sB_vec, float* C, int64_t ldc,
                             const float* R, const float* clip, bool clip_vec, float* workspace,
                             int64_t workspace_elems, int sms, cudaStream_t st) {
    using namespace stepp;
    PrepPlan pl;
    if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return false;
    if (!ste_prep_plan(Mg, Ng, Kg, ldc, sms, workspace_elems, pl)) return false;
    const int64_t Mt = pl.Mt, Nt = pl.Nt, KT = pl.KT, S = pl.S, slots = pl.slots, kps = pl.kps;
    const int CZ = (int)pl.CZ;
    uint4* Ap = reinterpret_cast<uint4*>(workspace + pl.part);
    uint4* Bp = reinterpret_cast<uint4*>(workspace + pl.part + round32(pl.a_elems));
    static unsigned configured = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(configured & (1u << (dev & 31)))) {
        cudaFuncSetAttribute(ste_pp_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        cudaFuncSetAttribute(ste_pp_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        configured |= 1u << (dev & 31);
    }
    const unsigned pg = (unsigned)std::min<int64_t>((Mt * KT * 512 + 255) / 256, 16 * (int64_t)sms);
    const int avec = ((lda & 3) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0) ? 1 : 0;
    if (ta) {
        if (sB_vec) ste_prep_a_kernel<true, true><<<pg, 256, 0, st>>>(Mg, Kg, A, lda, sB, KT, avec, Ap);
        else ste_prep_a_kernel<true, false><<<pg, 256, 0, st>>>(Mg, Kg, A, lda, sB, KT, avec, Ap);
    } else {
        if (sB_vec) ste_prep_a_kernel<false, true><<<pg, 256, 0, st>>>(Mg, Kg, A, lda, sB, KT, avec, Ap);
        else ste_prep_a_kernel<false, false><<<pg, 256, 0, st>>>(Mg, Kg, A, lda, sB, KT, avec, Ap);
    }
    const unsigned pb = (unsigned)std::min<int64_t>((Nt * KT * 128 + 255) / 256, 16 * (int64_t)sms);
    const int bvec = ((ldb & 3) == 0 && (reinterpret_cast<uintptr_t>(B) & 3) == 0) ? 1 : 0;
    ste_prep_b_kernel<<<pb, 256, 0, st>>>(Ng, Kg, B, ldb, KT, bvec, Bp);
    float* out = slots > 1 ? workspace : C;
    const int cv = clip_vec ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)Mt, (unsigned)Nt, (unsigned)S);
    cfg.blockDim = dim3(128, 1, 1);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = (unsigned)CZ;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (sB_vec)
        cudaLaunchKernelEx(&cfg, ste_pp_kernel<true>, Mg, Ng, KT, (const uint4*)Ap, (const uint4*)Bp, sB, out, ldc, R, ldc,
                           clip, cv, kps, CZ);
    else
        cudaLaunchKernelEx(&cfg, ste_pp_kernel<false>, Mg, Ng, KT, (const uint4*)Ap, (const uint4*)Bp, sB, out, ldc, R,
                           ldc, clip, cv, kps, CZ);
    if (slots > 1)
        ste_reduce_kernel<<<(unsigned)std::min<int64_t>((Mg * ldc + 255) / 256, 8 * sms), 256, 0, st>>>(
            (int)slots, Mg * ldc, Ng, workspace, C, R, clip, cv);
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

// gb = column sums of gy [M][N], deterministic: RB row blocks (a function of M and N only, sized
// for ~2 blocks per SM of a 148-SM part) summed by ste_colsum_part_kernel, then added in order;
// RB = 1 (or no workspace for the RB x N partials): one pass straight into gb.
static void ste_colsum(int64_t M, int64_t N, const float* gy, float* gb, float* workspace, int64_t workspace_elems,
                       cudaStream_t st) {
    const int64_t cg = (N + 31) / 32;
    int64_t RB = std::min<int64_t>({(296 + cg - 1) / cg, COLSUM_RB, (M + 255) / 256});
    if (RB < 2 || !workspace || workspace_elems < RB * N) RB = 1;
    if (RB > 1) {
        ste_colsum_part_kernel<<<dim3((unsigned)cg, (unsigned)RB), 256, 0, st>>>(M, N, gy, N, workspace);
        ste_colsum_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(RB, N, workspace, N, gb);
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
    const int64_t cg = (N + 31) / 32;
    const int64_t RB = std::min<int64_t>({(296 + cg - 1) / cg, COLSUM_RB, (M + 255) / 256});
    return RB >= 2 ? RB * N : 0;
}
static int64_t ste_product_need(int64_t Mg, int64_t Ng, int64_t Kg, int64_t ldc, int sms) {
    PrepPlan pl;
    if (Mg <= 0 || Ng <= 0 || Kg <= 0) return 0;
    if (!ste_prep_plan(Mg, Ng, Kg, ldc, sms, INT64_MAX / 4, pl)) return 0;
    return pl.need;
}
}  // namespace axq

extern "C" int64_t axq_ste_linear_workspace_elems(int64_t M, int64_t N, int64_t K) {
    using namespace axq;
    if (M < 0 || N < 0 || K < 0 || M >= ((int64_t)1 << 40) || N >= ((int64_t)1 << 40) || K >= ((int64_t)1 << 40))
        return -1;
    const int sms = ste_sms();
    return std::max<int64_t>({ste_product_need(M, K, N, K, sms), ste_product_need(N, K, M, K, sms),
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
    if (gw) {   // gw[k][(r, s, c)] = mask * sum_m gy[m][k] * fq(im2col(qx)[m][(r, s, c)])
        const axq_status r = axq_im2col_nhwc_i8(qx, d->N, d->H, d->W, d->C, 0, d->R, d->S, d->stride_h, d->stride_w,
                                                d->pad_h, d->pad_w, cols, ldcols, stream);
        if (r != AXQ_OK) return r;
        ste_product(true, No, Kc, M, gy, No, cols, ldcols, d_scale_a, false, gw, Kc, w, cw, d_clip_w_ch != nullptr,
                    workspace, workspace_elems, st);
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

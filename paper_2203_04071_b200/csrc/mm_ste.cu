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
// Both products are one fp32 SIMT GEMM kernel (128 x 128 x 16 tiles, 8 x 8 outputs per thread,
// fp32 FMA accumulation): the int8 operand is dequantized while it is staged into shared memory
// and the STE mask is applied in the epilogue.  fp32 FMA, not tensor cores: the result is
// compared with the fp64 oracle under the fp32 dot-product error bound (tests/test_gpu_ste.py).
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "axq.h"

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

// C[i] = mask(i) * sum_{z < S} part[z][i], the splits added in order (deterministic)
__global__ void ste_reduce_kernel(int S, int64_t MN, int64_t N, const float* __restrict__ part,
                                  float* __restrict__ C, const float* __restrict__ R,
                                  const float* __restrict__ clip) {
    const float cl = R ? *clip : 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < MN; i += (int64_t)gridDim.x * blockDim.x) {
        float v = part[i];
        for (int z = 1; z < S; ++z) v = __fadd_rn(v, part[(int64_t)z * MN + i]);
        if (R && !(fabsf(R[i]) <= cl)) v = 0.f;
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
// One STE product C[Mg][Ng] = mask * A(Mg x Kg) . fq(B[Kg][ldb]) (R: mask operand [Mg][Ng] or null):
// split K (deterministic, through the workspace) until ~2 CTAs per SM
static void ste_product(bool ta, int64_t Mg, int64_t Ng, int64_t Kg, const float* A, int64_t lda,
                        const int8_t* B, int64_t ldb, const float* sB, float* C, int64_t ldc, const float* R,
                        const float* clip, float* workspace, int64_t workspace_elems, cudaStream_t st) {
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = ((Ng + ste::BN - 1) / ste::BN) * ((Mg + ste::BM - 1) / ste::BM);
    // (a conv's weight gradient sums over all N*Ho*Wo positions into a few tiles: up to 128 slices)
    int64_t S = std::min<int64_t>({(2 * (int64_t)sms + tiles - 1) / tiles, 128, std::max<int64_t>(1, Kg / 64)});
    S = workspace ? std::min<int64_t>(S, workspace_elems / std::max<int64_t>(1, Mg * ldc)) : 1;
    if (S < 2) S = 1;
    const int64_t kc = ((Kg + S - 1) / S + ste::BK - 1) / ste::BK * ste::BK;
    S = (Kg + kc - 1) / kc;
    dim3 grid((unsigned)((Ng + ste::BN - 1) / ste::BN), (unsigned)((Mg + ste::BM - 1) / ste::BM), (unsigned)S);
    float* out = S > 1 ? workspace : C;
    if (ta) ste_gemm_kernel<true><<<grid, ste::NT, 0, st>>>(Mg, Ng, Kg, A, lda, B, ldb, sB, out, ldc, R, ldc, clip, kc);
    else ste_gemm_kernel<false><<<grid, ste::NT, 0, st>>>(Mg, Ng, Kg, A, lda, B, ldb, sB, out, ldc, R, ldc, clip, kc);
    if (S > 1)
        ste_reduce_kernel<<<(unsigned)std::min<int64_t>((Mg * ldc + 255) / 256, 8 * sms), 256, 0, st>>>(
            (int)S, Mg * ldc, Ng, workspace, C, R, clip);
}

// gb = column sums of gy [M][N]: two deterministic passes through the workspace when M is large
static void ste_colsum(int64_t M, int64_t N, const float* gy, float* gb, float* workspace, int64_t workspace_elems,
                       cudaStream_t st) {
    if (M >= 4096 && workspace && workspace_elems >= COLSUM_RB * N) {
        ste_colsum_part_kernel<<<dim3((unsigned)((N + 31) / 32), COLSUM_RB), 256, 0, st>>>(M, N, gy, N, workspace);
        ste_colsum_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(COLSUM_RB, N, workspace, N, gb);
    } else {
        ste_colsum_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(M, N, gy, N, gb);
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
}  // namespace axq

extern "C" axq_status axq_ste_linear_backward(int64_t M, int64_t N, int64_t K, const float* gy,
                                              const int8_t* qa, const float* d_scale_a, const float* x,
                                              const float* d_clip_a, const int8_t* qw,
                                              const float* d_scale_w, const float* w,
                                              const float* d_clip_w, float* gx, float* gw, float* gb,
                                              float* workspace, int64_t workspace_elems, void* stream) {
    using namespace axq;
    if (M < 0 || N < 0 || K < 0) return AXQ_ERR_INVALID;
    if (M == 0 || N == 0) {   // empty sums: every gradient that exists is zero
        cudaStream_t st = (cudaStream_t)stream;
        cudaError_t e = cudaSuccess;
        if (gx && M * K > 0) e = cudaMemsetAsync(gx, 0, M * K * sizeof(float), st);
        if (e == cudaSuccess && gw && N * K > 0) e = cudaMemsetAsync(gw, 0, N * K * sizeof(float), st);
        if (e == cudaSuccess && gb && N > 0) e = cudaMemsetAsync(gb, 0, N * sizeof(float), st);
        return e == cudaSuccess ? AXQ_OK : cuda_fail_ext((int)e);
    }
    if (!gy) return AXQ_ERR_INVALID;
    if (gx && (!qw || !d_scale_w || (x && !d_clip_a))) return AXQ_ERR_INVALID;
    if (gw && (!qa || !d_scale_a || (w && !d_clip_w))) return AXQ_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    if (gx && K > 0) ste_product(false, M, K, N, gy, N, qw, K, d_scale_w, gx, K, x, d_clip_a, workspace, workspace_elems, st);
    if (gw && K > 0) ste_product(true, N, K, M, gy, N, qa, K, d_scale_a, gw, K, w, d_clip_w, workspace, workspace_elems, st);
    if (gb) ste_colsum(M, N, gy, gb, workspace, workspace_elems, st);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? AXQ_OK : cuda_fail_ext((int)e);
}

// NEXT-4 for convolution (groups = 1, dilation 1): the STE backward through the explicit im2col
// of the forward's codes (the conv is the GEMM of its im2col matrix), see include/axq.h.
extern "C" axq_status axq_ste_conv2d_backward(const axq_conv_desc* d, const float* gy, const int8_t* qx,
                                              const float* d_scale_a, const float* x, const float* d_clip_a,
                                              const int8_t* qw, const float* d_scale_w, const float* w,
                                              const float* d_clip_w, float* gx, float* gw, float* gb,
                                              int8_t* cols, int64_t ldcols, float* gcols, float* workspace,
                                              int64_t workspace_elems, void* stream) {
    using namespace axq;
    if (!d || d->groups != 1 || d->dil_h != 1 || d->dil_w != 1 || (d->c_valid && d->c_valid != d->C) ||
        d->N < 0 || d->H <= 0 || d->W <= 0 || d->C <= 0 || d->K <= 0 || d->R <= 0 || d->S <= 0 ||
        d->stride_h <= 0 || d->stride_w <= 0 || d->pad_h < 0 || d->pad_w < 0)
        return AXQ_ERR_INVALID;
    const int64_t Ho = (d->H + 2 * d->pad_h - d->R) / d->stride_h + 1, Wo = (d->W + 2 * d->pad_w - d->S) / d->stride_w + 1;
    if (Ho <= 0 || Wo <= 0) return AXQ_ERR_INVALID;
    const int64_t M = d->N * Ho * Wo, Kc = d->R * d->S * d->C, No = d->K;
    if (M >= ((int64_t)1 << 31) || d->N * d->H * d->W * d->C >= ((int64_t)1 << 40)) return AXQ_ERR_INVALID;
    if (!gy && M > 0) return AXQ_ERR_INVALID;
    if (gw && (!qx || !d_scale_a || !cols || ldcols < Kc || (ldcols & 15) || (w && !d_clip_w))) return AXQ_ERR_INVALID;
    if (gx && (!qw || !d_scale_w || !gcols || (x && !d_clip_a))) return AXQ_ERR_INVALID;
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
        ste_product(true, No, Kc, M, gy, No, cols, ldcols, d_scale_a, gw, Kc, w, d_clip_w, workspace,
                    workspace_elems, st);
    }
    if (gx) {   // gcols = gy . fq(W) [M][(r, s, c)], then the adjoint of im2col, masked
        ste_product(false, M, Kc, No, gy, No, qw, Kc, d_scale_w, gcols, Kc, nullptr, nullptr, workspace,
                    workspace_elems, st);
        const int64_t total = d->N * d->H * d->W * d->C;
        int sms = 148, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        ste_col2im_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 16 * sms), 256, 0, st>>>(
            total, (int)d->H, (int)d->W, (int)d->C, (int)d->R, (int)d->S, (int)d->stride_h, (int)d->stride_w,
            (int)d->pad_h, (int)d->pad_w, (int)Ho, (int)Wo, gcols, Kc, x, d_clip_a, gx);
    }
    if (gb) ste_colsum(M, No, gy, gb, workspace, workspace_elems, st);
    e = cudaGetLastError();
    return e == cudaSuccess ? AXQ_OK : cuda_fail_ext((int)e);
}

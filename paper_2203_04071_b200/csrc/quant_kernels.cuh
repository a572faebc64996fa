// quant_kernels.cuh -- amax / scale / quantize / dequantize kernels (sm_100a).
//
// The quantizer is the paper's affine map "real_value = A x quantized_value + B" with
// B = 0 (§III.A) and a per-tensor max-calibrated scale (BASELINE.json
// north_star; A5/A6).  Every fp32 step is pinned with explicit round-to-nearest
// intrinsics so that the integer codes are bit-identical to the CPU oracle (A1, A3, A14):
//   scale      s = __fdiv_rn(amax, qmax)                (amax == 0 -> 1, A4)
//   quantize   q = __float2int_rn(clamp(__fdiv_rn(x, s)))  (half-to-even, A1)
//   dequant    y = __fadd_rn(__fmul_rn(__int2float_rn(acc), __fmul_rn(sa, sw)), bias)
// All of these are HBM-bound streaming kernels; grids are sized in multiples of the SM
// count and use 16-byte vector accesses where the layout allows.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "epilogue.cuh"

namespace axq {

__device__ __forceinline__ float qmax_of(int bits) { return (float)((1 << (bits - 1)) - 1); }

__device__ __forceinline__ int8_t quantize_one(float x, float s, float qmax) {
    float t = div_rn_nz(x, s);
    t = fminf(fmaxf(t, -qmax), qmax);
    return (int8_t)__float2int_rn(t);
}

__device__ __forceinline__ float dequant_one(int32_t acc, float sc, float b) {
    return __fadd_rn(__fmul_rn(__int2float_rn(acc), sc), b);
}

// ---- amax: max |x| (exact).  |x| >= 0 so the IEEE bit pattern orders like an unsigned int,
// which lets one atomicMax per block combine block maxima. ----
__global__ void amax_kernel(const float* __restrict__ x, int64_t n, unsigned int* out) {
    float m = 0.f;
    int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    bool vec = ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    int64_t n4 = vec ? n / 4 : 0;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int64_t i = tid; i < n4; i += stride) {
        float4 v = __ldcs(x4 + i);
        m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    for (int64_t i = n4 * 4 + tid; i < n; i += stride) m = fmaxf(m, fabsf(x[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ float wm[32];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) wm[wid] = m;
    __syncthreads();
    if (wid == 0) {
        m = lane < (int)(blockDim.x >> 5) ? wm[lane] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) atomicMax(out, __float_as_uint(m));
    }
}

__global__ void scale_kernel(const float* d_amax, int bits, float* d_scale) {
    float a = *d_amax;
    *d_scale = (a == 0.f) ? 1.0f : __fdiv_rn(a, qmax_of(bits));
}

// ---- quantize, layout preserving ----
__global__ void quantize_kernel(const float* __restrict__ x, int64_t n,
                                const float* __restrict__ d_scale, int bits,
                                int8_t* __restrict__ q) {
    const float s = *d_scale, qm = qmax_of(bits);
    int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    bool vec = ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
               ((reinterpret_cast<uintptr_t>(q) & 3) == 0);
    int64_t n4 = vec ? n / 4 : 0;
    for (int64_t i = tid; i < n4; i += stride) {
        float4 v = __ldcs(reinterpret_cast<const float4*>(x) + i);
        uint32_t w = (uint32_t)(uint8_t)quantize_one(v.x, s, qm) |
                     ((uint32_t)(uint8_t)quantize_one(v.y, s, qm) << 8) |
                     ((uint32_t)(uint8_t)quantize_one(v.z, s, qm) << 16) |
                     ((uint32_t)(uint8_t)quantize_one(v.w, s, qm) << 24);
        reinterpret_cast<uint32_t*>(q)[i] = w;
    }
    for (int64_t i = n4 * 4 + tid; i < n; i += stride) q[i] = quantize_one(x[i], s, qm);
}

// ---- quantize NCHW fp32 -> NHWC int8 [N][HW][Cq] (channels >= C written as 0).
// Tiled transpose: a 256-thread block owns (image, 64 hw positions, 64 channels); reads are
// float4 rows along hw, the int8 tile is transposed in shared memory and written as 32-bit
// words along c. ----
__global__ void __launch_bounds__(256)
quantize_nchw_to_nhwc_kernel(const float* __restrict__ x, int64_t C, int64_t HW, int64_t Cq,
                             const float* __restrict__ d_scale, int bits, int8_t* __restrict__ q) {
    __shared__ __align__(16) uint8_t tile[64][68];
    const float s = *d_scale, qm = qmax_of(bits);
    const int64_t img = blockIdx.z;
    const int64_t hw0 = (int64_t)blockIdx.x * 64, c0 = (int64_t)blockIdx.y * 64;
    const int tid = threadIdx.x;
    const float* xi = x + img * C * HW;
    const bool vec = ((HW & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
#pragma unroll
    for (int it = 0; it < 4; ++it) {
        const int idx = tid + 256 * it;
        const int cl = idx >> 4, h4 = (idx & 15) * 4;
        const int64_t c = c0 + cl, hw = hw0 + h4;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (c < C) {
            if (vec && hw + 3 < HW) {
                float4 t = __ldcs(reinterpret_cast<const float4*>(xi + c * HW + hw));
                v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
            } else {
                for (int j = 0; j < 4; ++j)
                    if (hw + j < HW) v[j] = xi[c * HW + hw + j];
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            tile[h4 + j][cl] = (uint8_t)((c < C) ? quantize_one(v[j], s, qm) : 0);
    }
    __syncthreads();
    int8_t* qi = q + img * HW * Cq;
    const bool wvec = ((Cq & 3) == 0) && ((reinterpret_cast<uintptr_t>(q) & 3) == 0);
#pragma unroll
    for (int it = 0; it < 4; ++it) {
        const int idx = tid + 256 * it;
        const int hl = idx >> 4, cw = (idx & 15) * 4;
        const int64_t hw = hw0 + hl, c = c0 + cw;
        if (hw >= HW || c >= Cq) continue;
        const uint32_t word = *reinterpret_cast<const uint32_t*>(&tile[hl][cw]);
        if (wvec && c + 3 < Cq) {
            *reinterpret_cast<uint32_t*>(qi + hw * Cq + c) = word;
        } else {
            for (int j = 0; j < 4; ++j)
                if (c + j < Cq) qi[hw * Cq + c + j] = (int8_t)((word >> (8 * j)) & 0xff);
        }
    }
}

// C <= 4 into Cq = 4 (the network input, C = 3 padded), N * HW < 2^31: one pixel per thread,
// 32-bit indices, requantize through the reciprocal with the exact fallback (epi_quant_r, the
// same integer as the IEEE division of A3)
__global__ void quantize_nchw_to_nhwc_c4_kernel(const float* __restrict__ x, int C, int HW, int total,
                                                const float* __restrict__ d_scale, int bits,
                                                int8_t* __restrict__ q) {
    const float s = *d_scale, qm = qmax_of(bits), r = __frcp_rn(s);
    const int gs = gridDim.x * blockDim.x;
    // 4 pixels per thread per iteration, all loads issued before any is used (memory-level
    // parallelism: one pixel at a time left the kernel latency-bound)
    for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += 4 * gs) {
        float v[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * gs;
            const int img = i / HW, hw = i - img * HW;
            const float* xp = x + (int64_t)img * C * HW + hw;
#pragma unroll
            for (int c = 0; c < 4; ++c) v[u][c] = (i < total && c < C) ? __ldcs(xp + c * HW) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * gs;
            if (i >= total) break;
            uint32_t w = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (c < C) w |= (uint32_t)(uint8_t)epi_quant_r(v[u][c], s, r, qm) << (8 * c);
            reinterpret_cast<uint32_t*>(q)[i] = w;
        }
    }
}

// Few channels (the network input, C = 3 padded to Cq = 4): one pixel per thread.
__global__ void quantize_nchw_to_nhwc_small_kernel(const float* __restrict__ x, int64_t N,
                                                   int64_t C, int64_t HW, int64_t Cq,
                                                   const float* __restrict__ d_scale, int bits,
                                                   int8_t* __restrict__ q) {
    const float s = *d_scale, qm = qmax_of(bits);
    const int64_t total = N * HW;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += gs) {
        const int64_t img = i / HW, hw = i - img * HW;
        const float* xp = x + img * C * HW + hw;
        int8_t* qp = q + i * Cq;
        if (Cq == 4 && (reinterpret_cast<uintptr_t>(q) & 3) == 0) {
            uint32_t w = 0;
            for (int c = 0; c < C && c < 4; ++c)
                w |= (uint32_t)(uint8_t)quantize_one(__ldcs(xp + c * HW), s, qm) << (8 * c);
            *reinterpret_cast<uint32_t*>(qp) = w;
        } else {
            for (int64_t c = 0; c < Cq; ++c)
                qp[c] = c < C ? quantize_one(__ldcs(xp + c * HW), s, qm) : (int8_t)0;
        }
    }
}

// ---- dequantize [M][ldacc] int32 -> [M][ldy] fp32 with bias[n] ----
__global__ void dequant_rows_kernel(int64_t M, int64_t N, const int32_t* __restrict__ acc,
                                    int64_t ldacc, const float* __restrict__ sa,
                                    const float* __restrict__ sw, const float* __restrict__ bias,
                                    float* __restrict__ y, int64_t ldy) {
    const float sc = __fmul_rn(*sa, *sw);
    int64_t total = M * N;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
        int64_t m = i / N, n = i - m * N;
        float b = bias ? bias[n] : 0.f;
        float v = __fmul_rn(__int2float_rn(acc[m * ldacc + n]), sc);
        y[m * ldy + n] = bias ? __fadd_rn(v, b) : v;
    }
}

// ---- dequantize NHWC int32 [N][HW][C] -> NCHW fp32 [N][C][HW] (tiled transpose) ----
__global__ void dequant_nhwc_to_nchw_kernel(const int32_t* __restrict__ acc, int64_t HW,
                                            int64_t C, const float* __restrict__ sa,
                                            const float* __restrict__ sw,
                                            const float* __restrict__ bias,
                                            float* __restrict__ y) {
    __shared__ float tile[32][33];
    const float sc = __fmul_rn(*sa, *sw);
    int64_t img = blockIdx.z;
    int64_t hw0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
    int tx = threadIdx.x, ty = threadIdx.y;
    const int32_t* ai = acc + img * HW * C;
    for (int hh = ty; hh < 32; hh += 8) {
        int64_t hw = hw0 + hh, c = c0 + tx;
        if (c < C && hw < HW) {
            float v = __fmul_rn(__int2float_rn(ai[hw * C + c]), sc);
            tile[hh][tx] = bias ? __fadd_rn(v, bias[c]) : v;
        }
    }
    __syncthreads();
    float* yi = y + img * C * HW;
    for (int cc = ty; cc < 32; cc += 8) {
        int64_t c = c0 + cc, hw = hw0 + tx;
        if (c < C && hw < HW) yi[c * HW + hw] = tile[tx][cc];
    }
}

// ===================== NEXT-1: the paper's quantizer (A30-A32) =====================

// Per-output-channel amax of W [rows][cols] (A31): one block per row (grid-stride over rows).
__global__ void amax_rows_kernel(const float* __restrict__ W, int64_t rows, int64_t cols,
                                 float* __restrict__ amax_r) {
    __shared__ float wm[32];
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const float* w = W + r * cols;
        float m = 0.f;
        for (int64_t i = threadIdx.x; i < cols; i += blockDim.x) m = fmaxf(m, fabsf(w[i]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        if (lane == 0) wm[wid] = m;
        __syncthreads();
        if (wid == 0) {
            m = lane < (int)(blockDim.x >> 5) ? wm[lane] : 0.f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) amax_r[r] = m;
        }
        __syncthreads();
    }
}

// s[i] = amax[i] / qmax, amax == 0 -> 1 (the scalar rule of scale_kernel, per element)
__global__ void scale_vec_kernel(const float* __restrict__ amax, int64_t n, int bits, float* __restrict__ s) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float a = amax[i];
        s[i] = (a == 0.f) ? 1.0f : __fdiv_rn(a, qmax_of(bits));
    }
}

// q[r][c] = quantize(W[r][c], s[r])
__global__ void quantize_rows_kernel(const float* __restrict__ W, int64_t rows, int64_t cols,
                                     const float* __restrict__ s_r, int bits, int8_t* __restrict__ q) {
    const float qm = qmax_of(bits);
    const int64_t n = rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        q[i] = quantize_one(W[i], s_r[i / cols], qm);
}

// Histogram of |x| over [0, amax] (A30): bin = min(trunc(fl(|x| / fl(amax / bins))), bins - 1).
// One shared sub-histogram per warp (ReLU / normal data pile into a few bins: per-warp copies
// keep the shared atomics from serialising across the block), summed into one atomicAdd per
// non-empty bin (counts are integers: exact, order-free).
__global__ void hist_kernel(const float* __restrict__ x, int64_t n, const float* __restrict__ d_amax,
                            int bins, int copies, unsigned int* __restrict__ hist) {
    extern __shared__ unsigned int hs[];
    for (int b = threadIdx.x; b < bins * copies; b += blockDim.x) hs[b] = 0u;
    __syncthreads();
    const float a = *d_amax;
    unsigned int* mine = hs + (size_t)((threadIdx.x >> 5) % copies) * bins;
    if (a > 0.f) {
        const float w = __fdiv_rn(a, (float)bins);
        const int64_t gs = (int64_t)gridDim.x * blockDim.x;
        const int64_t n4 = ((reinterpret_cast<uintptr_t>(x) & 15) == 0) ? n / 4 : 0;
        const float4* x4 = reinterpret_cast<const float4*>(x);
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += gs) {
            const float4 v = __ldcs(x4 + i);
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int b = (int)div_rn_nz(fabsf(vv[j]), w);
                atomicAdd(mine + (b > bins - 1 ? bins - 1 : b), 1u);
            }
        }
        for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += gs) {
            const int b = (int)div_rn_nz(fabsf(x[i]), w);
            atomicAdd(mine + (b > bins - 1 ? bins - 1 : b), 1u);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < bins; b += blockDim.x) {
        unsigned int t = 0;
        for (int c = 0; c < copies; ++c) t += hs[(size_t)c * bins + b];
        if (t) atomicAdd(hist + b, t);
    }
}

// calib_max = fl((i + 1) * w) for the first bin i with cum * p_den >= n * p_num; s = calib_max / qmax
// (0 -> 1).  One block: each thread owns a contiguous run of bins; a block-wide exclusive scan
// of the run totals gives every bin's cumulative count; the first crossing wins (atomicMin).
__global__ void percentile_kernel(const unsigned int* __restrict__ hist, int bins, int64_t n,
                                  const float* __restrict__ d_amax, int64_t p_num, int64_t p_den,
                                  int bits, float* __restrict__ d_calib_max, float* __restrict__ d_scale) {
    __shared__ long long wsum[32];
    __shared__ int first;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
    const int per = (bins + nt - 1) / nt, b0 = tid * per, b1 = min(bins, b0 + per);
    long long run = 0;
    for (int b = b0; b < b1; ++b) run += hist[b];
    // inclusive warp scan, then across warps
    long long inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[wid] = inc;
    if (tid == 0) first = bins - 1;
    __syncthreads();
    if (wid == 0) {
        long long v = lane < (nt >> 5) ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        if (lane < (nt >> 5)) wsum[lane] = v;
    }
    __syncthreads();
    long long cum = inc - run + (wid > 0 ? wsum[wid - 1] : 0);   // count before bin b0
    for (int b = b0; b < b1; ++b) {
        cum += hist[b];
        if (cum * p_den >= n * p_num) {
            atomicMin(&first, b);
            break;
        }
    }
    __syncthreads();
    if (tid != 0) return;
    const float a = *d_amax;
    float cm = 0.f;
    if (a > 0.f && n > 0) cm = __fmul_rn((float)(first + 1), __fdiv_rn(a, (float)bins));
    if (d_calib_max) *d_calib_max = cm;
    if (d_scale) *d_scale = (cm == 0.f) ? 1.0f : __fdiv_rn(cm, qmax_of(bits));
}

}  // namespace axq

// epilogue.cuh -- the dequantize epilogue shared by the LUT kernels and the stand-alone
// epilogue kernel (split-K path).  Pinned fp32 order (A13/A14, A17):
//   v = fl(fl((float)acc) * fl(s_a * s_w));  v = fl(v + bias[n]);  v = fl(v + residual[m][n]);
//   v = relu ? max(v, 0) : v;   y = v;   q = clamp(rint(fl(v / s_out)))
// "real_value = A x quantized_value" with both operands' scales, "+ b"; the
// residual add / ReLU / requantize serve the ResNet-50 driver (BJ configs[3], A16/A17).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace axq {

struct EpiArgs {
    const float* sa;        // device scalar
    const float* sw;        // device scalar
    const float* bias;      // [N] or null
    const float* residual;  // [M][ldr] fp32 or null (row layout only)
    int64_t ldr;
    int relu;
    float* y;               // fp32 output or null
    int64_t ldy;            // row layout stride
    int y_nchw;             // 1: y[img][n][pix] with pix in [0, hw)
    int64_t hw;
    int8_t* q;              // requantized codes [M][ldq] or null
    int64_t ldq;
    const float* s_out;     // device scalar
    int bits_out;
    const float* sw_ch;     // per-output-channel weight scales [N] or null (NEXT-1, A32)
    int64_t nchw_ld;        // NCHW: channels per image (0 -> N; a group's slice: all channels)
};

// The dequantization factor of column n: fl(s_a * s_w) (per tensor, precomputed as sc) or
// fl(s_a * s_w[n]) with per-channel weight scales (A32).
__device__ __forceinline__ float epi_sc(const EpiArgs& e, float sc, int64_t n) {
    return e.sw_ch ? __fmul_rn(*e.sa, e.sw_ch[n]) : sc;
}

__device__ __forceinline__ float epi_value(int32_t acc, int64_t m, int64_t n, float sc,
                                           const EpiArgs& e) {
    float v = __fmul_rn(__int2float_rn(acc), epi_sc(e, sc, n));
    if (e.bias) v = __fadd_rn(v, e.bias[n]);
    if (e.residual) v = __fadd_rn(v, e.residual[m * e.ldr + n]);
    if (e.relu) v = v > 0.f ? v : 0.f;
    return v;
}

// IEEE round-to-nearest x / s (A3) with x == 0 answered without the division: 0 / s = +0
// exactly, and a zero dividend would otherwise send the whole warp down __fdiv_rn's slow
// path (ReLU outputs are half zeros).  Bit-identical to __fdiv_rn(x, s) for every x, s != 0.
__device__ __forceinline__ float div_rn_nz(float x, float s) {
    const float t = __fdiv_rn(x == 0.f ? s : x, s);
    return x == 0.f ? __int_as_float(__float_as_int(x) ^ (__float_as_int(s) & 0x80000000)) : t;
}

__device__ __forceinline__ int8_t epi_quant(float v, float s, float qm) {
    float t = div_rn_nz(v, s);
    t = fminf(fmaxf(t, -qm), qm);
    return (int8_t)__float2int_rn(t);
}

// clamp(rint(fl(v / s))) from a precomputed r = RN(1/s), bit-identical to epi_quant: t = RN(v*r)
// is within 3 ulp of fl(v/s), so when t sits more than 4 ulp away from a rounding boundary
// (k + 1/2) both round to the same integer; near a boundary (rare) or for NaN the IEEE division
// decides.  |t| beyond qm + 3/4 clamps either way.  Saves the per-element division.
__device__ __forceinline__ int8_t epi_quant_r(float v, float s, float r, float qm) {
    const float t = __fmul_rn(v, r);
    const float at = fabsf(t);
    if (at >= qm + 0.75f) return (int8_t)(t > 0.f ? (int)qm : -(int)qm);
    const float ti = rintf(t);
    if (fabsf(t - ti) <= __fsub_rn(0.5f, __fmul_rn(at, 4.76837158e-7f)))   // 4 * 2^-23 relative
        return (int8_t)__float2int_rn(fminf(fmaxf(ti, -qm), qm));          // rint then clamp == clamp then rint
    return epi_quant(v, s, qm);
}

// epi_quant_r for v >= 0 (a ReLU output: +0 or positive, never NaN), bit-identical to
// epi_quant: the same boundary test without the sign cases; returns the code as 0..qm
__device__ __forceinline__ uint32_t epi_quant_r_nn(float v, float s, float r, float qm) {
    const float t = __fmul_rn(v, r);
    const float ti = rintf(t);
    if (t >= qm + 0.75f || fabsf(t - ti) <= __fsub_rn(0.5f, __fmul_rn(t, 4.76837158e-7f)))
        return (uint32_t)__float2int_rn(fminf(ti, qm));
    return (uint32_t)(int)epi_quant(v, s, qm);
}

__device__ __forceinline__ void epi_store(float v, int64_t m, int64_t n, int64_t N,
                                          const EpiArgs& e, float s_out, float qm) {
    if (e.y) {
        if (e.y_nchw) {
            const int64_t img = m / e.hw, pix = m - img * e.hw;
            __stcs(e.y + (img * (e.nchw_ld ? e.nchw_ld : N) + n) * e.hw + pix, v);
        } else {
            e.y[m * e.ldy + n] = v;
        }
    }
    if (e.q) e.q[m * e.ldq + n] = epi_quant(v, s_out, qm);
}

// Stand-alone epilogue over an int32 [M][N] accumulator (split-K path).
// zero_acc: the workspace-accumulator form re-zeroes what it read, so a workspace is left
// zero-filled for the stream-K kernel (lut_p4w.cuh), which relies on that.
static __global__ void epilogue_kernel(int64_t M, int64_t N, const int32_t* __restrict__ acc,
                                int64_t ldacc, const EpiArgs e, int32_t* zero_acc = nullptr) {
    const float sc = __fmul_rn(*e.sa, *e.sw);
    const float s_out = e.q ? *e.s_out : 1.f;
    const float qm = (float)((1 << (e.bits_out > 0 ? e.bits_out - 1 : 7)) - 1);
    const int64_t total = M * N;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t m = i / N, n = i - m * N;
        epi_store(epi_value(acc[m * ldacc + n], m, n, sc, e), m, n, N, e, s_out, qm);
        if (zero_acc) zero_acc[m * ldacc + n] = 0;
    }
}

}  // namespace axq

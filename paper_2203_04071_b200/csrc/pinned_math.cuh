// pinned_math.cuh -- the pinned fp32 transcendentals of the LSTM cell (A18), shared
// by lstm_cell_kernel (glue_kernels.cuh) and the persistent recurrence (lstm_rec.cuh).
#pragma once
#include <cuda_runtime.h>

namespace axq {

// E(x): clamp to [-80, 80]; n = rint(x*log2e); r = (x - n*355/512) - n*fl32(ln2 - 355/512);
// p = degree-7 Taylor polynomial of e^r (Horner, fp32 coefficients 1/k!); E = p * 2^n.
__device__ __forceinline__ float pinned_exp(float x) {
    x = fminf(fmaxf(x, -80.f), 80.f);
    const float n = rintf(__fmul_rn(x, 1.4426950216293335f));
    const float r = __fsub_rn(__fsub_rn(x, __fmul_rn(n, 0.693359375f)),
                              __fmul_rn(n, -0.00021219444170128554f));
    float p = 0.00019841270113829523f;               // 1/7!
    p = __fadd_rn(__fmul_rn(p, r), 0.0013888889225199819f);  // 1/6!
    p = __fadd_rn(__fmul_rn(p, r), 0.008333333767950535f);     // 1/5!
    p = __fadd_rn(__fmul_rn(p, r), 0.0416666679084301f);       // 1/4!
    p = __fadd_rn(__fmul_rn(p, r), 0.1666666716337204f);         // 1/3!
    p = __fadd_rn(__fmul_rn(p, r), 0.5f);                                  // 1/2!
    p = __fadd_rn(__fmul_rn(p, r), 1.0f);                                  // 1/1!
    p = __fadd_rn(__fmul_rn(p, r), 1.0f);                                  // 1/0!
    const float two_n = __int_as_float(((int)n + 127) << 23);              // exact 2^n, n in [-116, 116]
    return __fmul_rn(p, two_n);
}

__device__ __forceinline__ float pinned_sigmoid(float x) {
    return __fdiv_rn(1.0f, __fadd_rn(1.0f, pinned_exp(-x)));
}

__device__ __forceinline__ float pinned_tanh(float x) {
    const float e = pinned_exp(__fmul_rn(-2.0f, fabsf(x)));
    const float t = __fdiv_rn(__fsub_rn(1.0f, e), __fadd_rn(1.0f, e));
    return copysignf(t, x);
}

}  // namespace axq

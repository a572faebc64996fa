// mm_wide.cu -- host side of the wide-ACU LUT-GEMM (wide.cuh).
#include "wide.cuh"

namespace axq {

int launch_wide(const WideArgs& a, int sms, cudaStream_t st) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lut_wide_kernel, wide::NT, 0);
    const int64_t tiles = ((a.M + wide::NT - 1) / wide::NT) * ((a.N + wide::TN - 1) / wide::TN);
    const int64_t resident = (int64_t)(per_sm > 0 ? per_sm : 1) * sms;
    lut_wide_kernel<<<(unsigned)(tiles < resident ? tiles : resident), wide::NT, 0, st>>>(a);
    return (int)cudaGetLastError();
}

int launch_quantize16(const float* x, int64_t n, const float* d_scale, int bits, int16_t* q, int sms,
                      cudaStream_t st) {
    const int64_t blocks = (n + 1023) / 1024;
    quantize16_kernel<<<(unsigned)(blocks < sms * 8 ? blocks : sms * 8), 256, 0, st>>>(x, n, d_scale, bits, q);
    return (int)cudaGetLastError();
}

}  // namespace axq

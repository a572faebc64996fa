// mm_wide.cu -- host side of the wide-ACU LUT-GEMM (wide.cuh).
#include "wide.cuh"
#include "wide_pk.cuh"

namespace axq {

int launch_wide(const WideArgs& a, int sms, cudaStream_t st) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lut_wide_kernel, wide::NT, 0);
    const int64_t tiles = ((a.M + wide::NT - 1) / wide::NT) * ((a.N + wide::TN - 1) / wide::TN);
    const int64_t resident = (int64_t)(per_sm > 0 ? per_sm : 1) * sms;
    lut_wide_kernel<<<(unsigned)(tiles < resident ? tiles : resident), wide::NT, 0, st>>>(a);
    return (int)cudaGetLastError();
}

template <int BITS>
static int launch_widepk_t(const WidePkArgs& a, int sms, cudaStream_t st) {
    using G = wpk::Geo<BITS>;
    static unsigned configured = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 31;
    if (!(configured & (1u << dev))) {
        cudaError_t e = cudaFuncSetAttribute(lut_widepk_kernel<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             G::SMEM_BYTES);
        if (e != cudaSuccess) return (int)e;
        configured |= 1u << dev;
    }
    const int64_t tiles = ((a.M + G::BM - 1) / G::BM) * ((a.N + G::TN - 1) / G::TN);
    lut_widepk_kernel<BITS><<<(unsigned)(tiles < sms ? tiles : sms), wpk::NT, G::SMEM_BYTES, st>>>(a);
    return (int)cudaGetLastError();
}

int launch_widepk(const WidePkArgs& a, int sms, cudaStream_t st) {
    switch (a.bits) {
        case 9: return launch_widepk_t<9>(a, sms, st);
        case 10: return launch_widepk_t<10>(a, sms, st);
        case 11: return launch_widepk_t<11>(a, sms, st);
        case 12: return launch_widepk_t<12>(a, sms, st);
        default: return (int)cudaErrorInvalidValue;
    }
}

// tile columns of the packed wide kernel at bit width b (4 x quads per tile)
int widepk_tn(int bits) { return bits >= 11 ? 4 : (bits == 10 ? 8 : 16); }

int widepk_pack(const int16_t* W, int64_t N, int64_t K, int64_t ldw, int64_t Kp, int bits, const int16_t* e16,
                uint2* tables, int16_t* wts, int sms, cudaStream_t st) {
    const int nq = widepk_tn(bits) / 4;
    const int64_t total = ((N + 4 * nq - 1) / (4 * nq)) * Kp * nq * ((int64_t)1 << bits);
    const int64_t blocks = (total + 255) / 256;
    widepk_pack_kernel<<<(unsigned)(blocks < (int64_t)sms * 16 ? blocks : (int64_t)sms * 16), 256, 0, st>>>(
        W, N, K, ldw, Kp, bits, nq, e16, tables, wts);
    return (int)cudaGetLastError();
}

int launch_quantize16(const float* x, int64_t n, const float* d_scale, int bits, int16_t* q, int sms,
                      cudaStream_t st) {
    const int64_t blocks = (n + 1023) / 1024;
    quantize16_kernel<<<(unsigned)(blocks < sms * 8 ? blocks : sms * 8), 256, 0, st>>>(x, n, d_scale, bits, q);
    return (int)cudaGetLastError();
}

}  // namespace axq

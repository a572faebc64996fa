// mm_p4.cu -- host side of the P4 LUT kernel (lut_p4.cuh): weight packing and launch.
#include "lut_p4.cuh"
#include "mm_launch.h"

namespace axq {

int p4_pack(const int8_t* W, int64_t N, int64_t K, int64_t ldw, int64_t Kp, const int8_t* dtab,
            uint32_t* tables, int8_t* wpk, cudaStream_t st) {
    const int64_t nb = (N + p4::TN - 1) / p4::TN;
    const int64_t t1 = nb * Kp * 4 * 256, t2 = nb * Kp * p4::TN;
    p4_pack_tables_kernel<<<(unsigned)std::min<int64_t>((t1 + 255) / 256, 148 * 16), 256, 0, st>>>(
        W, N, K, ldw, Kp, dtab, tables);
    p4_pack_w_kernel<<<(unsigned)std::min<int64_t>((t2 + 255) / 256, 148 * 16), 256, 0, st>>>(W, N, K, ldw, Kp, wpk);
    return (int)cudaGetLastError();
}

int launch_p4(const P4Args& a, cudaStream_t st) {
    static unsigned configured = 0;
    static int sms[32] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 31;
    if (!(configured & (1u << dev))) {
        cudaError_t e = cudaFuncSetAttribute(lut_p4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             p4::SMEM_BYTES);
        if (e != cudaSuccess) return (int)e;
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        sms[dev] = n > 0 ? n : 148;
        configured |= 1u << dev;
    }
    const int64_t work = ((a.mm.M + p4::BM - 1) / p4::BM) * ((a.mm.N + p4::TN - 1) / p4::TN);
    const unsigned g = (unsigned)std::min<int64_t>(work, sms[dev]);
    lut_p4_kernel<<<g, p4::NT, p4::SMEM_BYTES, st>>>(a);
    return (int)cudaGetLastError();
}

}  // namespace axq

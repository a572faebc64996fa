// mm_gconv.cu -- host side of the grouped / depthwise LUT conv (gconv.cuh).
#include "gconv.cuh"

namespace axq {

template <int REPR>
static int launch_gconv_t(const GConvArgs& a, cudaStream_t st) {
    const int smem = REPR == REPR_I32 ? 0 : a.table_bytes;
    static bool configured[32] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 31;
    if (!configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(lut_gconv_kernel<REPR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             128 * 1024);
        if (e != cudaSuccess) return (int)e;
        configured[dev] = true;
    }
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lut_gconv_kernel<REPR>, 256, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t work = ((a.M + 31) / 32) * ((a.K + 7) / 8);
    const int64_t resident = (int64_t)(per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 148);
    const unsigned g = (unsigned)(work < resident ? work : resident);
    lut_gconv_kernel<REPR><<<g, 256, smem, st>>>(a);
    return (int)cudaGetLastError();
}

template <int REPR, int KR, int KS>
static int launch_dw_t(const GConvArgs& a, cudaStream_t st) {
    const int smem = REPR == REPR_I32 ? 0 : a.table_bytes;
    static bool configured[32] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 31;
    if (!configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(lut_dwconv_kernel<REPR, KR, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             128 * 1024);
        if (e != cudaSuccess) return (int)e;
        configured[dev] = true;
    }
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lut_dwconv_kernel<REPR, KR, KS>, 256, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // total threads a multiple of C/4 (each thread keeps one channel quad), at most resident
    const int64_t C4 = a.C / 4, resident = (int64_t)(per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 148) * 256;
    int64_t threads = (resident / C4) * C4;
    const int64_t need = a.M * C4;
    if (threads > need) threads = ((need + C4 - 1) / C4) * C4;
    int64_t blocks = (threads + 255) / 256;
    // keep nthreads % C4 == 0 with whole blocks: grow the block count until it holds
    while ((blocks * 256) % C4) ++blocks;
    lut_dwconv_kernel<REPR, KR, KS><<<(unsigned)blocks, 256, smem, st>>>(a);
    return (int)cudaGetLastError();
}

template <int REPR>
static int launch_dw_repr(const GConvArgs& a, cudaStream_t st) {
    if (a.R == 3 && a.S == 3) return launch_dw_t<REPR, 3, 3>(a, st);
    if (a.R == 5 && a.S == 5) return launch_dw_t<REPR, 5, 5>(a, st);
    if (a.R == 7 && a.S == 7) return launch_dw_t<REPR, 7, 7>(a, st);
    if (a.R == 1 && a.S == 1) return launch_dw_t<REPR, 1, 1>(a, st);
    return -1;
}

template <bool QR>
static int launch_dw3_t(const GConvArgs& a, cudaStream_t st) {
    static bool configured[32] = {false};
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    dev &= 31;
    if (!configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(lut_dw3_kernel<QR>, cudaFuncAttributeMaxDynamicSharedMemorySize, dw3::SMEM);
        if (e != cudaSuccess) return (int)e;
        configured[dev] = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lut_dw3_kernel<QR>, dw3::NT, dw3::SMEM);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t items = (int64_t)((a.C + dw3::CB - 1) / dw3::CB) * ((a.Wo + 29) / 30) * a.N;
    const int64_t resident = (int64_t)(per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 148);
    lut_dw3_kernel<QR><<<(unsigned)(items < resident ? items : resident), dw3::NT, dw3::SMEM, st>>>(a);
    return (int)cudaGetLastError();
}

static int launch_dw3(const GConvArgs& a, cudaStream_t st) {
    const EpiArgs& e = a.ep;
    const bool qr = !a.C_out && e.q && !e.y && e.relu && !e.residual && (a.C % dw3::CB) == 0 &&
                    ((e.ldq & 15) == 0) && ((reinterpret_cast<uintptr_t>(e.q) & 15) == 0);
    return qr ? launch_dw3_t<true>(a, st) : launch_dw3_t<false>(a, st);
}

int launch_gconv(int repr, const GConvArgs& a, cudaStream_t st) {
    // depthwise 3x3 / stride 1 / pad 1 with a delta8 table: the input-stationary packed kernel
    if (repr == REPR_DELTA8 && a.C == a.G && a.K == a.C && a.R == 3 && a.S == 3 && a.sh == 1 && a.sw == 1 &&
        a.ph == 1 && a.pw == 1 && a.dh == 1 && a.dw == 1 && a.Ho == a.H && a.Wo == a.Wd && a.N < (1 << 30))
        return launch_dw3(a, st);
    const bool dw = a.C == a.G && a.K == a.C && (a.C % 4) == 0 &&
                    (reinterpret_cast<uintptr_t>(a.X) & 3) == 0 &&
                    (!a.C_out || (reinterpret_cast<uintptr_t>(a.C_out) & 15) == 0);
    if (dw) {
        const int rc = repr == REPR_DELTA8 ? launch_dw_repr<REPR_DELTA8>(a, st)
                     : repr == REPR_I16    ? launch_dw_repr<REPR_I16>(a, st)
                                           : launch_dw_repr<REPR_I32>(a, st);
        if (rc != -1) return rc;
    }
    if (repr == REPR_DELTA8) return launch_gconv_t<REPR_DELTA8>(a, st);
    if (repr == REPR_I16) return launch_gconv_t<REPR_I16>(a, st);
    return launch_gconv_t<REPR_I32>(a, st);
}

}  // namespace axq

// mm_lstm.cu -- host side of the persistent LSTM recurrence (lstm_rec.cuh).
#include "lstm_rec.cuh"

namespace axq {

// Return 0, or a cudaError_t code; -1: the shape cannot run co-resident on this device.
int launch_lstm_rec(const LstmRecArgs& a, int sms, cudaStream_t st) {
    const int rg = (a.B + 31) / 32;
    int G = sms < a.H ? sms : a.H;
    const int nu = (a.H + G - 1) / G;
    if (nu * rg > lstmr::NT / 32 || (a.H % 16) != 0) return -1;
    const size_t smem = lstmr::TABLE + (size_t)nu * 4 * a.H + (size_t)a.B * (a.H + lstmr::H_PAD) +
                        (lstmr::NT / 32) * 4 * 32 * 4;
    if (smem > 227 * 1024) return -1;
    static size_t configured[32] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 31;
    if (configured[dev] < smem) {
        cudaError_t e = cudaFuncSetAttribute(lstm_rec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        configured[dev] = smem;
    }
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lstm_rec_kernel, lstmr::NT, smem);
    if (e != cudaSuccess) return (int)e;
    if (per_sm < 1 || G > per_sm * sms) return -1;
    e = cudaMemsetAsync(a.bar, 0, sizeof(unsigned int), st);
    if (e != cudaSuccess) return (int)e;
    LstmRecArgs args = a;
    void* params[] = {&args};
    e = cudaLaunchCooperativeKernel((const void*)lstm_rec_kernel, dim3(G), dim3(lstmr::NT), params, smem, st);
    return (int)e;
}

}  // namespace axq

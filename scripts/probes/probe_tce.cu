// probe_tce.cu -- microbenchmark for the TCE design question: cycles per tcgen05.mma kind::i8
// (M = 128, K = 32) at N = 16 / 32 / 64 / 256 with A from TMEM or shared memory, back to back from
// one thread, and the latency of tcgen05.st.32x32b.x16 + wait::st.  Not part of the library.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2203_04071_b200/csrc/async_copy.cuh"
#include "../../paper_2203_04071_b200/csrc/tc_common.cuh"
using namespace axq;

template <int N, bool ATMEM>
__global__ void probe(long long* out, int reps) {
    __shared__ __align__(1024) uint8_t sm[40960];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    for (int i = tid; i < 40960 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    if (tid == 0) { mbar_init(smem_u32(&bar), blockDim.x / 32); asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    // STTM latency: warp 0 stores 16 columns and waits, 64 times
    if (tid < 32) {
        uint32_t v[16];
        for (int j = 0; j < 16; ++j) v[j] = tid + j;
        long long t0 = clock64();
        for (int r = 0; r < 64; ++r) { v[0] += r; tmem_st16(tmem + 256 + (r & 7) * 16, v); tmem_wait_st(); }
        long long t1 = clock64();
        if (tid == 0) out[1] = (t1 - t0) / 64;
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const int nw = blockDim.x / 32;   // issuing warps: lane 0 of each
    if ((tid & 31) == 0) {
        constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t bdesc = umma_desc_kmajor(smem_u32(sm) + 32768, 256u, 128u);
        const uint64_t adesc = umma_desc_kmajor(smem_u32(sm), 256u, 128u);
        const uint32_t dcol = (uint32_t)((tid >> 5) * 32);
        long long t0 = clock64();
        for (int r = 0; r < reps; r += 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (ATMEM) umma_i8_ts(tmem + dcol, tmem + 256 + u * 8, bdesc, IDESC, 1u);
                else umma_i8(tmem + dcol, adesc, bdesc, IDESC, 1u);
            }
        }
        long long t1 = clock64();
        umma_commit(smem_u32(&bar));
        if (tid == 0) {
            mbar_wait(smem_u32(&bar), 0);
            long long t2 = clock64();
            out[0] = t2 - t0;
            out[2] = t1 - t0;
        }
    }
    (void)nw;
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
}

template <int N, bool AT>
void run(long long* d, int reps, int warps = 4) {
    probe<N, AT><<<1, 32 * warps>>>(d, reps);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[3];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("N=%3d A=%s reps=%d: %.1f cyc/MMA total, %.1f cyc/MMA issue, sttm+wait %lld cyc  (%s)\n", N,
           AT ? "tmem" : "smem", reps, (double)h[0] / reps, (double)h[2] / reps, h[1], cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    for (int w : {1, 2, 4, 8}) {
        printf("issuing warps %d (reps per warp; total time = all warps' MMAs)\n", w);
        run<16, true>(d, 1024, w); run<16, false>(d, 1024, w); run<64, true>(d, 1024, w);
    }
    return 0;
}

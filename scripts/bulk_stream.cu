// Micro-benchmark: HBM -> shared-memory streaming rate of cp.async.bulk rings (one CTA per SM),
// for choosing the stage size / depth of the packed-table kernels when they are table-stream
// bound (small M).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bs scripts/bulk_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) stream_kernel(const uint8_t* src, int64_t bytes_per_cta, int stage_bytes,
                                                        int stages, int pieces, unsigned long long* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[16];
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const uint8_t* base = src + (int64_t)blockIdx.x * bytes_per_cta;
    const int64_t n_items = bytes_per_cta / stage_bytes;
    unsigned long long acc = 0;
    const int piece = stage_bytes / pieces;
    if (tid == 0) {
        auto issue = [&](int64_t it) {
            const int s = (int)(it % stages);
            const uint32_t b = su32(&bar[s]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(stage_bytes) : "memory");
            for (int p = 0; p < pieces; ++p)
                asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                             ::"r"(su32(sm + (size_t)s * stage_bytes + p * piece)),
                             "l"(base + it * stage_bytes + p * piece), "r"(piece), "r"(b)
                             : "memory");
        };
        for (int64_t it = 0; it < stages && it < n_items; ++it) issue(it);
        for (int64_t it = 0; it < n_items; ++it) {
            const int s = (int)(it % stages);
            const uint32_t b = su32(&bar[s]);
            const uint32_t ph = (uint32_t)((it / stages) & 1);
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                             : "=r"(done) : "r"(b), "r"(ph) : "memory");
            acc += sm[(size_t)s * stage_bytes + (it & 1023)];
            if (it + stages < n_items) issue(it + stages);
        }
        sink[blockIdx.x] = acc;
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t per_cta = 2 << 20;   // 2 MiB per CTA: ~296 MiB total (> L2)
    uint8_t* src;
    unsigned long long* sink;
    cudaMalloc(&src, per_cta * sms);
    cudaMemset(src, 1, per_cta * sms);
    cudaMalloc(&sink, sms * 8);
    uint8_t* flush;
    cudaMalloc(&flush, 256 << 20);
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int cfg[][3] = {{65536, 2, 1}, {65536, 2, 4}, {65536, 3, 1}, {32768, 4, 1}, {32768, 6, 1},
                          {16384, 8, 1}, {16384, 12, 1}, {8192, 16, 1}, {49152, 4, 1}, {65536, 3, 8}};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (auto& c : cfg) {
        const int sb = c[0], st = c[1], pc = c[2];
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemsetAsync(flush, rep, 256 << 20);
            cudaEventRecord(e0);
            stream_kernel<<<sms, 128, (size_t)sb * st>>>(src, per_cta, sb, st, pc, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        printf("stage %6d B x %2d stages, %d piece(s): %8.1f us  %7.0f GB/s  %s\n", sb, st, pc, best * 1e3,
               (double)per_cta * sms / (best * 1e-3) / 1e9, cudaGetErrorString(err));
    }
    return 0;
}

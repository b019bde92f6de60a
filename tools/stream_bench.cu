// stream_bench.cu — development microbenchmark: HBM streaming rate of the
// load mechanisms K2 can use on sm_100a (cp.async.bulk rings vs LDG.128).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_bench tools/stream_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(128, 1) bulk_ring(const uint8_t* __restrict__ src, size_t per_cta, int chunk, int depth,
                                                    int hint, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + depth * chunk);
    if (threadIdx.x == 0) {
        for (int i = 0; i < depth; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint8_t* base = src + blockIdx.x * per_cta;
    const int n = static_cast<int>(per_cta / chunk);
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    auto issue = [&](int i) {
        const int s = i % depth;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(chunk) : "memory");
        if (hint)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                             smem_u32(sm + s * chunk)),
                         "l"(base + size_t(i) * chunk), "r"(chunk), "r"(smem_u32(&bar[s])), "l"(pol)
                         : "memory");
        else
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             smem_u32(sm + s * chunk)),
                         "l"(base + size_t(i) * chunk), "r"(chunk), "r"(smem_u32(&bar[s]))
                         : "memory");
    };
    for (int i = 0; i < depth && i < n; ++i) issue(i);
    unsigned long long acc = 0;
    for (int i = 0; i < n; ++i) {
        const int s = i % depth;
        const uint32_t ph = (i / depth) & 1;
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(ok)
                         : "r"(smem_u32(&bar[s])), "r"(ph)
                         : "memory");
        acc += sm[s * chunk];
        if (i + depth < n) issue(i + depth);
    }
    sink[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(512) ldg_stream(const uint4* __restrict__ src, size_t n16, unsigned long long* sink) {
    uint32_t x = 0;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
#pragma unroll 8
    for (; i < n16; i += stride) {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
        x ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (x == 0x12345678) sink[0] = x;
}

int main() {
    const size_t bytes = size_t(1) << 30;  // 1 GiB > L2
    uint8_t* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    unsigned long long* sink;
    cudaMalloc(&sink, 4096 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int sms = 148;
    for (int total_mb : {16, 64, 1024}) {
        const size_t tot = size_t(total_mb) << 20;
        for (int chunk : {4096, 8192, 16384}) {
            for (int depth : {4, 8, 12, 24}) {
                if (size_t(chunk) * depth > 200 * 1024) continue;
                for (int hint : {0, 1}) {
                    const size_t per = (tot / sms) / chunk * chunk;
                    const int smem = chunk * depth + 1024;
                    cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                    for (int w = 0; w < 2; ++w) bulk_ring<<<sms, 128, smem>>>(buf, per, chunk, depth, hint, sink);
                    cudaEventRecord(e0);
                    const int reps = 10;
                    for (int r = 0; r < reps; ++r) bulk_ring<<<sms, 128, smem>>>(buf + (r % 2) * (512u << 20) * (total_mb < 512), per, chunk, depth, hint, sink);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    const double us = ms * 1e3 / reps;
                    printf("bulk total=%4dMB chunk=%5d depth=%2d hint=%d: %8.2f us  %7.0f GB/s\n", total_mb, chunk, depth, hint,
                           us, per * sms / us / 1e3);
                }
            }
        }
        const size_t n16 = tot / 16;
        for (int blocks : {148, 296, 592}) {
            ldg_stream<<<blocks, 512>>>(reinterpret_cast<const uint4*>(buf), n16, sink);
            cudaEventRecord(e0);
            for (int r = 0; r < 10; ++r) ldg_stream<<<blocks, 512>>>(reinterpret_cast<const uint4*>(buf + (r % 2) * (512u << 20) * (total_mb < 512)), n16, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double us = ms * 1e3 / 10;
            printf("ldg  total=%4dMB blocks=%d: %8.2f us  %7.0f GB/s\n", total_mb, blocks, us, tot / us / 1e3);
        }
    }
    // per-CTA streaming cap: few CTAs, 2 MB each
    for (int ctas : {1, 8, 32, 74, 113, 148}) {
        for (int chunk : {16384, 32768}) {
            const int depth = chunk == 16384 ? 12 : 6;
            const size_t per = size_t(2) << 20;
            const int smem = chunk * depth + 1024;
            cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            bulk_ring<<<ctas, 128, smem>>>(buf, per, chunk, depth, 1, sink);
            cudaEventRecord(e0);
            for (int r = 0; r < 10; ++r) bulk_ring<<<ctas, 128, smem>>>(buf + (r % 2) * (400u << 20), per, chunk, depth, 1, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double us = ms * 1e3 / 10;
            printf("percta ctas=%3d chunk=%5d depth=%2d: %8.2f us  %7.1f GB/s per CTA  %7.0f GB/s total\n", ctas, chunk, depth, us,
                   per / us / 1e3, per * ctas / us / 1e3);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}

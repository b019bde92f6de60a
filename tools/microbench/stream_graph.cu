// stream_graph.cu — development microbenchmark: how fast can back-to-back
// launches of a pure bulk-copy streaming kernel (same smem/threads shape as K2)
// go inside a CUDA graph, with and without PDL? Per-launch bytes = `mb` MB.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_graph tools/stream_graph.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(512, 1) bulk_ring(const uint8_t* __restrict__ src, size_t per_cta, int chunk, int depth,
                                                    unsigned long long* sink, int hold) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + depth * chunk);
    if (threadIdx.x == 0) {
        for (int i = 0; i < depth; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x != 0) {
        if (hold) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            __syncthreads();
        }
        return;
    }
    const uint8_t* base = src + blockIdx.x * per_cta;
    const int n = static_cast<int>(per_cta / chunk);
    auto issue = [&](int i) {
        const int s = i % depth;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(sm + s * chunk)),
                     "l"(base + size_t(i) * chunk), "r"(chunk), "r"(smem_u32(&bar[s]))
                     : "memory");
    };
    for (int i = 0; i < depth && i < n; ++i) issue(i);
    asm volatile("griddepcontrol.wait;" ::: "memory");
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
    if (hold) __syncthreads();
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    const size_t total = size_t(2) << 30;
    uint8_t* buf;
    cudaMalloc(&buf, total);
    cudaMemset(buf, 1, total);
    unsigned long long* sink;
    cudaMalloc(&sink, 4096 * 8);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mb : {10, 35, 70}) {
        for (int hold : {0}) {
          for (int big : {0, 1}) {
            const int ctas = 148, pdl = 1;
            {
              for (int cd : {0, 1, 2}) {
                const int chunk = cd == 0 ? 32768 : cd == 1 ? 16384 : 8192, depth = cd == 0 ? 6 : cd == 1 ? 12 : 24;
                const size_t per = std::max<size_t>(chunk, (size_t(mb) << 20) / ctas / chunk * chunk);
                const int smem = big ? 232448 : chunk * depth + 1024 + 512;
                cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                const int nl = 20;
                const size_t stride = per * ctas;
                auto launch = [&](int i) {
                    cudaLaunchConfig_t cfg{};
                    cfg.gridDim = dim3(ctas);
                    cfg.blockDim = dim3(512);
                    cfg.dynamicSmemBytes = smem;
                    cfg.stream = st;
                    cudaLaunchAttribute a[1];
                    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    a[0].val.programmaticStreamSerializationAllowed = 1;
                    cfg.attrs = a;
                    cfg.numAttrs = pdl;
                    const uint8_t* src = buf + (size_t(i) * stride) % (total - stride);
                    cudaLaunchKernelEx(&cfg, bulk_ring, src, per, chunk, depth, sink, hold);
                };
                cudaGraph_t g;
                cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
                for (int i = 0; i < nl; ++i) launch(i);
                cudaStreamEndCapture(st, &g);
                cudaGraphExec_t ge;
                cudaGraphInstantiate(&ge, g, 0);
                cudaGraphLaunch(ge, st);
                cudaStreamSynchronize(st);
                cudaEventRecord(e0, st);
                cudaGraphLaunch(ge, st);
                cudaEventRecord(e1, st);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double us = ms * 1e3 / nl;
                printf("graph stream %4d MB/launch chunk=%5d depth=%2d hold=%d smem=%6d: %7.2f us/launch  %6.0f GB/s\n", mb, chunk, depth, hold, smem, us,
                       double(per * ctas) / us / 1e3);
                cudaGraphExecDestroy(ge);
                cudaGraphDestroy(g);
              }
            }
          }
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}

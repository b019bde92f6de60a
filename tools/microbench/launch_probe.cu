// launch_probe.cu — development microbenchmark for the decode launch shape:
// back-to-back launches (CUDA graph, PDL) of a pure bulk-copy streaming kernel
// (148 CTAs x 512 threads, 227 KB smem, 32 KB chunks x 6) that
//  (a) takes its arguments in a ~1 KB __grid_constant__ struct and reads `chain`
//      dependent words from different 128 B lines before the first copy, and
//  (b) runs in thread-block clusters of `cl` CTAs (1 / 2 / 4), optionally with a
//      DSMEM reduction at the end (every CTA st.async's 8 KB into rank 0).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/launch_probe tools/microbench/launch_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <algorithm>

struct Big {
    int w[256];
    const uint8_t* src;
    size_t per;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(512, 1) probe(const __grid_constant__ Big p, int chain, int red, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    constexpr int chunk = 32768, depth = 6;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + depth * chunk);
    uint64_t* rbar = bar + depth;
    if (threadIdx.x == 0) {
        for (int i = 0; i < depth; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(rbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (red) asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    unsigned crank = 0, csize = 1;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
    if (threadIdx.x == 0) {
        int idx = 0;
        for (int c = 0; c < chain; ++c) idx = p.w[(idx + 32 * (c + 1)) & 255];  // dependent loads, one line each
        const uint8_t* base = p.src + blockIdx.x * p.per + idx;
        const int n = static_cast<int>(p.per / chunk);
        auto issue = [&](int i) {
            const int s = i % depth;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(chunk) : "memory");
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
                asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}"
                             : "=r"(ok) : "r"(smem_u32(&bar[s])), "r"(ph) : "memory");
            acc += sm[s * chunk];
            if (i + depth < n) issue(i + depth);
        }
        sink[blockIdx.x] = acc;
    }
    __syncthreads();
    if (red && csize > 1) {
        // every non-zero rank pushes 8 KB (512 threads x 16 B) into rank 0's stage 0 slot `crank`
        if (crank == 0 && threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(rbar)), "r"((csize - 1) * 8192) : "memory");
        asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (crank != 0) {
            uint32_t dst = smem_u32(sm + crank * 8192 + threadIdx.x * 16), rb = smem_u32(rbar), rd, rrb;
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rd) : "r"(dst));
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rrb) : "r"(rb));
            uint32_t v = threadIdx.x;
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %1, %1, %1}, [%2];" ::"r"(rd), "r"(v), "r"(rrb) : "memory");
        } else {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0; selp.u32 %0,1,0,q;}"
                             : "=r"(ok) : "r"(smem_u32(rbar)) : "memory");
            if (threadIdx.x == 0) sink[1024 + blockIdx.x] = sm[8192];
        }
        asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    const size_t total = size_t(2) << 30;
    uint8_t* buf;
    cudaMalloc(&buf, total);
    cudaMemset(buf, 0, total);
    unsigned long long* sink;
    cudaMalloc(&sink, 4096 * 8);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int smem = 232448;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cl : {2, 4, 8}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(148 / cl * cl);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cl;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        int n = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe, &cfg);
        printf("cluster %d: max active clusters %d (%d CTAs) %s\n", cl, n, n * cl, cudaGetErrorString(e));
    }
    for (int mb : {10, 35}) {
        for (int ctas : {33, 50, 66, 74, 100, 148}) {
            const size_t per = std::max<size_t>(32768, (size_t(mb) << 20) / ctas / 32768 * 32768);
            Big p{};
            p.per = per;
            const int nl = 20;
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
                cfg.numAttrs = 1;
                p.src = buf + (size_t(i) * per * ctas) % (total - per * ctas);
                return cudaLaunchKernelEx(&cfg, probe, p, 0, 0, sink);
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
            for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, st);
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double us = ms * 1e3 / (nl * 5);
            printf("%3d MB on %3d CTAs (%4zu KB each): %6.2f us/launch %6.0f GB/s  %5.0f GB/s per SM\n", mb, ctas, per >> 10, us,
                   double(per * ctas) / us / 1e3, double(per) / us / 1e3);
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        }
    }
    for (int mb : {10}) {
        for (int chain : {0}) {
            for (int cl : {1, 2, 4}) {
                for (int red : {0, 1}) {
                    if (red && cl == 1) continue;
                    if (cl > 1 && chain != 0) continue;
                    const int ctas = 148 / cl * cl;
                    const size_t per = std::max<size_t>(32768, (size_t(mb) << 20) / ctas / 32768 * 32768);
                    Big p{};
                    for (int i = 0; i < 256; ++i) p.w[i] = 0;
                    p.per = per;
                    const int nl = 20;
                    auto launch = [&](int i) {
                        cudaLaunchConfig_t cfg{};
                        cfg.gridDim = dim3(ctas);
                        cfg.blockDim = dim3(512);
                        cfg.dynamicSmemBytes = smem;
                        cfg.stream = st;
                        cudaLaunchAttribute a[2];
                        a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                        a[0].val.programmaticStreamSerializationAllowed = 1;
                        a[1].id = cudaLaunchAttributeClusterDimension;
                        a[1].val.clusterDim.x = cl;
                        a[1].val.clusterDim.y = 1;
                        a[1].val.clusterDim.z = 1;
                        cfg.attrs = a;
                        cfg.numAttrs = cl > 1 ? 2 : 1;
                        p.src = buf + (size_t(i) * per * ctas) % (total - per * ctas);
                        return cudaLaunchKernelEx(&cfg, probe, p, chain, red, sink);
                    };
                    cudaGraph_t g;
                    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
                    cudaError_t le = cudaSuccess;
                    for (int i = 0; i < nl; ++i) le = launch(i);
                    cudaStreamEndCapture(st, &g);
                    if (le != cudaSuccess) {
                        printf("launch error %s\n", cudaGetErrorString(le));
                        continue;
                    }
                    cudaGraphExec_t ge;
                    cudaGraphInstantiate(&ge, g, 0);
                    cudaGraphLaunch(ge, st);
                    cudaStreamSynchronize(st);
                    cudaEventRecord(e0, st);
                    for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, st);
                    cudaEventRecord(e1, st);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    const double us = ms * 1e3 / (nl * 5);
                    printf("%3d MB chain=%d cluster=%d dsmem_red=%d: %6.2f us/launch %6.0f GB/s\n", mb, chain, cl, red, us,
                           double(per * ctas) / us / 1e3);
                    cudaGraphExecDestroy(ge);
                    cudaGraphDestroy(g);
                }
            }
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}

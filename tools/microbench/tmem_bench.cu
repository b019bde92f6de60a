// TMEM read-throughput probe: W warps (W/4 per lane quarter) repeatedly
// tcgen05.ld 32x32b.xC from their quarter, one wait::ld per batch of B loads.
#include <cstdio>
#include <cstdint>
#include "../paper_2412_14590_b200/csrc/kernels/mq_layout.cuh"
#include "../paper_2412_14590_b200/csrc/kernels/mq_ptx.cuh"
using namespace mq;

__device__ __forceinline__ void ld32(uint32_t ta, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(ta));
}
__device__ __forceinline__ void ld16x2(uint32_t ta, uint32_t (&v)[32]) {
    ptx::tmem_ld16(ta, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
    ptx::tmem_ld16(ta + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
}

template <int MODE>
__global__ void tmem_rd(int iters, unsigned long long* out, uint32_t* sink) {
    __shared__ uint32_t holder;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) ptx::tmem_alloc<512>(&holder);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t base = holder + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * 32);
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t v[32];
        if (MODE == 0) ld32(base + (i & 7) * 64 % 256, v);
        else ld16x2(base + (i & 7) * 64 % 256, v);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 32; ++q) acc += v[q];
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<512>(holder);
}

int main() {
    unsigned long long* d; uint32_t* sink;
    cudaMalloc(&d, 148 * 8); cudaMalloc(&sink, 148 * 1024 * 4);
    const int iters = 4096;
    for (int mode = 0; mode < 2; ++mode)
        for (int warps : {4, 8, 16}) {
            if (mode == 0) tmem_rd<0><<<148, warps * 32>>>(iters, d, sink);
            else tmem_rd<1><<<148, warps * 32>>>(iters, d, sink);
            unsigned long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            const double bytes = double(iters) * warps * 32 * 32 * 4;  // per CTA
            printf("%s warps=%2d: %8llu cycles  %.1f B/cycle/SM\n", mode ? "ld16x2" : "ld32  ", warps, h[0], bytes / h[0]);
        }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}

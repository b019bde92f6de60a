// tcgen05.mma kind::i8 issue/execute rate: M=128, N in {16..256}, K=32 per
// instruction, A from TMEM (ts) or SMEM (ss), B from SMEM; 1 CTA per SM.
#include <cstdio>
#include <cstdint>
#include "../paper_2412_14590_b200/csrc/kernels/mq_layout.cuh"
#include "../paper_2412_14590_b200/csrc/kernels/mq_ptx.cuh"
using namespace mq;
__device__ __forceinline__ bool elect1() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}

template <bool kTs>
__global__ void __launch_bounds__(128) mma_rate(int n_mma, uint32_t N, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t holder;
    __shared__ __align__(8) uint64_t bar;
    uint8_t* base = sm + ((1024 - (ptx::smem_u32(sm) & 1023)) & 1023);
    for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(base)[i] = 0x01010101u * (i & 3);
    ptx::fence_proxy_async_smem();
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
    if (threadIdx.x < 32) ptx::tmem_alloc<512>(&holder);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = holder;
    const uint32_t idesc = idesc_i8(N, true, true);
    const uint32_t a_s = ptx::smem_u32(base), b_s = ptx::smem_u32(base + 16384);
    if (threadIdx.x < 32) {
        const unsigned long long t0 = clock64();
        if (elect1()) {
            for (int i = 0; i < n_mma; ++i) {
                const int k = i & 3;
                if (kTs) ptx::mma_i8_ts(tm, tm + 256 + 8 * k, ptx::umma_desc_sw128(b_s + 32 * k), idesc, i > 0);
                else ptx::mma_i8_ss(tm, ptx::umma_desc_sw128(a_s + 32 * k), ptx::umma_desc_sw128(b_s + 32 * k), idesc, i > 0);
            }
            ptx::tc_commit(&bar);
        }
        __syncwarp();
        const unsigned long long t1 = clock64();
        ptx::mbar_wait(&bar, 0);
        const unsigned long long t2 = clock64();
        if (threadIdx.x == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t0; }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) ptx::tmem_dealloc<512>(tm);
}

int main() {
    unsigned long long* d; cudaMalloc(&d, 148 * 16);
    const int smem = 65536 + 1024;
    cudaFuncSetAttribute(mma_rate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(mma_rate<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int ts = 0; ts < 2; ++ts)
        for (uint32_t N : {16u, 32u, 64u, 128u, 256u}) {
            const int n = 2048;
            for (int rep = 0; rep < 2; ++rep) {
                if (ts) mma_rate<true><<<148, 128, smem>>>(n, N, d);
                else mma_rate<false><<<148, 128, smem>>>(n, N, d);
            }
            unsigned long long h[2];
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            printf("%s N=%3u: issue %.1f cyc/mma, complete %.1f cyc/mma (ideal %.1f)\n", ts ? "A=tmem" : "A=smem", N,
                   double(h[0]) / n, double(h[1]) / n, 128.0 * N / 256.0);
        }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}

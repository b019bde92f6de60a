// Bulk (TMA) shared->global store throughput: each CTA streams one 32 KB smem
// tile to successive 32 KB destinations (bulk_group, no reuse hazard).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
template <int CH>
__global__ void __launch_bounds__(128) bulk_store(char* Y, int per_cta) {
    __shared__ __align__(128) char st[32768];
    for (int i = threadIdx.x; i < 32768 / 16; i += 128) reinterpret_cast<int4*>(st)[i] = make_int4(i, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32768 / CH && threadIdx.x < 32) {
        for (int k = 0; k < per_cta; ++k) {
            char* dst = Y + (int64_t(blockIdx.x) * per_cta + k) * 32768;
            for (int c = threadIdx.x; c < 32768 / CH; c += 32)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * CH), "r"(smem_u32(st + c * CH)), "n"(CH) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}
__global__ void stg16(int4* Y, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) Y[i] = make_int4(0, 0, 0, 0);
}
int main() {
    char* Y; cudaMalloc(&Y, size_t(1) << 30);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int MB : {15, 60, 240}) {
        const int64_t bytes = int64_t(MB) << 20;
        const int per = int(bytes / 32768 / 148);
        float ms;
        for (int rep = 0; rep < 3; ++rep) { cudaEventRecord(a); bulk_store<32768><<<148, 128>>>(Y, per); cudaEventRecord(b); cudaEventSynchronize(b); }
        cudaEventElapsedTime(&ms, a, b); printf("%4d MB bulk 32KB : %7.2f us %7.0f GB/s\n", MB, ms * 1e3, per * 148.0 * 32768 / ms / 1e6);
        for (int rep = 0; rep < 3; ++rep) { cudaEventRecord(a); bulk_store<256><<<148, 128>>>(Y, per); cudaEventRecord(b); cudaEventSynchronize(b); }
        cudaEventElapsedTime(&ms, a, b); printf("%4d MB bulk 256B : %7.2f us %7.0f GB/s\n", MB, ms * 1e3, per * 148.0 * 32768 / ms / 1e6);
        for (int rep = 0; rep < 3; ++rep) { cudaEventRecord(a); stg16<<<148 * 8, 256>>>(reinterpret_cast<int4*>(Y), bytes / 16); cudaEventRecord(b); cudaEventSynchronize(b); }
        cudaEventElapsedTime(&ms, a, b); printf("%4d MB STG.128  : %7.2f us %7.0f GB/s\n", MB, ms * 1e3, bytes / ms / 1e6);
        for (int rep = 0; rep < 3; ++rep) { cudaEventRecord(a); cudaMemsetAsync(Y, 0, bytes); cudaEventRecord(b); cudaEventSynchronize(b); }
        cudaEventElapsedTime(&ms, a, b); printf("%4d MB memset   : %7.2f us %7.0f GB/s\n", MB, ms * 1e3, bytes / ms / 1e6);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}

// Microbenchmark: partition-order tile output ([tile][M][128] fp16, one 32 KB
// bulk S2G per unit) + a permute pass Y[m][c] = P[tile(c)][m][row(c)].
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_fp16.h>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(256) tile_store(__half* P, int M, int tiles, int units) {
    __shared__ __align__(128) __half st[128 * 128];
    const int r = threadIdx.x & 127, e = threadIdx.x >> 7;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int tile = u % tiles, tb = u / tiles;
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 64; ++j) st[(e * 64 + j) * 128 + r] = __float2half_rn(float(j + r));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            __half* dst = P + (int64_t(tile) * M + int64_t(tb) * 128) * 128;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(st)), "r"(128 * 128 * 2) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// one thread = 8 consecutive output columns of one token row
__global__ void __launch_bounds__(256) permute(const __half* __restrict__ P, const int* __restrict__ inv, __half* __restrict__ Y, int M, int N) {
    const int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
    const int per = N / 8;
    if (i >= int64_t(M) * per) return;
    const int m = int(i / per), c0 = int(i % per) * 8;
    const int4 i0 = __ldg(reinterpret_cast<const int4*>(inv + c0));
    const int4 i1 = __ldg(reinterpret_cast<const int4*>(inv + c0 + 4));
    const int iv[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
    __align__(16) __half v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = P[(int64_t(iv[q] >> 7) * M + m) * 128 + (iv[q] & 127)];
    *reinterpret_cast<int4*>(Y + int64_t(m) * N + c0) = *reinterpret_cast<const int4*>(v);
}

int main() {
    const int N = 14336, M = 512, tiles = N / 128, units = tiles * (M / 128);
    std::vector<int> cm(N), inv(N);
    std::mt19937 g(1);
    std::vector<int> idx(N);
    for (int i = 0; i < N; ++i) idx[i] = i;
    std::shuffle(idx.begin(), idx.end(), g);
    std::vector<int> s8(idx.begin(), idx.begin() + N / 10), s4(idx.begin() + N / 10, idx.end());
    std::sort(s8.begin(), s8.end()); std::sort(s4.begin(), s4.end());
    int k = 0;
    for (int c : s8) cm[k++] = c;
    for (int c : s4) cm[k++] = c;
    for (int p = 0; p < N; ++p) inv[cm[p]] = p;
    int* dinv; __half *Y, *P;
    cudaMalloc(&dinv, N * 4); cudaMalloc(&Y, size_t(M) * N * 2); cudaMalloc(&P, size_t(M) * N * 2);
    cudaMemcpy(dinv, inv.data(), N * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b, c; cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        tile_store<<<148, 256>>>(P, M, tiles, units);
        cudaEventRecord(b);
        permute<<<(M * (N / 8) + 255) / 256, 256>>>(P, dinv, Y, M, N);
        cudaEventRecord(c);
        cudaEventSynchronize(c);
        float m1, m2; cudaEventElapsedTime(&m1, a, b); cudaEventElapsedTime(&m2, b, c);
        printf("tile_store %.2f us   permute %.2f us (%.0f GB/s)\n", m1 * 1e3, m2 * 1e3, 2.0 * M * N * 2 / m2 / 1e6);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}

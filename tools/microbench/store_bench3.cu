// Store-throughput probe: bytes per lane, and whether successive warp stores of a
// thread hit the same row (dense) or hop a 28 KB row stride (the K2 output pattern).
#include <cstdio>
#include <cstdint>

template <typename T, bool kHop>
__global__ void __launch_bounds__(256) wr(T* Y, int rows_per_cta, int row_el) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T v{};
    if (kHop) {
        // CTA owns rows [b*R, b*R+R) x a 256-element column window; warp w: columns w*32.., rows j
        const int64_t col = (int64_t(blockIdx.x) % (row_el / 256)) * 256 + w * 32 + lane;
        const int64_t r0 = (int64_t(blockIdx.x) / (row_el / 256)) * rows_per_cta;
#pragma unroll 16
        for (int j = 0; j < rows_per_cta; ++j) Y[(r0 + j) * row_el + col] = v;
    } else {
        const int64_t base = int64_t(blockIdx.x) * rows_per_cta * 256;
#pragma unroll 16
        for (int j = 0; j < rows_per_cta; ++j) Y[base + int64_t(j) * 256 + w * 32 + lane] = v;
    }
}

template <typename T, bool kHop>
void run(const char* nm, char* Y, size_t bytes) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int R = 64;
    const int row_el = int(28672 / sizeof(T));                 // 28 KB rows
    const int64_t total_el = bytes / sizeof(T);
    const int grid = int(total_el / (int64_t(R) * 256));
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        wr<T, kHop><<<grid, 256>>>(reinterpret_cast<T*>(Y), R, row_el);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep == 2) printf("%-28s grid %6d: %7.2f us  %7.0f GB/s\n", nm, grid, ms * 1e3, bytes / ms / 1e6);
    }
}

int main() {
    const size_t bytes = size_t(512) * 28672;
    char* Y; cudaMalloc(&Y, bytes);
    run<uint16_t, false>("2B/lane dense", Y, bytes);
    run<uint16_t, true>("2B/lane row-hop", Y, bytes);
    run<uint32_t, false>("4B/lane dense", Y, bytes);
    run<uint32_t, true>("4B/lane row-hop", Y, bytes);
    run<uint4, false>("16B/lane dense", Y, bytes);
    run<uint4, true>("16B/lane row-hop", Y, bytes);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}

// mixed_gemm_simt.cu — debug GEMM on CUDA cores over the SAME packed layout
// (mq_layout.cuh) with the reference's exact op order (gemm.cpp:51-85). It is
// the GPU cross-check used while validating the tcgen05 kernel
// (mq_exec_opts.gemm_impl = 1), never the measured path.
// Also the permute kernel that puts all-gathered shards back in column order.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "mq_kernels.hpp"

namespace mq {
namespace {

constexpr int kTok = 16;

__device__ __forceinline__ void store_out(void* Y, int dt, int64_t idx, float v) {
    if (dt == 0) static_cast<float*>(Y)[idx] = v;
    else if (dt == 1) static_cast<__half*>(Y)[idx] = __float2half_rn(v);
    else static_cast<__nv_bfloat16*>(Y)[idx] = __float2bfloat16_rn(v);
}

// grid (num_tiles, ceil(M/16)), block 128: thread = tile row.
__global__ void __launch_bounds__(128) mixed_gemm_simt_kernel(const GemmParams p, const int8_t* __restrict__ codes,
                                                              int64_t ldc, int mode, int w8_unsigned) {
    const TileInfo td = tile_info(p, blockIdx.x);
    const int r = threadIdx.x;
    const int64_t m0 = int64_t(blockIdx.y) * kTok;
    if (r >= td.rows) return;
    const int cb = td.blk;
    float acc[kTok];
#pragma unroll
    for (int t = 0; t < kTok; ++t) acc[t] = 0.0f;
    for (int g = 0; g < p.G; ++g) {
        const uint8_t* blk = p.wq + td.off + int64_t(g) * cb;
        const uint8_t* meta = blk + (td.is8 ? kCodes8Bytes : kCodes4Bytes);
        const float sw = reinterpret_cast<const float*>(meta)[r];
        const int z = td.is8 ? 0 : meta[512 + r];
        int32_t s[kTok];
#pragma unroll
        for (int t = 0; t < kTok; ++t) s[t] = 0;
        for (int ch = 0; ch < 8; ++ch) {
            int wv[16];
            if (td.is8) {
                for (int j = 0; j < 16; ++j) {
                    const uint8_t b = blk[sw128_offset(r, ch * 16 + j)];
                    wv[j] = w8_unsigned ? int(b) : int(int8_t(b));
                }
            } else {
                const uint32_t w0 = *reinterpret_cast<const uint32_t*>(blk + sub4_chunk_offset(r, ch));
                const uint32_t w1 = *reinterpret_cast<const uint32_t*>(blk + sub4_chunk_offset(r, ch) + 4);
                for (int j = 0; j < 4; ++j) {
                    wv[j] = int((w0 >> (8 * j)) & 15u) - z;
                    wv[4 + j] = int((w0 >> (8 * j + 4)) & 15u) - z;
                    wv[8 + j] = int((w1 >> (8 * j)) & 15u) - z;
                    wv[12 + j] = int((w1 >> (8 * j + 4)) & 15u) - z;
                }
            }
            for (int t = 0; t < kTok; ++t) {
                const int64_t m = m0 + t;
                if (m >= p.M) break;
                const int64_t k0 = int64_t(g) * kGroupK + ch * 16;
                for (int j = 0; j < 16; ++j)
                    if (k0 + j < p.K) s[t] += int(codes[m * ldc + k0 + j]) * wv[j];
            }
        }
        for (int t = 0; t < kTok; ++t) {
            const int64_t m = m0 + t;
            if (m >= p.M) break;
            const float gs = __int2float_rn(s[t]);
            if (mode == kFastToken) {
                acc[t] = __fmaf_rn(gs, sw, acc[t]);
            } else {
                const float sa = p.sa_rm[int64_t(g) * p.sa_gstride + m];
                acc[t] = __fadd_rn(acc[t], __fmul_rn(gs, __fmul_rn(sa, sw)));
            }
        }
    }
    const int col = p.colmap[blockIdx.x * kTileRows + r];
    for (int t = 0; t < kTok; ++t) {
        const int64_t m = m0 + t;
        if (m >= p.M) break;
        float v = acc[t];
        if (mode == kFastToken) v = __fmul_rn(v, p.sa_rm[m]);
        store_out(p.Y, p.out_dtype, m * p.ldy + col, v);
    }
}

template <typename T>
__global__ void permute_kernel(const T* __restrict__ gathered, const int32_t* __restrict__ colmap,
                               int world, int64_t sc, int64_t M, int64_t N, T* __restrict__ Y) {
    const int64_t total = int64_t(world) * M * sc;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t j = i % sc;
        const int64_t rm = i / sc;
        const int64_t m = rm % M;
        const int64_t r = rm / M;
        const int32_t col = colmap[r * sc + j];
        if (col >= 0) Y[m * N + col] = gathered[i];
    }
}

}  // namespace

cudaError_t launch_mixed_gemm_simt(const GemmParams& p, const int8_t* codes, int64_t ldc, int mode,
                                   int w8_unsigned, cudaStream_t stream) {
    if (p.M == 0 || p.T8 + p.T4 == 0) return cudaSuccess;
    const dim3 grid(p.T8 + p.T4, static_cast<unsigned>((p.M + kTok - 1) / kTok));
    mixed_gemm_simt_kernel<<<grid, 128, 0, stream>>>(p, codes, ldc, mode, w8_unsigned);
    return cudaGetLastError();
}

cudaError_t launch_permute(const void* gathered, const int32_t* colmap, int world, int64_t sc,
                           int64_t M, int64_t N, void* Y, int dtype, cudaStream_t stream) {
    const int64_t total = int64_t(world) * M * sc;
    if (total == 0) return cudaSuccess;
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
    if (dtype == 0)
        permute_kernel<float><<<grid, 256, 0, stream>>>(static_cast<const float*>(gathered), colmap, world, sc, M, N, static_cast<float*>(Y));
    else
        permute_kernel<uint16_t><<<grid, 256, 0, stream>>>(static_cast<const uint16_t*>(gathered), colmap, world, sc, M, N, static_cast<uint16_t*>(Y));
    return cudaGetLastError();
}

// Cross-rank completion barrier for the fused-gather epilogue: rank `rank`
// raises its flag in every rank's flag array (release at system scope, so its
// peer stores are visible first), then waits until every rank's flag in its
// own array reached `epoch` (acquire). One thread per rank.
__device__ __forceinline__ void peer_barrier_body(uint32_t* const* flags, int world, int rank, uint32_t epoch) {
    const int t = threadIdx.x;
    if (t < world) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flags[t] + rank), "r"(epoch) : "memory");
    __syncthreads();
    if (t < world) {
        uint32_t v;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags[rank] + t) : "memory");
            if (int32_t(v - epoch) >= 0) break;
            __nanosleep(64);
        }
    }
}

struct PeerFlags {
    uint32_t* f[kMaxPeers];
};
__global__ void peer_barrier_kernel_v(PeerFlags pf, int world, int rank, uint32_t epoch) {
    peer_barrier_body(pf.f, world, rank, epoch);
}

cudaError_t launch_peer_barrier(uint32_t* const* flags, int world, int rank, uint32_t epoch, cudaStream_t stream) {
    if (world < 1 || world > kMaxPeers) return cudaErrorInvalidValue;
    PeerFlags pf{};
    for (int i = 0; i < world; ++i) pf.f[i] = flags[i];
    peer_barrier_kernel_v<<<1, 32, 0, stream>>>(pf, world, rank, epoch);
    return cudaGetLastError();
}

}  // namespace mq

// mq_kernels.hpp — launcher interface between the host code and the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "mq_layout.cuh"

namespace mq {

enum GemmMode : int {
    kExactGroup = 0,  // reference op order, group-wise s_a: f32 mul then add
    kFastGroup = 1,   // FFMA rescale, group-wise s_a, split-K allowed
    kFastToken = 2,   // per-token s_a factored out: acc += gs*s_w, y = s_a*acc
    kDumpPartials = 3 // int32 group sums to a [G, M, rows] buffer
};

struct GemmParams {
    const TileDesc* tiles;
    int32_t num_tiles;
    int32_t G;            // K-groups
    int64_t K;
    const uint8_t* wq;    // codes blocks
    const uint8_t* wmeta; // meta blocks
    const int32_t* colmap;
    const float* sa;      // activation scales
    int32_t sa_cols;      // G (group-wise) or 1 (per-token)
    int64_t M;
    void* Y;
    int32_t out_dtype;    // mq_dtype
    int64_t ldy;
    int32_t ksplit;
    int32_t token_blocks;
    float* ws;            // split-K partials
    uint32_t* counters;   // split-K arrival counters [num_tiles * token_blocks]
    uint32_t idesc8;      // instruction descriptor bits for sub8 tiles (u8 or s8 A)
    int32_t* partials;    // dump mode
    int32_t partial_rows;
};

// tcgen05 product kernel. token_tile in {16,32,64,128}; mode per GemmMode.
cudaError_t launch_mixed_gemm_tc(const GemmParams& p, const void* tmap_act, int token_tile,
                                 int mode, int num_sms, cudaStream_t stream);
// SIMT debug kernel (same layout, exact op order); parity aid, not the product.
cudaError_t launch_mixed_gemm_simt(const GemmParams& p, const int8_t* codes, int64_t ldc,
                                   int mode, int w8_unsigned, cudaStream_t stream);
cudaError_t launch_act_quant(const void* A, int a_dtype, int64_t M, int64_t K, int64_t lda,
                             int group, int f16_scales, int8_t* codes, int64_t ldc, float* scales,
                             int32_t* err, cudaStream_t stream);
cudaError_t launch_permute(const void* gathered, const int32_t* colmap, int world,
                           int64_t shard_cols, int64_t M, int64_t N, void* Y, int dtype,
                           cudaStream_t stream);
size_t gemm_smem_bytes(int token_tile, int* stages);

}  // namespace mq

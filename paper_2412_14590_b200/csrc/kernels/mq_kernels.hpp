// mq_kernels.hpp — launcher interface between the host code and the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "mq_layout.cuh"

namespace mq {

enum GemmMode : int {
    kExactGroup = 0,  // reference op order (f32 mul then add), no split-K
    kFastGroup = 1,   // FFMA rescale, group-wise s_a, stream-K splits
    kFastToken = 2,   // per-token s_a factored out: acc += gs*s_w, y = s_a*acc
    kDumpPartials = 3 // int32 group sums to a [G, M, rows] buffer
};

// One contiguous run of K-groups [g0, g1) of one (tile, token block) work
// item, processed by one CTA. Items split across CTAs (stream-K) publish f32
// partial tiles to slot `pslot`; the last arriving segment sums the item's
// nseg partials in sidx order (deterministic).
struct Seg {
    int32_t tile, tb, g0, g1;
    int32_t nseg, sidx, pslot, pad;
};
static_assert(sizeof(Seg) == 32, "Seg is 32 bytes");

struct GemmParams {
    const TileDesc* tiles;
    int32_t num_tiles;
    int32_t G;             // K-groups
    int64_t K;
    const uint8_t* wq;     // codes blocks
    const uint8_t* wmeta;  // meta blocks
    const int32_t* colmap;
    const float* sa;       // activation scales, group-major: sa[g * sa_gstride + m]
    int64_t sa_gstride;    // lds (group-wise) or 0 (per-token)
    int64_t M;
    void* Y;
    int32_t out_dtype;     // mq_dtype
    int64_t ldy;
    int32_t token_blocks;
    const Seg* segs;
    const int32_t* cta_seg;  // [grid + 1] segment ranges per CTA
    float* ws;               // stream-K partial tiles [slots][128][BN]
    uint32_t* counters;      // arrival counters [num_tiles * token_blocks]
    uint32_t idesc8;         // instruction descriptor bits for sub8 tiles (u8 or s8 A)
    int32_t* partials;       // dump mode
    int32_t partial_rows;
};

// tcgen05 product kernel. token_tile in {16,32,64,128}; mode per GemmMode;
// grid = number of CTAs in the schedule; pdl = launch with programmatic
// stream serialization (prologue + weight prefetch overlap the previous kernel).
cudaError_t launch_mixed_gemm_tc(const GemmParams& p, const void* tmap_act, int token_tile, int mode,
                                 int grid, bool pdl, cudaStream_t stream);
int gemm_stages(int token_tile);
// SIMT debug kernel (same layout, exact op order); parity aid, not the product.
cudaError_t launch_mixed_gemm_simt(const GemmParams& p, const int8_t* codes, int64_t ldc,
                                   int mode, int w8_unsigned, cudaStream_t stream);
// K1. scales are written group-major: scales[g * lds + m] (per-token: scales[m]).
cudaError_t launch_act_quant(const void* A, int a_dtype, int64_t M, int64_t K, int64_t lda,
                             int group, int f16_scales, int8_t* codes, int64_t ldc, float* scales,
                             int64_t lds, int32_t* err, bool pdl, cudaStream_t stream);
cudaError_t launch_permute(const void* gathered, const int32_t* colmap, int world,
                           int64_t shard_cols, int64_t M, int64_t N, void* Y, int dtype,
                           cudaStream_t stream);

}  // namespace mq

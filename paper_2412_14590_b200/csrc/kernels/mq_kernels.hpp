// mq_kernels.hpp — launcher interface between the host code and the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "mq_layout.cuh"

namespace mq {

enum GemmMode : int {
    kExactGroup = 0,  // reference op order (f32 mul then add), whole work items
    kFastGroup = 1,   // FFMA rescale, group-wise s_a, stream-K splits
    kFastToken = 2,   // per-token s_a factored out: acc += gs*s_w, y = s_a*acc
    kDumpPartials = 3 // int32 group sums to a [G, M, rows] buffer
};

// Everything the kernel needs is scalar: tile descriptors and the stream-K
// schedule are recomputed arithmetically in every CTA (no dependent global
// loads before the first weight copy). Work = items (tile, token block) x G
// K-groups, linearised item-major with the sub8 tiles first; CTA c owns the
// linear group range [cut(c), cut(c+1)) — cost-weighted (sub8 groups stream
// ~2x the bytes of sub4 groups) when split, whole items otherwise.
struct GemmParams {
    int32_t T8, T4;         // 128-row tiles of sub8 / sub4
    int64_t n8, n4;         // rows of sub8 / sub4
    int32_t G;              // K-groups
    int32_t TB;             // token blocks (BN tokens each)
    int64_t K;
    const uint8_t* wq;      // codes blocks (mq_layout.cuh)
    const uint8_t* wmeta;   // meta blocks
    const int32_t* colmap;  // [ (T8+T4)*128 ] output column of every tile row
    const float* sa;        // activation scales, group-major: sa[g * sa_gstride + m]
    int64_t sa_gstride;     // lds (group-wise) or 0 (per-token)
    int64_t M;
    void* Y;
    int32_t out_dtype;      // mq_dtype
    int64_t ldy;
    int32_t P;              // CTAs
    int32_t split;          // 1: stream-K (cuts inside items), 0: whole items
    int32_t c8, c4;         // per-group stream costs (split mode)
    float* ws;              // stream-K partial tiles [2*P][128][BN]
    uint32_t* counters;     // arrival counters [items]
    uint32_t idesc8;        // instruction descriptor bits for sub8 tiles (u8 or s8 A)
    int32_t* partials;      // dump mode
    int32_t partial_rows;
    int32_t dbg;            // development: pipeline-stage bypass bits (MQ_DBG env), 0 in production
};

// tcgen05 product kernel. token_tile in {16,32,64,128}; mode per GemmMode;
// pdl = launch with programmatic stream serialization (prologue + weight
// prefetch overlap the previous kernel).
cudaError_t launch_mixed_gemm_tc(const GemmParams& p, const void* tmap_act, int token_tile, int mode,
                                 bool pdl, cudaStream_t stream);
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

// Tile descriptor of tile t (sub8 tiles first), identical to the host packer.
struct TileInfo {
    int64_t codes_off, meta_off;
    int32_t is8, rows, copy_bytes, first;
};
__host__ __device__ inline TileInfo tile_info(const GemmParams& p, int t) {
    TileInfo ti;
    ti.is8 = t < p.T8;
    const int64_t G = p.G;
    if (ti.is8) {
        ti.first = t * kTileRows;
        ti.codes_off = int64_t(t) * G * kCodes8Bytes;
        ti.meta_off = int64_t(t) * G * kMeta8Bytes;
        const int64_t rem = p.n8 - ti.first;
        ti.rows = int32_t(rem < kTileRows ? rem : kTileRows);
        ti.copy_bytes = (ti.rows + 7) / 8 * 1024;
    } else {
        const int u = t - p.T8;
        ti.first = u * kTileRows;
        ti.codes_off = int64_t(p.T8) * G * kCodes8Bytes + int64_t(u) * G * kCodes4Bytes;
        ti.meta_off = int64_t(p.T8) * G * kMeta8Bytes + int64_t(u) * G * kMeta4Bytes;
        const int64_t rem = p.n4 - ti.first;
        ti.rows = int32_t(rem < kTileRows ? rem : kTileRows);
        ti.copy_bytes = ti.rows * 64;
    }
    return ti;
}

// The stream-K partition (see GemmParams).
struct Schedule {
    int64_t X8, X, U, items;
    int32_t G, P, split, c8, c4;
    __host__ __device__ Schedule(const GemmParams& p) {
        items = int64_t(p.T8 + p.T4) * p.TB;
        X8 = int64_t(p.T8) * p.TB * p.G;
        X = items * p.G;
        G = p.G;
        P = p.P;
        split = p.split;
        c8 = p.c8;
        c4 = p.c4;
        U = X8 * c8 + (X - X8) * c4;
    }
    __host__ __device__ int64_t cut(int c) const {
        if (c <= 0) return 0;
        if (c >= P) return X;
        if (!split) return (int64_t(c) * items / P) * G;
        const int64_t t = (U / P) * c + ((U % P) * c) / P;  // floor(U*c/P) without overflow
        const int64_t x = t <= X8 * c8 ? (t + c8 - 1) / c8 : X8 + (t - X8 * c8 + c4 - 1) / c4;
        return x < X ? x : X;
    }
    __host__ __device__ int cta_of(int64_t x) const {  // the CTA whose range holds x (split mode)
        const int64_t cx = x <= X8 ? x * c8 : X8 * c8 + (x - X8) * c4;
        int c = int((cx * P) / (U > 0 ? U : 1));
        if (c > P - 1) c = P - 1;
        while (c > 0 && cut(c) > x) --c;
        while (c < P - 1 && cut(c + 1) <= x) ++c;
        return c;
    }
};

}  // namespace mq

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
    kDumpPartials = 3, // int32 group sums to a [G, M, rows] buffer
    kExactToken = 4   // reference op order with a per-token s_a broadcast over groups
};

// Everything the kernel needs is scalar: tile descriptors and the stream-K
// schedule are recomputed arithmetically in every CTA (no dependent global
// loads before the first weight copy). Work = items (tile, token block) x G
// K-groups, linearised item-major with the sub8 tiles first; CTA c owns the
// linear group range [cut(c), cut(c+1)) — cost-weighted (sub8 groups stream
// ~2x the bytes of sub4 groups) when split, whole items otherwise.
constexpr int kMaxCtas = 160;  // >= SM count (148 on B200)

struct GemmParams {
    int32_t T8, T4;         // 128-row tiles of sub8 / sub4
    int64_t n8, n4;         // rows of sub8 / sub4
    int32_t G;              // K-groups
    int32_t TB;             // token blocks (BN tokens each)
    int64_t K;
    const uint8_t* wq;      // merged code+meta blocks (mq_layout.cuh)
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
    int32_t cuts[kMaxCtas + 1];  // CTA c owns linear groups [cuts[c], cuts[c+1]) (param space: no loads)
    int32_t dbg;            // development: pipeline-stage bypass bits (MQ_DBG env), 0 in production
    unsigned long long* trace;  // development: per-CTA globaltimer stamps [P][8] (MQ_DBG & 32)
};

// tcgen05 product kernel. token_tile in {16,32,64,128}; mode per GemmMode;
// tmap_act: 3-D tensor map {128, M, G} over the int8 codes (box {128, BN, GPS});
// tmap_sa: 2-D tensor map {M, G} over the group-major scales (box {BN, GPS});
// pdl = launch with programmatic stream serialization (prologue + weight
// prefetch overlap the previous kernel).
cudaError_t launch_mixed_gemm_tc(const GemmParams& p, const void* tmap_act, const void* tmap_sa, int token_tile,
                                 int mode, bool pdl, cudaStream_t stream);
// groups of a sub4 tile per pipeline stage (sub8: half) for a token tile
#ifndef MQ_GPS_SMALL
#define MQ_GPS_SMALL 4
#endif
constexpr int gemm_gps(int token_tile) { return token_tile <= 32 ? MQ_GPS_SMALL : (token_tile == 64 ? 2 : 1); }
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
    int64_t off;     // byte offset of the tile's group-0 block
    int32_t is8, rows, first, blk;
};
__host__ __device__ inline TileInfo tile_info(const GemmParams& p, int t) {
    TileInfo ti;
    ti.is8 = t < p.T8;
    const int64_t G = p.G;
    if (ti.is8) {
        ti.first = t * kTileRows;
        ti.off = int64_t(t) * G * kBlock8Bytes;
        ti.blk = kBlock8Bytes;
        const int64_t rem = p.n8 - ti.first;
        ti.rows = int32_t(rem < kTileRows ? rem : kTileRows);
    } else {
        const int u = t - p.T8;
        ti.first = u * kTileRows;
        ti.off = int64_t(p.T8) * G * kBlock8Bytes + int64_t(u) * G * kBlock4Bytes;
        ti.blk = kBlock4Bytes;
        const int64_t rem = p.n4 - ti.first;
        ti.rows = int32_t(rem < kTileRows ? rem : kTileRows);
    }
    return ti;
}

// CTA owning linear group x (binary search over the parameter-space cut table).
__host__ __device__ inline int cta_owner(const GemmParams& p, int32_t x) {
    int lo = 0, hi = p.P - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p.cuts[mid] <= x) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// The stream-K partition (see GemmParams); evaluated once on the host to fill
// GemmParams::cuts.
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

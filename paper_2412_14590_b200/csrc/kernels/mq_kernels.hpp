// mq_kernels.hpp — launcher interface between the host code and the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "mq_layout.cuh"

namespace mq {

enum GemmMode : int {
    kExactGroup = 0,    // reference op order (f32 mul then add), no K splitting
    kFastGroup = 1,     // FFMA rescale, group-wise s_a, cluster split-K
    kFastToken = 2,     // per-token s_a factored out: acc += gs*s_w, y = s_a*acc
    kDumpPartials = 3,  // int32 group sums to a [G, M, rows] buffer
    kExactToken = 4     // reference op order with a per-token s_a broadcast over groups
};

// ---------------------------------------------------------------------------
// Engine activation layout (EAL), written by K1 and streamed by K2 with plain
// bulk copies (one per chunk when the batch fits one token tile):
//   codes  uint8 [G][Mpad][128]: byte (g, m, k) at g*Mpad*128 + m*128 +
//          ((((k >> 4) ^ (m & 7)) << 4) | (k & 15))  — each (group, token-tile)
//          is a ready UMMA K-major SWIZZLE_128B operand image;
//   scales f32   [G][Mpad] (group-wise) or [Mpad] (per-token);
//   asum   int32 [G][Mpad] sum of each (group, token)'s codes.
// Mpad = TB * BN (token tile BN); rows m >= M are zero. Ragged K groups are
// zero-padded to 128.
__host__ __device__ inline uint32_t eal_offset(uint32_t m, uint32_t k) {
    return m * 128u + ((((k >> 4) ^ (m & 7u)) << 4) | (k & 15u));
}

// ---------------------------------------------------------------------------
// K2 schedule. Work UNITS = (token block, weight tile, K-slice), run by a
// persistent grid of <= #SM CTAs (CTA b takes units b, b + grid, ...; no
// clusters: cluster launches cost several us per kernel at decode sizes).
// Per token block the units are: S8 slices of every sub8 tile (tile-major),
// then S4 slices of every sub4 tile. Decode uses S8 = 2*S4 so every CTA
// streams about the same bytes (a sub8 group is twice a sub4 group). When an
// item (tile, token block) is split (S > 1), each slice writes its f32 partial
// tile to its own workspace slot and bumps the item's counter; the LAST slice
// to arrive sums the S partials in slice order (deterministic) and scatters
// the result, then re-arms the counter.
// Stream-K schedule (FAST modes, host-planned, GemmParams::sk): the work is
// the sequence of ITEMS (token block, tile) x G groups, in cost units (a sub8
// group costs c8 = 2 at decode, where bytes rule, and 1 when token-tiled);
// CTA b runs positions [skb[b], skb[b+1]) packed as item << 8 | group, cut at
// chunk boundaries. Items cut between CTAs are reduced by the piece that
// completes their G groups (arrival counter counts groups).
constexpr int kSkMax = 160;  // >= SMs of the device
constexpr int kMaxPeers = 8;  // ranks of one NVLink domain the fused-gather epilogue writes to
// Counter words at the start of every forward workspace, indexed by item (a
// launch with split items has TB == 1, or fewer items than SMs) or by
// stream-K boundary (<= kSkMax): a fixed region, so one workspace serves any M
// and any layer. Every launch leaves the words it used at zero.
constexpr int kCntWords = 8192;
// per-token activation quantization (EAL row kernel): one CTA holds a whole row
constexpr int64_t kPerTokenKMax = 32768;

struct GemmParams {
    // Hot fields first: every role decodes its first unit from these before its
    // first chunk, so they share one 64-byte constant-cache line (cold param
    // lines cost a dependent constant-bank miss each at kernel start).
    int32_t sk;             // 1: stream-K schedule (skb), 0: unit schedule (units/S8/S4)
    int32_t units;          // work units (token block x tile x K-slice)
    int32_t T8, T4;         // 128-row tiles of sub8 / sub4
    int32_t TB;             // token blocks (BN tokens each)
    int32_t G;              // K-groups
    int32_t S8, S4;         // K-slices per sub8 / sub4 item (powers of two)
    int32_t lgS8, lgS4;     // log2 of S8 / S4: unit decoding uses shifts, not divisions
    int32_t rotate;         // 1: each CTA starts its K loop at a CTA-dependent chunk (FAST modes)
    int32_t T;              // T8 + T4
    int32_t dbg;            // development: pipeline-stage bypass bits (MQ_DBG env), 0 in production
    int32_t grid;           // persistent CTAs (<= SMs): CTA b runs units b, b + grid, ...
    const uint8_t* wq;      // merged code+meta blocks (mq_layout.cuh)
    int64_t n8, n4;         // rows of sub8 / sub4
    const int32_t* colmap;  // [ (T8+T4)*128 ] output column of every tile row
    // EAL activations (tensor-core kernel)
    const uint8_t* acts;    // [G][Mpad][128]
    const float* sa;        // [G][Mpad] (group-wise) or [Mpad] (per-token)
    const int32_t* asum;    // [G][Mpad] per-(group, token) code sums (zero-point correction)
    int64_t Mpad;
    int64_t M;
    unsigned long long* trace;  // development: per-CTA globaltimer stamps [P][8] (MQ_DBG & 32)
    int64_t K;
    // row-major activations (SIMT debug kernel): scales sa_rm[g * sa_gstride + m]
    const float* sa_rm;
    int64_t sa_gstride;
    void* Y;
    int32_t out_dtype;      // mq_dtype
    uint32_t idesc8;        // instruction descriptor bits for sub8 tiles (u8 or s8 A)
    int64_t ldy;
    float* part;            // split-K partial tiles [units][BN][128] (slot = unit index); stream-K: tails
    float* part2;           // stream-K: head partial tiles [grid + 1][BN][128]
    uint32_t* cnt;          // arrival counters [kCntWords] (item, or stream-K boundary), zero between launches
    int32_t no_spin;        // 1: no cross-CTA spin-waits (concurrent launches may hold SMs)
    int32_t partial_rows;
    const uint8_t* pf;      // next layer's packed weights: prefetched into L2 once this launch's reads are issued
    int64_t pf_bytes;       // bytes of pf to prefetch (0: none), split evenly over the CTAs
    int32_t* partials;      // dump mode
    int32_t npeer;          // fused gather: every output also goes to ypeer[1 .. npeer) (Y == ypeer[0])
    void* ypeer[kMaxPeers];  // peer ranks' full outputs [M, N] (UVA / NVLink peer-mapped)
    uint32_t skb[kSkMax + 1];  // stream-K CTA boundaries (item << 8 | group)
};

// One unit's work: rows of `tile` x tokens of block `tb` x groups [g0, g1);
// slice `sl` of S; the item's slices are units [cta0, cta0 + S).
struct Work {
    int tile, tb, g0, g1, S, sl, cta0, item;
};
// Decoding is on every role's critical path at kernel start (a chain of integer
// divisions costs ~1 us per CTA), so slices are powers of two and decode uses
// shifts; only token-tiled launches (TB > 1, prefill) divide.
__host__ __device__ inline Work work_of(const GemmParams& p, int cta) {
    Work w;
    const int per_tb = (p.T8 << p.lgS8) + (p.T4 << p.lgS4);
    w.tb = p.TB == 1 ? 0 : cta / per_tb;
    int u = cta - w.tb * per_tb;
    if (u < (p.T8 << p.lgS8)) {
        w.tile = u >> p.lgS8, w.S = p.S8, w.sl = u & (p.S8 - 1);
    } else {
        u -= p.T8 << p.lgS8;
        w.tile = p.T8 + (u >> p.lgS4), w.S = p.S4, w.sl = u & (p.S4 - 1);
    }
    w.cta0 = cta - w.sl;
    w.item = w.tb * (p.T8 + p.T4) + w.tile;
    const int lg = w.S == p.S8 ? p.lgS8 : p.lgS4;
    w.g0 = (w.sl * p.G) >> lg;
    w.g1 = ((w.sl + 1) * p.G) >> lg;
    return w;
}

// tcgen05 product kernel. token_tile in {16,32,64,128}; mode per GemmMode;
// pdl = launch with programmatic stream serialization (prologue + weight
// prefetch overlap the previous kernel).
cudaError_t launch_mixed_gemm_tc(const GemmParams& p, int token_tile, int mode, bool pdl, cudaStream_t stream);
// groups of a sub4 tile per pipeline stage (sub8: half) for a token tile
#ifndef MQ_GPS_SMALL
#define MQ_GPS_SMALL 4
#endif
// (A/B in graph: 16- and 32-token tiles stream best with 4-group chunks — at
// decode the per-chunk hand-offs dominate; M = 24-32 stack -3..5% vs 2-group
// chunks with 4 activation stages; 64-token tiles 2, 128-token tiles 1 (TMEM))
#ifndef MQ_GPS32
#define MQ_GPS32 4
#endif
constexpr int gemm_gps(int token_tile) {
    return token_tile <= 16 ? MQ_GPS_SMALL : token_tile <= 32 ? MQ_GPS32 : (token_tile <= 64 ? 2 : 1);
}
int gemm_stages(int token_tile);
// SIMT debug kernel (same weight layout, exact op order, row-major activations).
cudaError_t launch_mixed_gemm_simt(const GemmParams& p, const int8_t* codes, int64_t ldc,
                                   int mode, int w8_unsigned, cudaStream_t stream);
// K1 (reference layout): codes [M, ldc] row-major; scales group-major scales[g * lds + m] (per-token: scales[m]).
cudaError_t launch_act_quant(const void* A, int a_dtype, int64_t M, int64_t K, int64_t lda,
                             int group, int f16_scales, int8_t* codes, int64_t ldc, float* scales,
                             int64_t lds, int32_t* err, bool pdl, cudaStream_t stream);
// K1 (engine layout, EAL): group == 128 (group-wise) or K (per-token). Also
// writes asum [G][Mpad] int32 = the sum of each (group, token)'s codes, the
// zero-point correction term of the decode GEMM (sum a(c - z) = sum a c - z sum a).
cudaError_t launch_act_quant_eal(const void* A, int a_dtype, int64_t M, int64_t K, int64_t lda, int group,
                                 int64_t Mpad, uint8_t* acts, float* sa, int32_t* asum, int32_t* err, int f16,
                                 bool pdl, cudaStream_t stream);
// Row-major codes [M, ldc] + group-major scales [G, lds] (or [M]) -> EAL (+ asum).
cudaError_t launch_repack_eal(const int8_t* codes, int64_t ldc, const float* scales, int64_t lds, int per_token,
                              int64_t M, int64_t K, int64_t Mpad, uint8_t* acts, float* sa, int32_t* asum,
                              cudaStream_t stream);
// Cross-rank completion barrier over peer-mapped flags (mq_peer_barrier).
cudaError_t launch_peer_barrier(uint32_t* const* flags, int world, int rank, uint32_t epoch, cudaStream_t stream);
cudaError_t launch_permute(const void* gathered, const int32_t* colmap, int world, int64_t shard_cols,
                           int64_t M, int64_t N, void* Y, int dtype, cudaStream_t stream);

// Offline weight quantization / prepack on the GPU (weight_quant.cu).
cudaError_t launch_weight_quant(const double* W, int64_t K, const int32_t* map, int64_t rows, int group, int bits,
                                int sym, int f16, uint8_t* codes, float* scales, uint8_t* zp, int32_t* err,
                                cudaStream_t stream);
cudaError_t launch_pack_nibbles(const uint8_t* codes, int64_t rows, int64_t K, uint8_t* payload, cudaStream_t stream);
cudaError_t launch_engine_pack(int32_t T8, int32_t T4, int64_t n8, int64_t n4, int64_t a8, int64_t a4, int32_t G,
                               int64_t K, const uint8_t* payload8, const float* scales8, const uint8_t* payload4,
                               const float* scales4, const uint8_t* zp4, uint8_t* wq, cudaStream_t stream);
cudaError_t launch_meta_check(const float* s8, int64_t n8, const float* s4, int64_t n4, const uint8_t* zp4,
                              int32_t* flags, cudaStream_t stream);

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

}  // namespace mq

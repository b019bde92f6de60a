// mq_layout.cuh — the engine's HBM layout of a packed mixed layer, shared by
// the host packer (mq_layer.cpp) and the sm_100a kernels.
//
// A layer is cut into 128-row TILES (tcgen05 M = 128): first the sub8 tiles,
// then the sub4 tiles. For every (tile, K-group of 128) there is one BLOCK
// holding the group's codes followed by its metadata, stored tile-major /
// group-minor, so a run of consecutive groups of one tile is ONE contiguous
// range the producer moves with a single cp.async.bulk (on sm_100a the bulk
// copy engine is bounded per operation, not per byte: few, large copies):
//   sub8 block 17408 B: codes 16384 B = 128 rows x 128 int8 already in the
//              UMMA K-major SWIZZLE_128B image (consumed by tcgen05.mma in
//              place, no conversion) | f32 scales[128] | 512 B pad (keeps every
//              block 1024-B aligned for the SW128 atoms);
//   sub4 block  8832 B: codes 8192 B of nibbles stored column-chunk-major —
//              the 32 codes [32q, 32q+32) of row r at q*2048 + r*16 (16-code
//              halves at +0 / +8, nibble order per pack_chunk4) so the
//              converter's per-row 16-byte loads are bank-conflict free and its
//              output words come out in K order | f32 scales[128] | u8 zero
//              points[128].
// Rows past the end of a ragged tile are zero.
#pragma once
#include <cstdint>

namespace mq {

constexpr int kTileRows = 128;      // tcgen05.mma M
constexpr int kGroupK = 128;        // K-group = one SWIZZLE_128B atom row of int8
constexpr int kCodes8Bytes = 16384; // 128 x 128 int8
constexpr int kCodes4Bytes = 8192;  // 128 x 128 nibbles
constexpr int kBlock8Bytes = 17408; // codes | scales | pad
constexpr int kBlock4Bytes = 8832;  // codes | scales | zero points

// byte offset of the 16-code chunk c (0..7) of row r inside a sub4 block
__host__ __device__ inline uint32_t sub4_chunk_offset(uint32_t r, uint32_t c) {
    return (c >> 1) * 2048u + r * 16u + (c & 1u) * 8u;
}

struct TileDesc {  // host-side bookkeeping of one tile
    int64_t codes_off;   // byte offset of the tile's group-0 block
    int32_t is8;         // 1: sub8 tile (int8 codes), 0: sub4 tile (u4 + zero points)
    int32_t rows;        // valid rows in the tile (1..128)
    int32_t first;       // first sub-problem row of the tile
    int32_t pad;
};

// Byte offset of int8 element (row r, k) inside a 128-row K-major
// SWIZZLE_128B image: 8-row x 128 B atoms, 16-byte chunks XOR-ed by r%8.
__host__ __device__ inline uint32_t sw128_offset(uint32_t r, uint32_t k) {
    return (r >> 3) * 1024u + (r & 7u) * 128u + ((((k >> 4) ^ (r & 7u)) << 4) | (k & 15u));
}

// tcgen05 instruction descriptor for kind::i8: D s32, A/B 8-bit (signedness per
// operand: the reference-compatible sub8 mode reads A as u8), both K-major,
// M = 128, N = n (cute::UMMA::InstrDescriptor bit layout).
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t n, bool a_signed, bool b_signed) {
    return (2u << 4)                        // c_format = S32
           | ((a_signed ? 1u : 0u) << 7)    // a_format: 1 = s8, 0 = u8
           | ((b_signed ? 1u : 0u) << 10)   // b_format
           | (0u << 15) | (0u << 16)        // a_major = b_major = K
           | ((n >> 3) << 17)               // N >> 3
           | ((128u >> 4) << 24);           // M >> 4
}

// sub4 chunk encoding: the 16 codes e[0..15] of (row r, chunk c) are stored
// as two little-endian words: w0 byte j = e[j] | e[4+j] << 4 and
// w1 byte j = e[8+j] | e[12+j] << 4, so (w & 0x0F0F0F0F) yields codes 0..3 and
// ((w >> 4) & 0x0F0F0F0F) codes 4..7 in byte order.
__host__ __device__ inline void pack_chunk4(const uint8_t* e, uint32_t* w0, uint32_t* w1) {
    uint32_t a = 0, b = 0;
    for (int j = 0; j < 4; ++j) {
        a |= uint32_t(e[j] | (e[4 + j] << 4)) << (8 * j);
        b |= uint32_t(e[8 + j] | (e[12 + j] << 4)) << (8 * j);
    }
    *w0 = a;
    *w1 = b;
}

}  // namespace mq

// weight_quant.cu — offline weight quantization and prepack on the GPU (SURVEY
// §8f row 4). The host packer walks every code byte by byte (~0.4 s per 4096²
// layer, minutes for a 70B model); these kernels do the same work bit for bit:
//
//   wq_quant_kernel   partition_and_quantize (proj/src/mixed.cpp:46-81): the
//                     gather of a sub-problem's rows through its index map fused
//                     with quantize_group_sym / quantize_group_asym<double>
//                     (proj/include/mixquant/quant.hpp:84-140). One warp per
//                     (row, group); every step in IEEE double exactly as the
//                     reference's scalar code: min/max (order-free), one
//                     division per scale and per code, round() half away from
//                     zero, the scale stored through f32 (optionally the f16
//                     grid, quant.cpp:81-86) with the reference's fallbacks.
//   wq_pack4_kernel   pack_nibbles (proj/src/tensor.cpp:63-78) of a 4-bit
//                     sub-problem's codes into the reference payload rows.
//   wq_engine_kernel  the engine's HBM layout (mq_layout.cuh) from reference
//                     layouts already in device memory: one CTA per (tile,
//                     group) block, one thread per tile row — the device twin
//                     of the host packer in mq_layer.cpp (same bytes).
//   wq_check_kernel   validate_quantized's scale / zero-point checks
//                     (proj/src/quant.cpp:81-101) on device metadata.
#include <cuda_fp16.h>

#include <cstdint>

#include "mq_kernels.hpp"

namespace mq {
namespace {

__device__ __forceinline__ double stored_scale(double s, double fallback, int f16) {
    float v = static_cast<float>(s);  // __double2float_rn
    if (v == 0.0f) v = static_cast<float>(fallback);
    if (f16) {  // round_scale_f16: RNE to binary16, clamp to the smallest subnormal
        v = __half2float(__float2half_rn(v));
        if (!(v > 0.0f)) v = 5.9604644775390625e-8f;
    }
    return static_cast<double>(v);
}

// codes [rows, K] one byte per code (8-bit: int8 bits, the reference payload;
// 4-bit: 0..15, packed afterwards), scales [rows, G] f32, zp [rows, G] (asym).
template <bool SYM>
__global__ void __launch_bounds__(256) wq_quant_kernel(const double* __restrict__ W, int64_t K,
                                                       const int32_t* __restrict__ map, int64_t rows, int g,
                                                       int64_t G, int qmax, int f16, uint8_t* __restrict__ codes,
                                                       float* __restrict__ scales, uint8_t* __restrict__ zp,
                                                       int32_t* err) {
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= rows * G) return;
    const int64_t row = wid / G, gi = wid - row * G;
    const int64_t b = gi * g;
    const int n = static_cast<int>(K - b < g ? K - b : g);
    const double* x = W + int64_t(map[row]) * K + b;
    bool finite = true;
    double amax = 0.0, mn = 0.0, mx = 0.0;
    bool any = false;
    for (int i = lane; i < n; i += 32) {
        const double v = x[i];
        finite &= isfinite(v);
        amax = fmax(amax, fabs(v));
        mn = any ? fmin(mn, v) : v;
        mx = any ? fmax(mx, v) : v;
        any = true;
    }
    finite = __all_sync(0xffffffffu, finite);
    if (!finite) {  // DataError (quant.hpp:56-64): report the first failing (row, group)
        if (lane == 0) atomicMin(err, static_cast<int32_t>(wid < INT32_MAX ? wid : INT32_MAX));
        return;
    }
    for (int o = 16; o; o >>= 1) {
        amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        const double omn = __shfl_xor_sync(0xffffffffu, mn, o), omx = __shfl_xor_sync(0xffffffffu, mx, o);
        const bool oany = __shfl_xor_sync(0xffffffffu, any, o);
        if (oany) {
            mn = any ? fmin(mn, omn) : omn;
            mx = any ? fmax(mx, omx) : omx;
            any = true;
        }
    }
    uint8_t* c = codes + row * K + b;
    if (SYM) {
        // quant.hpp:117-140: s = amax / qmax (1e-8 when amax == 0), fallback max(amax, 1e-8)
        const double s = stored_scale(amax == 0.0 ? 1e-8 : amax / double(qmax), fmax(amax, 1e-8), f16);
        for (int i = lane; i < n; i += 32) {
            long long q = llround(round(x[i] / s));
            q = q < -qmax ? -qmax : (q > qmax ? qmax : q);
            c[i] = static_cast<uint8_t>(static_cast<int8_t>(q));
        }
        if (lane == 0) scales[row * G + gi] = static_cast<float>(s);
    } else {
        // quant.hpp:84-112: s = (max - min) / qmax, z = clamp(round(-min / s), 0, qmax)
        const double fb = fmax(fmax(fabs(mn), fabs(mx)), 1e-8);
        const double s = stored_scale(mx == mn ? fb : (mx - mn) / double(qmax), fb, f16);
        long long z = llround(round(-mn / s));
        z = z < 0 ? 0 : (z > qmax ? qmax : z);
        for (int i = lane; i < n; i += 32) {
            long long q = llround(round(x[i] / s)) + z;
            q = q < 0 ? 0 : (q > qmax ? qmax : q);
            c[i] = static_cast<uint8_t>(q);
        }
        if (lane == 0) {
            scales[row * G + gi] = static_cast<float>(s);
            zp[row * G + gi] = static_cast<uint8_t>(z);
        }
    }
}

// tensor.cpp:63-78: byte k = v[2k] | v[2k+1] << 4, odd count pads the high nibble with 0
__global__ void wq_pack4_kernel(const uint8_t* __restrict__ codes, int64_t rows, int64_t K,
                                uint8_t* __restrict__ payload) {
    const int64_t stride = (K + 1) / 2;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows * stride) return;
    const int64_t r = i / stride, k = i - r * stride;
    const uint8_t* c = codes + r * K;
    const uint8_t lo = c[2 * k], hi = 2 * k + 1 < K ? c[2 * k + 1] : 0;
    payload[i] = static_cast<uint8_t>(lo | (hi << 4));
}

// One CTA per (tile, group) block of the engine layout, thread r = tile row.
// a8 / a4: first global sub row of this shard; rows past the sub-problem
// (ragged tiles) and codes past K are zero.
__global__ void __launch_bounds__(128) wq_engine_kernel(int32_t T8, int64_t n8, int64_t n4, int64_t a8,
                                                        int64_t a4, int32_t G, int64_t K,
                                                        const uint8_t* __restrict__ payload8,
                                                        const float* __restrict__ scales8,
                                                        const uint8_t* __restrict__ payload4,
                                                        const float* __restrict__ scales4,
                                                        const uint8_t* __restrict__ zp4, uint8_t* __restrict__ wq) {
    const int64_t blk = blockIdx.x;
    const int t = static_cast<int>(blk / G), g = static_cast<int>(blk - int64_t(t) * G);
    const int r = threadIdx.x;
    const int64_t k0 = int64_t(g) * kGroupK;
    if (t < T8) {
        uint8_t* cb = wq + (int64_t(t) * G + g) * kBlock8Bytes;
        const int64_t lr = int64_t(t) * kTileRows + r;
        const bool live = lr < n8;
        const uint8_t* src = payload8 + (a8 + lr) * K;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
            uint32_t w[4] = {0u, 0u, 0u, 0u};
            if (live)
                for (int j = 0; j < 16; ++j) {
                    const int64_t k = k0 + ch * 16 + j;
                    if (k < K) w[j >> 2] |= uint32_t(src[k]) << (8 * (j & 3));
                }
            *reinterpret_cast<uint4*>(cb + sw128_offset(uint32_t(r), uint32_t(ch * 16))) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        reinterpret_cast<float*>(cb + kCodes8Bytes)[r] = live ? scales8[(a8 + lr) * G + g] : 0.0f;
        reinterpret_cast<uint32_t*>(cb + kCodes8Bytes + 512)[r] = 0u;  // alignment pad
        return;
    }
    const int u = t - T8;
    uint8_t* cb = wq + int64_t(T8) * G * kBlock8Bytes + (int64_t(u) * G + g) * kBlock4Bytes;
    const int64_t lr = int64_t(u) * kTileRows + r;
    const bool live = lr < n4;
    const int64_t stride4 = (K + 1) / 2;
    const uint8_t* src = payload4 + (a4 + lr) * stride4;
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
        uint8_t e[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int64_t k = k0 + ch * 16 + j;
            e[j] = (live && k < K) ? ((k & 1) ? (src[k >> 1] >> 4) : (src[k >> 1] & 0x0F)) : 0;
        }
        uint32_t w0, w1;
        pack_chunk4(e, &w0, &w1);
        *reinterpret_cast<uint2*>(cb + sub4_chunk_offset(uint32_t(r), uint32_t(ch))) = make_uint2(w0, w1);
    }
    reinterpret_cast<float*>(cb + kCodes4Bytes)[r] = live ? scales4[(a4 + lr) * G + g] : 0.0f;
    cb[kCodes4Bytes + 512 + r] = live ? zp4[(a4 + lr) * G + g] : 0;
}

// flags[0]: a non-positive scale, flags[1]: a 4-bit zero point > 15
__global__ void wq_check_kernel(const float* __restrict__ s8, int64_t n8, const float* __restrict__ s4, int64_t n4,
                                const uint8_t* __restrict__ zp4, int32_t* flags) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n8 + n4; i += int64_t(gridDim.x) * blockDim.x) {
        const float s = i < n8 ? s8[i] : s4[i - n8];
        if (!(s > 0.0f)) flags[0] = 1;
        if (i >= n8 && zp4[i - n8] > 15) flags[1] = 1;
    }
}

}  // namespace

cudaError_t launch_weight_quant(const double* W, int64_t K, const int32_t* map, int64_t rows, int group, int bits,
                                int sym, int f16, uint8_t* codes, float* scales, uint8_t* zp, int32_t* err,
                                cudaStream_t stream) {
    const int64_t G = (K + group - 1) / group;
    const int64_t warps = rows * G;
    if (warps == 0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>((warps * 32 + 255) / 256);
    const int qmax = sym ? (1 << (bits - 1)) - 1 : (1 << bits) - 1;
    if (sym) wq_quant_kernel<true><<<grid, 256, 0, stream>>>(W, K, map, rows, group, G, qmax, f16, codes, scales, zp, err);
    else wq_quant_kernel<false><<<grid, 256, 0, stream>>>(W, K, map, rows, group, G, qmax, f16, codes, scales, zp, err);
    return cudaGetLastError();
}

cudaError_t launch_pack_nibbles(const uint8_t* codes, int64_t rows, int64_t K, uint8_t* payload, cudaStream_t stream) {
    const int64_t n = rows * ((K + 1) / 2);
    if (n == 0) return cudaSuccess;
    wq_pack4_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(codes, rows, K, payload);
    return cudaGetLastError();
}

cudaError_t launch_engine_pack(int32_t T8, int32_t T4, int64_t n8, int64_t n4, int64_t a8, int64_t a4, int32_t G,
                               int64_t K, const uint8_t* payload8, const float* scales8, const uint8_t* payload4,
                               const float* scales4, const uint8_t* zp4, uint8_t* wq, cudaStream_t stream) {
    const int64_t blocks = int64_t(T8 + T4) * G;
    if (blocks == 0) return cudaSuccess;
    wq_engine_kernel<<<static_cast<unsigned>(blocks), 128, 0, stream>>>(T8, n8, n4, a8, a4, G, K, payload8, scales8,
                                                                        payload4, scales4, zp4, wq);
    return cudaGetLastError();
}

cudaError_t launch_meta_check(const float* s8, int64_t n8, const float* s4, int64_t n4, const uint8_t* zp4,
                              int32_t* flags, cudaStream_t stream) {
    if (n8 + n4 == 0) return cudaSuccess;
    wq_check_kernel<<<148, 256, 0, stream>>>(s8, n8, s4, n4, zp4, flags);
    return cudaGetLastError();
}

}  // namespace mq

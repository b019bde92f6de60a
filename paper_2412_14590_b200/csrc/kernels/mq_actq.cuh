// mq_actq.cuh — the K1 per-(token, group) arithmetic of the activation-
// quantization kernels (act_quant.cu). Restates quantize_group_sym<float>
// (proj/include/mixquant/quant.hpp:117-140) bit for bit: see act_quant.cu.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "mq_kernels.hpp"

namespace mq {
namespace actq {

template <int DT>
__device__ __forceinline__ float load_act(const void* A, int64_t i) {
    if constexpr (DT == 0) return __ldg(static_cast<const float*>(A) + i);
    else if constexpr (DT == 1) return __half2float(static_cast<const __half*>(A)[i]);
    else return __bfloat162float(static_cast<const __nv_bfloat16*>(A)[i]);
}

__device__ __forceinline__ float act_scale(float amax, int f16) {
    float s = (amax == 0.0f) ? 1e-8f : __fdiv_rn(amax, 127.0f);
    if (s == 0.0f) s = fmaxf(amax, 1e-8f);
    if (f16) {
        s = __half2float(__float2half_rn(s));
        if (!(s > 0.0f)) s = 5.9604644775390625e-8f;
    }
    return s;
}

__device__ __forceinline__ int8_t quant_one(float x, float s) {
    float q = roundf(__fdiv_rn(x, s));
    q = fminf(fmaxf(q, -127.0f), 127.0f);
    return static_cast<int8_t>(static_cast<int>(q));
}

// 4 consecutive activations (k .. k+3 of one row), zero past K
template <int DT>
__device__ __forceinline__ void load4(const void* A, int64_t base, int64_t k, int64_t K, bool vec, float (&x)[4]) {
    if (vec && k + 3 < K) {
        if constexpr (DT == 0) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(A) + base + k));
            x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
        } else {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(A) + base + k));
            const uint32_t w[2] = {v.x, v.y};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint16_t h = uint16_t(w[i >> 1] >> (16 * (i & 1)));
                if constexpr (DT == 1) x[i] = __half2float(__ushort_as_half(h));
                else x[i] = __bfloat162float(__ushort_as_bfloat16(h));
            }
        }
        return;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = k + i < K ? load_act<DT>(A, base + k + i) : 0.0f;
}

// EAL (mq_kernels.hpp) output of one (token m < Mpad, group g) by one warp:
// lane l owns codes [4l, 4l+4) and stores them as one 32-bit word; lane 0
// writes the group's scale and code sum. Rows m >= M are written as zeros.
template <int DT>
__device__ __forceinline__ void quant_pair_eal(const void* __restrict__ A, int64_t M, int64_t K, int64_t lda, int G,
                                               int64_t Mpad, uint8_t* __restrict__ acts, float* __restrict__ sa,
                                               int32_t* __restrict__ asum, int32_t* err, int64_t m, int g, int lane,
                                               int f16) {
    const int64_t b = int64_t(g) * 128;
    const int len = static_cast<int>(K - b < 128 ? K - b : 128);
    float x[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    float amax = 0.0f;
    bool finite = true;
    if (m < M) {
        const bool vec = (lda % 4 == 0) && ((reinterpret_cast<uintptr_t>(A) & (DT == 0 ? 15 : 7)) == 0);
        load4<DT>(A, m * lda, b + 4 * lane, K, vec, x);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            finite &= isfinite(x[i]);
            amax = fmaxf(amax, fabsf(x[i]));
        }
    }
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    finite = __all_sync(0xffffffffu, finite);
    uint32_t word = 0;
    float s = 0.0f;
    int csum = 0;
    if (m < M) {
        if (!finite && lane == 0 && err) atomicMin(err, static_cast<int32_t>(m * G + g));
        s = act_scale(amax, f16);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (4 * lane + i < len) {
                const int8_t c = quant_one(x[i], s);
                csum += c;
                word |= uint32_t(uint8_t(c)) << (8 * i);
            }
    }
    for (int o = 16; o; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
    *reinterpret_cast<uint32_t*>(acts + int64_t(g) * Mpad * 128 + eal_offset(uint32_t(m), uint32_t(4 * lane))) = word;
    if (lane == 0) {
        sa[int64_t(g) * Mpad + m] = s;
        asum[int64_t(g) * Mpad + m] = csum;  // sum of the group's codes: the zero-point correction term
    }
}

}  // namespace actq
}  // namespace mq

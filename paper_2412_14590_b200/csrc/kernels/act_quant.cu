// act_quant.cu — K1: dynamic symmetric int8 activation quantization.
//
// Restates quantize_group_sym<float> (proj/include/mixquant/quant.hpp:117-140)
// as called by execute_mixed_linear (proj/src/gemm.cpp:190), bit for bit:
//   amax = max|x| (f32), s = amax == 0 ? 1e-8f : amax / 127.0f (IEEE division),
//   s == 0 -> max(amax, 1e-8f), optional f16 rounding (quant.cpp:81-86),
//   code = clamp(roundf(x / s), -127, 127) with IEEE division and
//   round-half-away-from-zero. Non-finite input sets *err to the smallest
//   flat group index m*G+g (the reference throws DataError, quant.hpp:56-64).
// Two launch shapes: a warp per (token, group) for the group-wise parity mode,
// a CTA per token for the per-token mode (group == K). HBM-bound: each element
// is read once (f32/f16/bf16) and written once as int8.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <climits>

#include "mq_actq.cuh"
#include "mq_kernels.hpp"

namespace mq {
namespace {

__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

using namespace actq;

// One warp per (token m, group g); group <= 4096.
template <int DT>
__global__ void act_quant_group_kernel(const void* __restrict__ A, int64_t M, int64_t K,
                                       int64_t lda, int group, int G, int f16,
                                       int8_t* __restrict__ codes, int64_t ldc,
                                       float* __restrict__ scales, int64_t lds, int32_t* err) {
    griddep_launch();  // the dependent GEMM may start its prologue + weight prefetch now
    griddep_wait();    // the previous kernel's outputs (our inputs) are complete
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= M * G) return;
    const int64_t m = wid / G;
    const int g = static_cast<int>(wid - m * G);
    const int64_t b = int64_t(g) * group;
    const int len = static_cast<int>(K - b < group ? K - b : int64_t(group));
    const int64_t base = m * lda + b;

    float amax = 0.0f;
    bool finite = true;
    for (int i = lane; i < len; i += 32) {
        const float x = load_act<DT>(A, base + i);
        finite &= isfinite(x);
        amax = fmaxf(amax, fabsf(x));
    }
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    finite = __all_sync(0xffffffffu, finite);
    if (!finite && lane == 0 && err) atomicMin(err, static_cast<int32_t>(wid));
    const float s = act_scale(amax, f16);
    int8_t* crow = codes + m * ldc + b;
    for (int i = lane; i < len; i += 32) crow[i] = quant_one(load_act<DT>(A, base + i), s);
    if (lane == 0) scales[int64_t(g) * lds + m] = s;  // group-major (TMA-able per group)
    // zero the padding columns [K, ldc) once per row (owned by the last group)
    if (g == G - 1)
        for (int64_t c = K + lane; c < ldc; c += 32) codes[m * ldc + c] = 0;
}

// One CTA per token (per-token mode, group == K).
template <int DT>
__global__ void __launch_bounds__(256) act_quant_row_kernel(
    const void* __restrict__ A, int64_t K, int64_t lda, int f16, int8_t* __restrict__ codes,
    int64_t ldc, float* __restrict__ scales, int32_t* err) {
    griddep_launch();  // the dependent GEMM may start its prologue + weight prefetch now
    griddep_wait();    // the previous kernel's outputs (our inputs) are complete
    __shared__ float red[8];
    __shared__ int bad[8];
    const int64_t m = blockIdx.x;
    const int64_t base = m * lda;
    float amax = 0.0f;
    bool finite = true;
    for (int64_t i = threadIdx.x; i < K; i += blockDim.x) {
        const float x = load_act<DT>(A, base + i);
        finite &= isfinite(x);
        amax = fmaxf(amax, fabsf(x));
    }
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const bool wfin = __all_sync(0xffffffffu, finite);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[w] = amax;
        bad[w] = !wfin;
    }
    __syncthreads();
    amax = red[0];
    int anybad = bad[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
        amax = fmaxf(amax, red[i]);
        anybad |= bad[i];
    }
    if (anybad && threadIdx.x == 0 && err) atomicMin(err, static_cast<int32_t>(m));
    const float s = act_scale(amax, f16);
    for (int64_t i = threadIdx.x; i < K; i += blockDim.x)
        codes[m * ldc + i] = quant_one(load_act<DT>(A, base + i), s);
    for (int64_t c = K + threadIdx.x; c < ldc; c += blockDim.x) codes[m * ldc + c] = 0;
    if (threadIdx.x == 0) scales[m] = s;
}

// ----------------------------------------------------------------------------
// EAL variants (mq_kernels.hpp): the same arithmetic, written straight into the
// engine's tiled, pre-swizzled operand layout so K2 streams each chunk's
// activations with one bulk copy. One warp per (token row m < Mpad, group g):
// lane l owns codes [4l, 4l+4) of the group and stores them as one 32-bit word.
template <int DT>
__global__ void act_quant_eal_group_kernel(const void* __restrict__ A, int64_t M, int64_t K, int64_t lda, int G,
                                           int64_t Mpad, uint8_t* __restrict__ acts, float* __restrict__ sa,
                                           int32_t* __restrict__ asum, int32_t* err, int f16) {
    griddep_launch();  // the dependent GEMM may start its prologue + weight prefetch now
    griddep_wait();    // the previous kernel's outputs (our inputs) are complete
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (wid >= Mpad * G) return;
    const int g = static_cast<int>(wid / Mpad);
    quant_pair_eal<DT>(A, M, K, lda, G, Mpad, acts, sa, asum, err, wid - int64_t(g) * Mpad, g, threadIdx.x & 31, f16);
}

// per-token (group == K): one CTA per token row m < Mpad
// per-token (group == K): one 1024-thread CTA per token row m < Mpad. The row
// is read ONCE into registers (4 values per thread per step, up to RV steps =
// K <= 4096 * RV) with all loads in flight together — a grid-stride loop of
// dependent loads here is latency-bound (~1 us per step).
template <int DT, int RV>
__global__ void __launch_bounds__(1024) act_quant_eal_row_kernel(const void* __restrict__ A, int64_t M, int64_t K,
                                                                 int64_t lda, int G, int64_t Mpad,
                                                                 uint8_t* __restrict__ acts, float* __restrict__ sa,
                                                                 int32_t* __restrict__ asum, int32_t* err, int f16) {
    griddep_launch();  // the dependent GEMM may start its prologue + weight prefetch now
    griddep_wait();    // the previous kernel's outputs (our inputs) are complete
    __shared__ float red[32];
    __shared__ int bad[32];
    const int64_t m = blockIdx.x;
    const bool live = m < M;
    const bool vec = (lda % 4 == 0) && ((reinterpret_cast<uintptr_t>(A) & (DT == 0 ? 15 : 7)) == 0);
    float x[RV][4];
    float amax = 0.0f;
    bool finite = true;
#pragma unroll
    for (int v = 0; v < RV; ++v) {
        const int64_t k = (int64_t(v) * blockDim.x + threadIdx.x) * 4;
        if (live) load4<DT>(A, m * lda, k, K, vec, x[v]);
        else x[v][0] = x[v][1] = x[v][2] = x[v][3] = 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            finite &= isfinite(x[v][i]);
            amax = fmaxf(amax, fabsf(x[v][i]));
        }
    }
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const bool wfin = __all_sync(0xffffffffu, finite);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[w] = amax;
        bad[w] = !wfin;
    }
    __syncthreads();
    amax = red[0];
    int anybad = bad[0];
    for (int i = 1; i < nw; ++i) {
        amax = fmaxf(amax, red[i]);
        anybad |= bad[i];
    }
    if (live && anybad && threadIdx.x == 0 && err) atomicMin(err, static_cast<int32_t>(m));
    const float s = live ? act_scale(amax, f16) : 0.0f;
    // a warp's 32 x 4 codes of step v are exactly one 128-wide group
#pragma unroll
    for (int v = 0; v < RV; ++v) {
        const int64_t k = (int64_t(v) * blockDim.x + threadIdx.x) * 4;
        const int g = static_cast<int>(k >> 7);
        uint32_t word = 0;
        int csum = 0;
        if (live)
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (k + i < K) {
                    const int8_t c = quant_one(x[v][i], s);
                    csum += c;
                    word |= uint32_t(uint8_t(c)) << (8 * i);
                }
        for (int o = 16; o; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
        if (g < G) {
            *reinterpret_cast<uint32_t*>(acts + int64_t(g) * Mpad * 128 + eal_offset(uint32_t(m), uint32_t(k & 127))) = word;
            if ((threadIdx.x & 31) == 0) asum[int64_t(g) * Mpad + m] = csum;
        }
    }
    if (threadIdx.x == 0) sa[m] = s;
}

// row-major codes/scales (reference layout) -> EAL; one thread per 4 codes
__global__ void repack_eal_kernel(const int8_t* __restrict__ codes, int64_t ldc, const float* __restrict__ scales,
                                  int64_t lds, int per_token, int64_t M, int64_t K, int G, int64_t Mpad,
                                  uint8_t* __restrict__ acts, float* __restrict__ sa, int32_t* __restrict__ asum) {
    const int64_t total = int64_t(G) * Mpad * 32;  // a multiple of 32: warps stay aligned to one (g, m)
    const int64_t tend = (total + int64_t(gridDim.x) * blockDim.x - 1) / (int64_t(gridDim.x) * blockDim.x) *
                         (int64_t(gridDim.x) * blockDim.x);
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < tend; i += int64_t(gridDim.x) * blockDim.x) {
        const bool in = i < total;
        const int g = in ? static_cast<int>(i / (Mpad * 32)) : 0;
        const int64_t rem = i - int64_t(g) * Mpad * 32;
        const int64_t m = rem >> 5;
        const int k0 = static_cast<int>(rem & 31) * 4;
        uint32_t word = 0;
        int csum = 0;
        if (in && m < M)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t k = int64_t(g) * 128 + k0 + j;
                if (k < K) {
                    csum += codes[m * ldc + k];
                    word |= uint32_t(uint8_t(codes[m * ldc + k])) << (8 * j);
                }
            }
        for (int o = 16; o; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
        if (!in) continue;
        if (k0 == 0) asum[int64_t(g) * Mpad + m] = csum;
        *reinterpret_cast<uint32_t*>(acts + int64_t(g) * Mpad * 128 + eal_offset(uint32_t(m), uint32_t(k0))) = word;
        if (k0 == 0) {
            if (per_token) {
                if (g == 0) sa[m] = m < M ? scales[m] : 0.0f;
            } else {
                sa[int64_t(g) * Mpad + m] = m < M ? scales[int64_t(g) * lds + m] : 0.0f;
            }
        }
    }
}

template <typename K, typename... Args>
cudaError_t launch_ex(K kern, dim3 grid, dim3 block, bool pdl, cudaStream_t stream, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace

cudaError_t launch_act_quant_eal(const void* A, int a_dtype, int64_t M, int64_t K, int64_t lda, int group,
                                 int64_t Mpad, uint8_t* acts, float* sa, int32_t* asum, int32_t* err, int f16,
                                 bool pdl, cudaStream_t stream) {
    if (Mpad == 0) return cudaSuccess;
    const int G = static_cast<int>((K + 127) / 128);
    if (group >= K) {
        const dim3 grid(static_cast<unsigned>(Mpad));
        const int64_t steps = (K + 4095) / 4096;  // 1024 threads x 4 values per step
        if (steps > 8) return cudaErrorInvalidValue;  // K > 32768: not a Llama shape
#define MQ_ROW(DT, RV) launch_ex(act_quant_eal_row_kernel<DT, RV>, grid, dim3(1024), pdl, stream, A, M, K, lda, G, Mpad, acts, sa, asum, err, f16)
#define MQ_ROWS(DT) (steps <= 1 ? MQ_ROW(DT, 1) : steps <= 2 ? MQ_ROW(DT, 2) : steps <= 4 ? MQ_ROW(DT, 4) : MQ_ROW(DT, 8))
        switch (a_dtype) {
            case 0: return MQ_ROWS(0);
            case 1: return MQ_ROWS(1);
            default: return MQ_ROWS(2);
        }
#undef MQ_ROWS
#undef MQ_ROW
    }
    // 4 warps per CTA: a small footprint, so the CTAs fit beside two decode K2
    // CTAs on an SM (the launch before and the launch after, mixed_gemm_sm100.cu)
    const int64_t warps = Mpad * G;
    const dim3 grid(static_cast<unsigned>((warps * 32 + 127) / 128));
    switch (a_dtype) {
        case 0: return launch_ex(act_quant_eal_group_kernel<0>, grid, dim3(128), pdl, stream, A, M, K, lda, G, Mpad, acts, sa, asum, err, f16);
        case 1: return launch_ex(act_quant_eal_group_kernel<1>, grid, dim3(128), pdl, stream, A, M, K, lda, G, Mpad, acts, sa, asum, err, f16);
        default: return launch_ex(act_quant_eal_group_kernel<2>, grid, dim3(128), pdl, stream, A, M, K, lda, G, Mpad, acts, sa, asum, err, f16);
    }
}

cudaError_t launch_repack_eal(const int8_t* codes, int64_t ldc, const float* scales, int64_t lds, int per_token,
                              int64_t M, int64_t K, int64_t Mpad, uint8_t* acts, float* sa, int32_t* asum,
                              cudaStream_t stream) {
    const int G = static_cast<int>((K + 127) / 128);
    const int64_t total = int64_t(G) * Mpad * 32;
    if (total == 0) return cudaSuccess;
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 8));
    repack_eal_kernel<<<grid, 256, 0, stream>>>(codes, ldc, scales, lds, per_token, M, K, G, Mpad, acts, sa, asum);
    return cudaGetLastError();
}

cudaError_t launch_act_quant(const void* A, int a_dtype, int64_t M, int64_t K, int64_t lda,
                             int group, int f16, int8_t* codes, int64_t ldc, float* scales,
                             int64_t lds, int32_t* err, bool pdl, cudaStream_t stream) {
    if (M == 0) return cudaSuccess;
    if (group >= K) {
        const dim3 grid(static_cast<unsigned>(M));
        switch (a_dtype) {
            case 0: return launch_ex(act_quant_row_kernel<0>, grid, dim3(256), pdl, stream, A, K, lda, f16, codes, ldc, scales, err);
            case 1: return launch_ex(act_quant_row_kernel<1>, grid, dim3(256), pdl, stream, A, K, lda, f16, codes, ldc, scales, err);
            default: return launch_ex(act_quant_row_kernel<2>, grid, dim3(256), pdl, stream, A, K, lda, f16, codes, ldc, scales, err);
        }
    }
    const int G = static_cast<int>((K + group - 1) / group);
    const int64_t warps = M * G;
    const dim3 grid(static_cast<unsigned>((warps * 32 + 255) / 256));
    switch (a_dtype) {
        case 0: return launch_ex(act_quant_group_kernel<0>, grid, dim3(256), pdl, stream, A, M, K, lda, group, G, f16, codes, ldc, scales, lds, err);
        case 1: return launch_ex(act_quant_group_kernel<1>, grid, dim3(256), pdl, stream, A, M, K, lda, group, G, f16, codes, ldc, scales, lds, err);
        default: return launch_ex(act_quant_group_kernel<2>, grid, dim3(256), pdl, stream, A, M, K, lda, group, G, f16, codes, ldc, scales, lds, err);
    }
}

}  // namespace mq

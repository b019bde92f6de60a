// mixed_gemm_sm100.cu — K2: the MixLLM W4/W8-A8 mixed-precision group GEMM on
// 5th-generation tensor cores (tcgen05.mma kind::i8, TMEM accumulators).
//
// Reference semantics (proj/src/gemm.cpp:51-85, the emulated kernel): for every
// output element and every K-group g in ascending order,
//   step 1  S_g = sum_i a[m, i] * (w[r, i] - z[r, g])        (int32, exact)
//   step 2  out += float(S_g) * (s_a[m, g] * s_w[r, g])     (f32 mul, f32 add)
// and the two sub-problems (8-bit / 4-bit output features) are scattered back
// to their original columns (proj/src/mixed.cpp:83-120).
//
// B200 design (one persistent warp-specialised kernel over both sub-problems):
//   warp 0      producer: cp.async.bulk of the packed weight codes + scales
//               (evict-first) and a TMA 2-D tile of the int8 activations
//               (SWIZZLE_128B) into an NS-deep shared-memory ring;
//   warps 4-7   converter (sub4 tiles): nibbles -> int8 (c - z) with the
//               carry-free bias trick ((x & 0x0F0F0F0F) + (128 - z)*0x01010101)
//               ^ 0x80808080 — the paper's step-1 zero-point subtraction
//                — written straight into the UMMA
//               K-major SW128 image; sub8 tiles arrive pre-swizzled and skip it;
//   warp 1      MMA issuer: 4 x tcgen05.mma (K = 32) per group into a fresh
//               int32 TMEM accumulator (double-buffered), tcgen05.commit
//               releases the smem stage and signals the epilogue;
//   warps 8..   epilogue: tcgen05.ld the group sums, exact int->float, rescale
//               and accumulate in f32 registers (step 2), then scatter the
//               tile to the original output columns in f32/f16/bf16.
// Tiles: 128 weight rows (MMA M) x BN tokens (MMA N). Split-K over K-groups
// (MQ_FAST) is reduced deterministically by the last-arriving CTA in fixed
// split order.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "mq_kernels.hpp"
#include "mq_ptx.cuh"

namespace mq {
namespace {

constexpr int kMaxStages = 16;
constexpr int kConvBytes = 16384;

template <int BN>
struct TcCfg {
    static constexpr int kStageA = 16384;
    static constexpr int kStageB = BN * 128;
    static constexpr int kStageMeta = 640;
    static constexpr int kStageBytes = ((kStageA + kStageB + kStageMeta) + 1023) / 1024 * 1024;
    static constexpr uint32_t kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
    static constexpr int NE = BN <= 64 ? 1 : 2;  // epilogue warpgroups
    static constexpr int BNE = BN / NE;          // tokens per epilogue warpgroup
    static constexpr int kThreads = 128 * (2 + NE);
    static constexpr int kFixedSmem = 1024 /*align slack*/ + 2 * kConvBytes + NE * 2 * BNE * 4 + 512;
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <typename T>
__device__ __forceinline__ T to_out(float v);
template <>
__device__ __forceinline__ float to_out<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half to_out<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 to_out<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ void store_out(void* Y, int dt, int64_t idx, float v) {
    if (dt == 0) static_cast<float*>(Y)[idx] = v;
    else if (dt == 1) static_cast<__half*>(Y)[idx] = __float2half_rn(v);
    else static_cast<__nv_bfloat16*>(Y)[idx] = __float2bfloat16_rn(v);
}

struct Unit {
    int tile, tb, g0, g1, ks;
};
__device__ __forceinline__ Unit decode_unit(int u, const GemmParams& p) {
    Unit w;
    w.tile = u % p.num_tiles;
    const int rest = u / p.num_tiles;
    w.tb = rest % p.token_blocks;
    w.ks = rest / p.token_blocks;
    w.g0 = (w.ks * p.G) / p.ksplit;
    w.g1 = ((w.ks + 1) * p.G) / p.ksplit;
    return w;
}

template <int BN, int MODE>
__global__ void __launch_bounds__(TcCfg<BN>::kThreads, 1)
mixed_gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_act, const GemmParams p, int NS) {
    using C = TcCfg<BN>;
    constexpr int NE = C::NE, BNE = C::BNE;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* conv = smem;
    uint8_t* stages = smem + 2 * kConvBytes;
    float* sa_buf = reinterpret_cast<float*>(stages + NS * C::kStageBytes);  // [NE][2][BNE]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sa_buf + NE * 2 * BNE);
    uint64_t* full = bars;
    uint64_t* empty = bars + kMaxStages;
    uint64_t* conv_full = bars + 2 * kMaxStages;
    uint64_t* conv_empty = conv_full + 2;
    uint64_t* tmem_full = conv_empty + 2;
    uint64_t* tmem_empty = tmem_full + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_empty + 2);
    volatile int* last_flag = reinterpret_cast<volatile int*>(tmem_holder + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto stageA = [&](int s) { return stages + s * C::kStageBytes; };
    auto stageB = [&](int s) { return stages + s * C::kStageBytes + C::kStageA; };
    auto stageMeta = [&](int s) { return stages + s * C::kStageBytes + C::kStageA + C::kStageB; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1 + 4 * NE);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&conv_full[i], 4);
            ptx::mbar_init(&conv_empty[i], 1);
            ptx::mbar_init(&tmem_full[i], 1);
            ptx::mbar_init(&tmem_empty[i], 4 * NE);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc<C::kTmemCols>(tmem_holder);
    if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tmap_act);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    const int units = p.num_tiles * p.token_blocks * p.ksplit;

    if (warp == 0) {
        // ============================== producer ==============================
        if (lane == 0) {
            const uint64_t pol_w = ptx::policy_evict_first();
            const uint64_t pol_a = ptx::policy_evict_last();
            uint32_t it = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const Unit w = decode_unit(u, p);
                const TileDesc td = p.tiles[w.tile];
                const int cb = td.is8 ? kCodes8Bytes : kCodes4Bytes;
                const int mb = td.is8 ? kMeta8Bytes : kMeta4Bytes;
                for (int g = w.g0; g < w.g1; ++g, ++it) {
                    const int s = it % NS;
                    const uint32_t ph = (it / NS) & 1;
                    ptx::mbar_wait(&empty[s], ph ^ 1);
                    ptx::mbar_arrive_expect_tx(&full[s], td.copy_bytes + mb + C::kStageB);
                    ptx::bulk_g2s(stageA(s), p.wq + td.codes_off + int64_t(g) * cb, td.copy_bytes, &full[s], pol_w);
                    ptx::bulk_g2s(stageMeta(s), p.wmeta + td.meta_off + int64_t(g) * mb, mb, &full[s], pol_w);
                    ptx::tma_load_2d(stageB(s), &tmap_act, g * kGroupK, w.tb * BN, &full[s], pol_a);
                }
            }
        }
    } else if (warp == 1) {
        // ============================== MMA issuer ============================
        if (lane == 0) {
            const uint32_t idesc4 = ptx::idesc_i8(BN, true, true);
            const uint32_t idesc8 = p.idesc8 | ((uint32_t(BN) >> 3) << 17);
            uint32_t it = 0, cit = 0, ait = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const Unit w = decode_unit(u, p);
                const TileDesc td = p.tiles[w.tile];
                for (int g = w.g0; g < w.g1; ++g, ++it, ++ait) {
                    const int s = it % NS;
                    const uint32_t ph = (it / NS) & 1;
                    const int a = ait & 1;
                    const uint32_t aph = (ait >> 1) & 1;
                    ptx::mbar_wait(&tmem_empty[a], aph ^ 1);
                    ptx::mbar_wait(&full[s], ph);
                    uint32_t a_addr;
                    int c = 0;
                    if (!td.is8) {
                        c = cit & 1;
                        ptx::mbar_wait(&conv_full[c], (cit >> 1) & 1);
                        ++cit;
                        a_addr = ptx::smem_u32(conv + c * kConvBytes);
                    } else {
                        a_addr = ptx::smem_u32(stageA(s));
                    }
                    ptx::tc_fence_after();
                    const uint32_t b_addr = ptx::smem_u32(stageB(s));
                    const uint32_t d_tmem = tmem_base + a * BN;
                    const uint32_t idesc = td.is8 ? idesc8 : idesc4;
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        ptx::mma_i8_ss(d_tmem, ptx::umma_desc_sw128(a_addr + 32 * k),
                                       ptx::umma_desc_sw128(b_addr + 32 * k), idesc, k > 0);
                    ptx::tc_commit(&tmem_full[a]);
                    ptx::tc_commit(&empty[s]);
                    if (!td.is8) ptx::tc_commit(&conv_empty[c]);
                }
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ============================== converter =============================
        const int ct = threadIdx.x - 128;
        uint32_t it = 0, cit = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            const Unit w = decode_unit(u, p);
            const TileDesc td = p.tiles[w.tile];
            if (td.is8) {
                it += w.g1 - w.g0;
                continue;
            }
            for (int g = w.g0; g < w.g1; ++g, ++it, ++cit) {
                const int s = it % NS;
                const int c = cit & 1;
                ptx::mbar_wait(&full[s], (it / NS) & 1);
                ptx::mbar_wait(&conv_empty[c], ((cit >> 1) & 1) ^ 1);
                const uint8_t* raw = stageA(s);
                const uint8_t* zp = stageMeta(s) + 512;
                uint8_t* dst = conv + c * kConvBytes;
#pragma unroll 4
                for (int i = 0; i < 16; ++i) {
                    const int q = i * 128 + ct;
                    const int r = q >> 3, ch = q & 7;
                    if (r < td.rows) {
                        const uint2 wv = *reinterpret_cast<const uint2*>(raw + r * 64 + ch * 8);
                        const uint32_t kk = uint32_t(128 - zp[r]) * 0x01010101u;
                        uint4 o;
                        o.x = ((wv.x & 0x0F0F0F0Fu) + kk) ^ 0x80808080u;
                        o.y = (((wv.x >> 4) & 0x0F0F0F0Fu) + kk) ^ 0x80808080u;
                        o.z = ((wv.y & 0x0F0F0F0Fu) + kk) ^ 0x80808080u;
                        o.w = (((wv.y >> 4) & 0x0F0F0F0Fu) + kk) ^ 0x80808080u;
                        *reinterpret_cast<uint4*>(dst + (r >> 3) * 1024 + (r & 7) * 128 + ((ch ^ (r & 7)) << 4)) = o;
                    }
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&conv_full[c]);
            }
        }
    } else if (warp >= 8) {
        // ============================== epilogue ==============================
        const int et = threadIdx.x - 256;  // 0 .. 128*NE-1
        const int e = et >> 7;             // epilogue warpgroup
        const int lt = et & 127;           // thread within the warpgroup
        const int wq = warp & 3;           // TMEM lane quarter this warp may access
        const int r = wq * 32 + lane;      // tile row (= TMEM lane)
        const int c0 = e * BNE;            // first token column of this warpgroup
        float* my_sa = sa_buf + e * 2 * BNE;
        uint32_t it = 0, ait = 0, jg = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            const Unit w = decode_unit(u, p);
            const TileDesc td = p.tiles[w.tile];
            const int64_t m0 = int64_t(w.tb) * BN + c0;  // first token of this warpgroup
            float acc[BNE];
#pragma unroll
            for (int j = 0; j < BNE; ++j) acc[j] = 0.0f;
            float sa_next = 0.0f;
            if constexpr (MODE == kExactGroup || MODE == kFastGroup) {
                if (lt < BNE && m0 + lt < p.M) sa_next = __ldg(p.sa + (m0 + lt) * p.sa_cols + (p.sa_cols == 1 ? 0 : w.g0));
            }
            for (int g = w.g0; g < w.g1; ++g, ++it, ++ait, ++jg) {
                const int s = it % NS;
                const int a = ait & 1;
                if constexpr (MODE == kExactGroup || MODE == kFastGroup) {
                    if (lt < BNE) my_sa[(jg & 1) * BNE + lt] = sa_next;
                    named_bar_sync(1 + e, 128);
                    if (lt < BNE && g + 1 < w.g1 && m0 + lt < p.M)
                        sa_next = __ldg(p.sa + (m0 + lt) * p.sa_cols + (p.sa_cols == 1 ? 0 : g + 1));
                }
                ptx::mbar_wait(&full[s], (it / NS) & 1);
                const float sw = reinterpret_cast<const float*>(stageMeta(s))[r];
                ptx::mbar_wait(&tmem_full[a], (ait >> 1) & 1);
                ptx::tc_fence_after();
                const float* sav = my_sa + (jg & 1) * BNE;
#pragma unroll
                for (int ch = 0; ch < BNE / 16; ++ch) {
                    uint32_t v[16];
                    ptx::tmem_ld16(tmem_base + (uint32_t(wq * 32) << 16) + uint32_t(a * BN + c0 + ch * 16), v);
                    ptx::tmem_wait_ld();
                    if constexpr (MODE == kDumpPartials) {
                        if (r < td.rows) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                const int64_t m = m0 + ch * 16 + j;
                                if (m < p.M)
                                    p.partials[(int64_t(g) * p.M + m) * p.partial_rows + td.sub_row0 + r] = int32_t(v[j]);
                            }
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const float gs = __int2float_rn(int32_t(v[j]));  // exact: |S| < 2^22
                            const int jj = ch * 16 + j;
                            if constexpr (MODE == kExactGroup) {
                                // gemm.cpp:81 — out += gs * (s_a * s_w), no contraction
                                acc[jj] = __fadd_rn(acc[jj], __fmul_rn(gs, __fmul_rn(sav[jj], sw)));
                            } else if constexpr (MODE == kFastGroup) {
                                acc[jj] = __fmaf_rn(gs, __fmul_rn(sav[jj], sw), acc[jj]);
                            } else {
                                acc[jj] = __fmaf_rn(gs, sw, acc[jj]);
                            }
                        }
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(&tmem_empty[a]);
                    ptx::mbar_arrive(&empty[s]);
                }
            }
            if constexpr (MODE == kDumpPartials) continue;

            const bool row_ok = r < td.rows;
            const int col = row_ok ? __ldg(p.colmap + td.colmap_off + r) : -1;
            bool do_store = true;
            if (p.ksplit > 1) {
                // deterministic split-K: publish this split's partial tile,
                // the last arriving CTA sums splits 0..S-1 in order.
                const int64_t tile_slot = int64_t(w.tile) * p.token_blocks + w.tb;
                float* part = p.ws + ((tile_slot * p.ksplit + w.ks) * 128 + r) * BN + c0;
#pragma unroll
                for (int j = 0; j < BNE; j += 4)
                    __stcg(reinterpret_cast<float4*>(part + j), make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]));
                __threadfence();
                named_bar_sync(3, 128 * NE);
                if (et == 0) {
                    const uint32_t prev = atomicAdd(p.counters + tile_slot, 1u);
                    *last_flag = (prev == uint32_t(p.ksplit - 1));
                }
                named_bar_sync(3, 128 * NE);
                do_store = *last_flag != 0;
                if (do_store) {
                    __threadfence();
                    const float* base = p.ws + (tile_slot * p.ksplit * 128 + r) * BN + c0;
#pragma unroll
                    for (int j = 0; j < BNE; j += 4) {
                        float4 t = __ldcg(reinterpret_cast<const float4*>(base + j));
                        acc[j] = t.x; acc[j + 1] = t.y; acc[j + 2] = t.z; acc[j + 3] = t.w;
                    }
                    for (int ks = 1; ks < p.ksplit; ++ks) {
                        const float* b2 = base + int64_t(ks) * 128 * BN;
#pragma unroll
                        for (int j = 0; j < BNE; j += 4) {
                            float4 t = __ldcg(reinterpret_cast<const float4*>(b2 + j));
                            acc[j] = __fadd_rn(acc[j], t.x);
                            acc[j + 1] = __fadd_rn(acc[j + 1], t.y);
                            acc[j + 2] = __fadd_rn(acc[j + 2], t.z);
                            acc[j + 3] = __fadd_rn(acc[j + 3], t.w);
                        }
                    }
                    if (et == 0) p.counters[tile_slot] = 0u;  // re-arm for the next launch
                }
            }
            if (do_store && row_ok) {
#pragma unroll
                for (int j = 0; j < BNE; ++j) {
                    const int64_t m = m0 + j;
                    if (m < p.M) {
                        float v = acc[j];
                        if constexpr (MODE == kFastToken) v = __fmul_rn(v, __ldg(p.sa + m));
                        store_out(p.Y, p.out_dtype, m * p.ldy + col, v);
                    }
                }
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}

template <int BN, int MODE>
cudaError_t launch_bn_mode(const GemmParams& p, const void* tmap, int num_sms, cudaStream_t stream) {
    using C = TcCfg<BN>;
    int NS = (227 * 1024 - C::kFixedSmem) / C::kStageBytes;
    NS = NS > kMaxStages ? kMaxStages : NS;
    const size_t smem = C::kFixedSmem + size_t(NS) * C::kStageBytes;
    auto kern = mixed_gemm_tc_kernel<BN, MODE>;
    static thread_local uint64_t configured = 0;  // per device ordinal bitmask
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(configured >> dev & 1)) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        configured |= uint64_t(1) << dev;
    }
    const int units = p.num_tiles * p.token_blocks * p.ksplit;
    const int grid = units < num_sms ? units : num_sms;
    if (grid <= 0) return cudaSuccess;
    kern<<<grid, C::kThreads, smem, stream>>>(*static_cast<const CUtensorMap*>(tmap), p, NS);
    return cudaGetLastError();
}

template <int BN>
cudaError_t launch_bn(const GemmParams& p, const void* tmap, int mode, int num_sms, cudaStream_t s) {
    switch (mode) {
        case kExactGroup: return launch_bn_mode<BN, kExactGroup>(p, tmap, num_sms, s);
        case kFastGroup: return launch_bn_mode<BN, kFastGroup>(p, tmap, num_sms, s);
        case kFastToken: return launch_bn_mode<BN, kFastToken>(p, tmap, num_sms, s);
        default: return launch_bn_mode<BN, kDumpPartials>(p, tmap, num_sms, s);
    }
}

}  // namespace

size_t gemm_smem_bytes(int bn, int* stages) {
    auto calc = [&](int fixed, int stage) {
        int ns = (227 * 1024 - fixed) / stage;
        ns = ns > kMaxStages ? kMaxStages : ns;
        if (stages) *stages = ns;
        return size_t(fixed) + size_t(ns) * stage;
    };
    switch (bn) {
        case 16: return calc(TcCfg<16>::kFixedSmem, TcCfg<16>::kStageBytes);
        case 32: return calc(TcCfg<32>::kFixedSmem, TcCfg<32>::kStageBytes);
        case 64: return calc(TcCfg<64>::kFixedSmem, TcCfg<64>::kStageBytes);
        default: return calc(TcCfg<128>::kFixedSmem, TcCfg<128>::kStageBytes);
    }
}

cudaError_t launch_mixed_gemm_tc(const GemmParams& p, const void* tmap, int token_tile, int mode,
                                 int num_sms, cudaStream_t stream) {
    switch (token_tile) {
        case 16: return launch_bn<16>(p, tmap, mode, num_sms, stream);
        case 32: return launch_bn<32>(p, tmap, mode, num_sms, stream);
        case 64: return launch_bn<64>(p, tmap, mode, num_sms, stream);
        case 128: return launch_bn<128>(p, tmap, mode, num_sms, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace mq

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
// B200 design: one persistent warp-specialised kernel over both sub-problems;
// each CTA owns an arithmetically derived stream-K range of (tile, token
// block, K-group) work (mq_kernels.hpp: Schedule), so the first weight copy
// issues right after barrier init with no dependent global loads:
//   warp 0      producer: cp.async.bulk of the packed weight codes + scales
//               (L2 evict-first) — the first NS stages BEFORE
//               griddepcontrol.wait so weight streaming overlaps the previous
//               kernel under PDL — then a TMA 2-D tile of the int8 activations
//               (SWIZZLE_128B) and the group's activation scales, NS-deep ring;
//   warps 4-7   converter (sub4 tiles), IN PLACE in the stage: nibbles -> int8
//               (c - z) with the carry-free bias trick
//               ((x & 0x0F0F0F0F) + (128 - z)*0x01010101) ^ 0x80808080 — the
//               paper's step-1 zero-point subtraction —
//               written as the UMMA K-major SW128 image; sub8 tiles arrive
//               pre-swizzled and skip it;
//   warp 1      TMEM allocation, then MMA issue: 4 x tcgen05.mma (K = 32) per
//               group into a fresh int32 TMEM accumulator (NACC-deep ring);
//               tcgen05.commit releases the stage and signals the epilogue;
//   warps 8..   epilogue: tcgen05.ld the group sums, exact int->float
//               (I2FP), rescale and accumulate in f32 registers (step 2), then
//               scatter the tile to the original output columns (f32/f16/bf16)
//               or publish a stream-K partial (last arriver reduces in order).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "mq_kernels.hpp"
#include "mq_ptx.cuh"

namespace mq {
namespace {

constexpr int kSmemMax = 232448;  // 227 KB opt-in dynamic shared memory per CTA

template <int BN>
struct TcCfg {
    static constexpr int kStageA = 16384;
    static constexpr int kStageB = BN * 128;
    static constexpr int kStageMeta = 640;
    static constexpr int kStageSa = BN * 4;
    static constexpr int kOffB = kStageA;
    static constexpr int kOffMeta = kStageA + kStageB;
    static constexpr int kOffSa = kOffMeta + kStageMeta;
    static constexpr int kStageBytes = ((kOffSa + kStageSa) + 1023) / 1024 * 1024;
    static constexpr int kFixed = 1024 /*alignment slack*/ + 1024 /*barriers*/;
    static constexpr int NS0 = (kSmemMax - kFixed) / kStageBytes;
    static constexpr int NS = NS0 > 16 ? 16 : NS0;
    static constexpr int NACC = BN <= 32 ? 8 : 4;  // TMEM accumulator ring
    static constexpr uint32_t kTmemCols = (NACC * BN <= 32) ? 32 : (NACC * BN <= 64) ? 64 : (NACC * BN <= 128) ? 128 : (NACC * BN <= 256) ? 256 : 512;
    static constexpr int NE = BN <= 64 ? 1 : 2;  // epilogue warpgroups
    static constexpr int BNE = BN / NE;          // tokens per epilogue warpgroup
    static constexpr int kThreads = 128 * (2 + NE);
    static constexpr int kSmem = kFixed + NS * kStageBytes;
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void store_out(void* Y, int dt, int64_t idx, float v) {
    if (dt == 0) static_cast<float*>(Y)[idx] = v;
    else if (dt == 1) static_cast<__half*>(Y)[idx] = __float2half_rn(v);
    else static_cast<__nv_bfloat16*>(Y)[idx] = __float2bfloat16_rn(v);
}

// ring position: stage index + phase parity, advanced per group
struct Ring {
    int idx = 0;
    uint32_t ph = 0;
    template <int N>
    __device__ __forceinline__ void next() {
        if (++idx == N) {
            idx = 0;
            ph ^= 1u;
        }
    }
};

// One contiguous run of K-groups of one work item inside this CTA's range.
struct Seg {
    int64_t x0;  // linear index of the first group
    int64_t item;
    int tile, tb, g0, g1;
};
__device__ __forceinline__ Seg seg_at(const GemmParams& p, int64_t x, int64_t xe) {
    Seg s;
    s.x0 = x;
    s.item = x / p.G;
    s.g0 = int(x - s.item * p.G);
    const int64_t end = (s.item + 1) * p.G;
    s.g1 = s.g0 + int((end < xe ? end : xe) - x);
    s.tile = int(s.item / p.TB);
    s.tb = int(s.item - int64_t(s.tile) * p.TB);
    return s;
}

template <int BN, int MODE>
__global__ void __launch_bounds__(TcCfg<BN>::kThreads, 1)
mixed_gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_act, const GemmParams p) {
    using C = TcCfg<BN>;
    constexpr int NS = C::NS, NACC = C::NACC, NE = C::NE, BNE = C::BNE;
    extern __shared__ uint8_t smem_raw[];
    // 1024-B aligned base (SWIZZLE_128B atoms), derived from smem_raw so the
    // compiler keeps shared-space provenance (LDS/STS, not generic LD/ST)
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* stages = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(stages + NS * C::kStageBytes);
    uint64_t* full = bars;                 // [NS] producer (expect_tx)
    uint64_t* conv = full + NS;            // [NS] converter -> MMA
    uint64_t* empty = conv + NS;           // [NS] MMA commit + epilogue warps
    uint64_t* tfull = empty + NS;          // [NACC] MMA commit -> epilogue
    uint64_t* tempty = tfull + NACC;       // [NACC] epilogue -> MMA
    uint64_t* tmem_ready = tempty + NACC;  // warp 1 -> epilogue
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_ready + 1);
    int* last_flag = reinterpret_cast<int*>(tmem_holder + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto stage = [&](int s) { return stages + s * C::kStageBytes; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&conv[s], 4);
            ptx::mbar_init(&empty[s], 1 + 4 * NE);
        }
        for (int i = 0; i < NACC; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 4 * NE);
        }
        ptx::mbar_init(tmem_ready, 1);
        ptx::fence_barrier_init();
    }
    __syncthreads();
    griddep_launch();  // let the next kernel in the stream start its prologue

    const Schedule S(p);
    const int64_t xb = S.cut(blockIdx.x), xe = S.cut(blockIdx.x + 1);

    if (warp == 0) {
        // ============================== producer ==============================
        if (lane == 0) {
            ptx::prefetch_tmap(&tmap_act);
            const uint64_t pol_w = ptx::policy_evict_first();
            const uint64_t pol_a = ptx::policy_evict_last();
            constexpr bool kSa = (MODE == kExactGroup || MODE == kFastGroup);
            const uint32_t b_bytes = (p.dbg & 8) ? 0u : uint32_t(C::kStageB);
            // pass 0: weights of the first NS groups (independent of the
            // previous kernel); pass 1: activations/scales + the rest.
            for (int pass = 0; pass < 2; ++pass) {
                if (pass == 1) griddep_wait();
                Ring rr;
                int n = 0;
                for (int64_t x = xb; x < xe && !(pass == 0 && n >= NS);) {
                    const Seg sg = seg_at(p, x, xe);
                    x += sg.g1 - sg.g0;
                    const TileInfo ti = tile_info(p, sg.tile);
                    const int cb = ti.is8 ? kCodes8Bytes : kCodes4Bytes;
                    const int mb = ti.is8 ? kMeta8Bytes : kMeta4Bytes;
                    const int64_t m0 = int64_t(sg.tb) * BN;
                    const int64_t mrem = p.M - m0;
                    const uint32_t sa_bytes = kSa && !(p.dbg & 8) ? uint32_t(((mrem < BN ? mrem : BN) + 3) / 4 * 16) : 0u;
                    for (int g = sg.g0; g < sg.g1; ++g, ++n) {
                        const bool pre = n < NS;
                        if (pass == 0 && !pre) break;
                        const int s = (pass == 0) ? n : rr.idx;
                        uint8_t* st = stage(s);
                        if (pass == 0 || !pre) {
                            if (pass == 1) ptx::mbar_wait(&empty[s], rr.ph ^ 1u);
                            ptx::mbar_arrive_expect_tx(&full[s], ti.copy_bytes + mb + b_bytes + sa_bytes);
                            ptx::bulk_g2s(st, p.wq + ti.codes_off + int64_t(g) * cb, ti.copy_bytes, &full[s], pol_w);
                            ptx::bulk_g2s(st + C::kOffMeta, p.wmeta + ti.meta_off + int64_t(g) * mb, mb, &full[s], pol_w);
                        }
                        if (pass == 1) {
                            if (b_bytes) ptx::tma_load_2d(st + C::kOffB, &tmap_act, g * kGroupK, int32_t(m0), &full[s], pol_a);
                            if (sa_bytes)
                                ptx::bulk_g2s(st + C::kOffSa, p.sa + int64_t(g) * p.sa_gstride + m0, sa_bytes, &full[s], pol_a);
                            rr.next<NS>();
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ======================= TMEM allocation + MMA issuer ==================
        ptx::tmem_alloc<C::kTmemCols>(tmem_holder);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            ptx::mbar_arrive(tmem_ready);
            ptx::tc_fence_after();
            const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_holder);
            const uint32_t idesc4 = idesc_i8(BN, true, true);
            const uint32_t idesc8 = p.idesc8 | ((uint32_t(BN) >> 3) << 17);
            Ring rs, ra;
            for (int64_t x = xb; x < xe;) {
                const Seg sg = seg_at(p, x, xe);
                x += sg.g1 - sg.g0;
                const bool is8 = sg.tile < p.T8;
                const uint32_t idesc = is8 ? idesc8 : idesc4;
                for (int g = sg.g0; g < sg.g1; ++g) {
                    ptx::mbar_wait(&tempty[ra.idx], ra.ph ^ 1u);
                    ptx::mbar_wait(&full[rs.idx], rs.ph);
                    if (!is8) ptx::mbar_wait(&conv[rs.idx], rs.ph);
                    ptx::tc_fence_after();
                    const uint32_t a_addr = ptx::smem_u32(stage(rs.idx));
                    const uint32_t b_addr = a_addr + C::kOffB;
                    const uint32_t d_tmem = tmem_base + uint32_t(ra.idx * BN);
                    if (!(p.dbg & 4)) {
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            ptx::mma_i8_ss(d_tmem, ptx::umma_desc_sw128(a_addr + 32 * k),
                                           ptx::umma_desc_sw128(b_addr + 32 * k), idesc, k > 0);
                    }
                    ptx::tc_commit(&tfull[ra.idx]);
                    ptx::tc_commit(&empty[rs.idx]);
                    rs.next<NS>();
                    ra.next<NACC>();
                }
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ====================== converter (in place, sub4) ====================
        const int ct = threadIdx.x - 128;
        Ring rs;
        for (int64_t x = xb; x < xe;) {
            const Seg sg = seg_at(p, x, xe);
            x += sg.g1 - sg.g0;
            const bool is8 = sg.tile < p.T8;
            for (int g = sg.g0; g < sg.g1; ++g, rs.next<NS>()) {
                ptx::mbar_wait(&full[rs.idx], rs.ph);
                if (is8 || (p.dbg & 2)) {
                    // keep conv[s] in lock-step with the ring (one phase per use
                    // of the stage) even though sub8 stages need no conversion
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&conv[rs.idx]);
                    continue;
                }
                uint8_t* st = stage(rs.idx);
                const uint8_t* zp = st + C::kOffMeta + 512;
                // 128 rows x 8 chunks of 16 codes = 1024 chunks: 8 per converter thread
                uint2 w[8];
                uint32_t kk[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int q = i * 128 + ct, r = q >> 3, ch = q & 7;
                    w[i] = *reinterpret_cast<const uint2*>(st + r * 64 + ch * 8);
                    kk[i] = uint32_t(128 - zp[r]) * 0x01010101u;
                }
                named_bar_sync(4, 128);  // every raw byte read before any int8 byte lands
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int q = i * 128 + ct, r = q >> 3, ch = q & 7;
                    uint4 o;
                    o.x = ((w[i].x & 0x0F0F0F0Fu) + kk[i]) ^ 0x80808080u;
                    o.y = (((w[i].x >> 4) & 0x0F0F0F0Fu) + kk[i]) ^ 0x80808080u;
                    o.z = ((w[i].y & 0x0F0F0F0Fu) + kk[i]) ^ 0x80808080u;
                    o.w = (((w[i].y >> 4) & 0x0F0F0F0Fu) + kk[i]) ^ 0x80808080u;
                    *reinterpret_cast<uint4*>(st + (r >> 3) * 1024 + (r & 7) * 128 + ((ch ^ (r & 7)) << 4)) = o;
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&conv[rs.idx]);
            }
        }
    } else if (warp >= 8) {
        // ============================== epilogue ==============================
        const int et = threadIdx.x - 256;  // 0 .. 128*NE-1
        const int e = et >> 7;             // epilogue warpgroup
        const int wq = warp & 3;           // TMEM lane quarter this warp may access
        const int r = wq * 32 + lane;      // tile row (= TMEM lane)
        const int c0 = e * BNE;            // first token column of this warpgroup
        ptx::mbar_wait(tmem_ready, 0);
        ptx::tc_fence_after();
        const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_holder);
        griddep_wait();  // workspace / scales / output of this launch are ours now
        Ring rs, ra;
        for (int64_t x = xb; x < xe;) {
            const Seg sg = seg_at(p, x, xe);
            x += sg.g1 - sg.g0;
            const TileInfo ti = tile_info(p, sg.tile);
            const int col = r < ti.rows ? __ldg(p.colmap + sg.tile * kTileRows + r) : -1;  // prefetch
            const int64_t m0 = int64_t(sg.tb) * BN + c0;  // first token of this warpgroup
            float acc[BNE];
#pragma unroll
            for (int j = 0; j < BNE; ++j) acc[j] = 0.0f;
            for (int g = sg.g0; g < sg.g1; ++g) {
                ptx::mbar_wait(&full[rs.idx], rs.ph);
                const uint8_t* st = stage(rs.idx);
                const float sw = reinterpret_cast<const float*>(st + C::kOffMeta)[r];
                const float* sav = reinterpret_cast<const float*>(st + C::kOffSa) + c0;
                ptx::mbar_wait(&tfull[ra.idx], ra.ph);
                ptx::tc_fence_after();
#pragma unroll
                for (int ch = 0; ch < BNE / 16; ++ch) {
                    if (p.dbg & 1) break;
                    uint32_t v[16];
                    ptx::tmem_ld16(tmem_base + (uint32_t(wq * 32) << 16) + uint32_t(ra.idx * BN + c0 + ch * 16), v);
                    ptx::tmem_wait_ld();
                    if constexpr (MODE == kDumpPartials) {
                        if (r < ti.rows) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                const int64_t m = m0 + ch * 16 + j;
                                if (m < p.M)
                                    p.partials[(int64_t(g) * p.M + m) * p.partial_rows + ti.first + r] = int32_t(v[j]);
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
                    ptx::mbar_arrive(&tempty[ra.idx]);
                    ptx::mbar_arrive(&empty[rs.idx]);
                }
                rs.next<NS>();
                ra.next<NACC>();
            }
            if constexpr (MODE == kDumpPartials) continue;

            bool do_store = true;
            const int64_t xs = sg.item * p.G;  // the item's linear group range [xs, xs + G)
            if (p.split && !(xb <= xs && xe >= xs + p.G)) {
                // stream-K: this CTA holds only part of the item. Publish the
                // partial tile to slot 2*c + (first segment of this CTA ? 0 : 1);
                // the last arriving CTA sums the item's partials in CTA order.
                const int c = blockIdx.x;
                const int slot = 2 * c + (sg.x0 == xb ? 0 : 1);
                float* part = p.ws + (int64_t(slot) * 128 + r) * BN + c0;
#pragma unroll
                for (int j = 0; j < BNE; j += 4)
                    __stcg(reinterpret_cast<float4*>(part + j), make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]));
                __threadfence();
                named_bar_sync(3, 128 * NE);
                const int ca = S.cta_of(xs), cz = S.cta_of(xs + p.G - 1);
                if (et == 0) {
                    const uint32_t prev = atomicAdd(p.counters + sg.item, 1u);
                    *reinterpret_cast<volatile int*>(last_flag) = (prev == uint32_t(cz - ca));
                }
                named_bar_sync(3, 128 * NE);
                do_store = *reinterpret_cast<volatile int*>(last_flag) != 0;
                if (do_store) {
                    __threadfence();
                    const bool ca_first = S.cut(ca) == xs;
                    for (int k = ca; k <= cz; ++k) {
                        const int sk = 2 * k + ((k == ca && !ca_first) ? 1 : 0);
                        const float* src = p.ws + (int64_t(sk) * 128 + r) * BN + c0;
#pragma unroll
                        for (int j = 0; j < BNE; j += 4) {
                            const float4 t = __ldcg(reinterpret_cast<const float4*>(src + j));
                            if (k == ca) {
                                acc[j] = t.x; acc[j + 1] = t.y; acc[j + 2] = t.z; acc[j + 3] = t.w;
                            } else {
                                acc[j] = __fadd_rn(acc[j], t.x);
                                acc[j + 1] = __fadd_rn(acc[j + 1], t.y);
                                acc[j + 2] = __fadd_rn(acc[j + 2], t.z);
                                acc[j + 3] = __fadd_rn(acc[j + 3], t.w);
                            }
                        }
                    }
                    if (et == 0) p.counters[sg.item] = 0u;  // re-arm for the next launch
                }
            }
            if (do_store && col >= 0) {
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
        ptx::tmem_dealloc<C::kTmemCols>(*reinterpret_cast<volatile uint32_t*>(tmem_holder));
    }
}

template <int BN, int MODE>
cudaError_t launch_bn_mode(const GemmParams& p, const void* tmap, bool pdl, cudaStream_t stream) {
    using C = TcCfg<BN>;
    auto kern = mixed_gemm_tc_kernel<BN, MODE>;
    static thread_local uint64_t configured = 0;  // per device ordinal bitmask
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(configured >> dev & 1)) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        if (e != cudaSuccess) return e;
        configured |= uint64_t(1) << dev;
    }
    if (p.P <= 0) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.P);
    cfg.blockDim = dim3(C::kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, *static_cast<const CUtensorMap*>(tmap), p);
}

template <int BN>
cudaError_t launch_bn(const GemmParams& p, const void* tmap, int mode, bool pdl, cudaStream_t s) {
    switch (mode) {
        case kExactGroup: return launch_bn_mode<BN, kExactGroup>(p, tmap, pdl, s);
        case kFastGroup: return launch_bn_mode<BN, kFastGroup>(p, tmap, pdl, s);
        case kFastToken: return launch_bn_mode<BN, kFastToken>(p, tmap, pdl, s);
        default: return launch_bn_mode<BN, kDumpPartials>(p, tmap, pdl, s);
    }
}

}  // namespace

int gemm_stages(int bn) {
    switch (bn) {
        case 16: return TcCfg<16>::NS;
        case 32: return TcCfg<32>::NS;
        case 64: return TcCfg<64>::NS;
        default: return TcCfg<128>::NS;
    }
}

cudaError_t launch_mixed_gemm_tc(const GemmParams& p, const void* tmap, int token_tile, int mode, bool pdl,
                                 cudaStream_t stream) {
    switch (token_tile) {
        case 16: return launch_bn<16>(p, tmap, mode, pdl, stream);
        case 32: return launch_bn<32>(p, tmap, mode, pdl, stream);
        case 64: return launch_bn<64>(p, tmap, mode, pdl, stream);
        case 128: return launch_bn<128>(p, tmap, mode, pdl, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace mq

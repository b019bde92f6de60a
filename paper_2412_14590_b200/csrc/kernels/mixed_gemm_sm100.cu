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
// CTA c owns the stream-K range [cuts[c], cuts[c+1]) of linearised
// (tile, token block, K-group) work (mq_kernels.hpp). Work moves in CHUNKS of
// up to GPS consecutive groups of one tile (GPS/2 for sub8); every hand-off
// between roles is per chunk, not per group (mbarrier round trips dominate
// at decode sizes):
//   warp 0      producer: per chunk one cp.async.bulk of the merged code+meta
//               blocks (L2 evict-first), one 3-D TMA of the chunk's int8
//               activation tiles (SWIZZLE_128B), one 2-D TMA of its activation
//               scales; the first NS weight copies issue BEFORE
//               griddepcontrol.wait so under PDL they overlap the previous kernel;
//   converter   (sub4) one thread per weight row: 4 conflict-free 16-B loads,
//               nibbles -> int8 (c - z) with the carry-free bias trick
//               ((x & 0x0F0F0F0F) + (128 - z)*0x01010101) ^ 0x80808080 — the
//               paper's step-1 zero-point subtraction — and a
//               tcgen05.st of the row straight into a TMEM A-operand ring;
//   warp 1      TMEM allocation, then MMA issue (elected lane): 4 x tcgen05.mma
//               (K = 32) per group, A from TMEM (sub4) or from the
//               pre-swizzled SMEM block (sub8), each group into a fresh int32
//               TMEM accumulator;
//   epilogue    tcgen05.ld the group sums, exact int->float (I2FP), rescale and
//               accumulate in f32 registers (step 2), then scatter the tile to
//               the original output columns (f32/f16/bf16) or publish a
//               stream-K partial (last arriver reduces in fixed order).
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
    static constexpr int GPS = gemm_gps(BN);                // sub4 groups per chunk
    static constexpr int GPS8 = GPS / 2 > 0 ? GPS / 2 : 1;  // sub8 groups per chunk
    static constexpr int kRaw0 = GPS * kBlock4Bytes > GPS8 * kBlock8Bytes ? GPS * kBlock4Bytes : GPS8 * kBlock8Bytes;
    static constexpr int kRaw = (kRaw0 + 1023) / 1024 * 1024;
    static constexpr int kOffB = kRaw;                     // [GPS][BN][128] int8, SW128
    static constexpr int kOffSa = kOffB + GPS * BN * 128;  // [GPS][BN] f32
    static constexpr int kStageBytes = ((kOffSa + GPS * BN * 4) + 1023) / 1024 * 1024;
    // TMEM rings (512 columns): NT accumulator chunk slots of GPS x BN int32
    // columns, NA A-operand chunk slots of GPS x 32 columns (128 int8 K per row).
    static constexpr uint32_t kAccPerChunk = GPS * BN, kAPerChunk = GPS * 32;
    static constexpr int NT = BN >= 128 ? 3 : 2;
    static constexpr int NA = int((512u - NT * kAccPerChunk) / kAPerChunk) > 4 ? 4 : int((512u - NT * kAccPerChunk) / kAPerChunk);
    static constexpr uint32_t kAccCols = NT * kAccPerChunk;
    static constexpr uint32_t kACol0 = kAccCols;
    static constexpr uint32_t kTmemNeed = kAccCols + NA * kAPerChunk;
    static constexpr uint32_t kTmemCols = kTmemNeed <= 32 ? 32 : kTmemNeed <= 64 ? 64 : kTmemNeed <= 128 ? 128 : kTmemNeed <= 256 ? 256 : 512;
    static_assert(kTmemNeed <= 512 && NA >= 2, "TMEM budget");
    // meta ring (per accumulator slot): weight scales [GPS][128] + act scales [GPS][BN],
    // copied out of the stage by the converter so stages free up before the epilogue runs
    static constexpr int kMetaSlot = GPS * (128 + BN) * 4;
    static constexpr int kMetaBytes = NT * kMetaSlot;
    static constexpr int kFixed = 1024 /*alignment slack*/ + 1024 /*barriers*/ + kMetaBytes;
    static constexpr int NS0 = (kSmemMax - kFixed) / kStageBytes;
#ifndef MQ_NS_MAX
#define MQ_NS_MAX 8
#endif
    static constexpr int NS = NS0 > MQ_NS_MAX ? MQ_NS_MAX : NS0;
    static constexpr int NE = BN <= 64 ? 1 : 2;  // epilogue warpgroups
    static constexpr int NC = BN <= 32 ? 2 : 1;  // converter warpgroups (decode is conversion-bound)
    static constexpr int BNE = BN / NE;          // tokens per epilogue warpgroup
    static constexpr int kEpiThread0 = 128 * (1 + NC);
    static constexpr int kThreads = 128 * (1 + NC + NE);
    static constexpr int kSmem = kFixed + NS * kStageBytes;
    static_assert(NS >= 2, "pipeline needs at least two stages");
    static_assert(GPS * BN <= 128, "act-scale copy: one converter thread per value");
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// one lane of a converged warp (elect.sync): keeps tcgen05/TMA operands warp-uniform
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void trace(const GemmParams& p, int ev) {
    if (p.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[blockIdx.x * 8 + ev] = t;
    }
}
// per-chunk event trace of one CTA (MQ_DBG & 64, CTA = MQ_DBG >> 8), in SM cycles
__device__ __forceinline__ void trace_chunk(const GemmParams& p, int ev, int n) {
    if (p.trace && (p.dbg & 64) && int(blockIdx.x) == (p.dbg >> 8) && n < 64)
        p.trace[148 * 8 + ev * 64 + n] = clock64();
}

__device__ __forceinline__ void store_out(void* Y, int dt, int64_t idx, float v) {
    if (dt == 0) static_cast<float*>(Y)[idx] = v;
    else if (dt == 1) static_cast<__half*>(Y)[idx] = __float2half_rn(v);
    else static_cast<__nv_bfloat16*>(Y)[idx] = __float2bfloat16_rn(v);
}

// ring position: slot index + phase parity
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
    int32_t x0;  // linear index of the first group
    int32_t item;
    int tile, tb, g0, g1;
};
__device__ __forceinline__ Seg seg_at(const GemmParams& p, int32_t x, int32_t xe) {
    Seg s;
    s.x0 = x;
    s.item = x / p.G;
    s.g0 = x - s.item * p.G;
    const int32_t end = (s.item + 1) * p.G;
    s.g1 = s.g0 + ((end < xe ? end : xe) - x);
    s.tile = s.item / p.TB;
    s.tb = s.item - s.tile * p.TB;
    return s;
}

// nibbles of one packed word -> two words of int8 (c - z): codes 0..3 and 4..7
__device__ __forceinline__ void unpack_word(uint32_t w, uint32_t kk, uint32_t& lo, uint32_t& hi) {
    lo = ((w & 0x0F0F0F0Fu) + kk) ^ 0x80808080u;
    hi = (((w >> 4) & 0x0F0F0F0Fu) + kk) ^ 0x80808080u;
}

template <int BN, int MODE>
__global__ void __launch_bounds__(TcCfg<BN>::kThreads, 1)
mixed_gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_act, const __grid_constant__ CUtensorMap tmap_sa,
                     const __grid_constant__ GemmParams p) {
    using C = TcCfg<BN>;
    constexpr int NS = C::NS, NE = C::NE, BNE = C::BNE, GPS = C::GPS, NA = C::NA, NT = C::NT, NC = C::NC;
    constexpr bool kSa = (MODE == kExactGroup || MODE == kFastGroup);
    extern __shared__ uint8_t smem_raw[];
    // 1024-B aligned base (SWIZZLE_128B atoms), derived from smem_raw so the
    // compiler keeps shared-space provenance (LDS/STS, not generic LD/ST)
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* stages = smem;  // [NS][kStageBytes]
    float* meta = reinterpret_cast<float*>(stages + NS * C::kStageBytes);  // [NT] x (sw [GPS][128] | sa [GPS][BN])
    uint64_t* bars = reinterpret_cast<uint64_t*>(stages + NS * C::kStageBytes + C::kMetaBytes);
    uint64_t* full = bars;                 // [NS] producer (expect_tx)
    uint64_t* empty = full + NS;           // [NS] MMA commit + converter warps
    uint64_t* afull = empty + NS;          // [NA] converter -> MMA (TMEM A tiles + meta written)
    uint64_t* aempty = afull + NA;         // [NA] MMA commit -> converter
    uint64_t* tfull = aempty + NA;         // [NT] MMA commit -> epilogue
    uint64_t* tempty = tfull + NT;         // [NT] epilogue -> MMA / converter (acc + meta slot free)
    uint64_t* mfull = tempty + NT;         // [NT] converter -> epilogue (meta slot written)
    uint64_t* tmem_ready = mfull + NT;     // warp 1 -> everyone using TMEM
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_ready + 1);
    int* last_flag = reinterpret_cast<int*>(tmem_holder + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto stage = [&](int s) { return stages + s * C::kStageBytes; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1 + 4 * NC);
        }
        for (int i = 0; i < NA; ++i) {
            ptx::mbar_init(&afull[i], 4 * NC);
            ptx::mbar_init(&aempty[i], 1);
        }
        for (int i = 0; i < NT; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 4 * NE);
            ptx::mbar_init(&mfull[i], 4 * NC);
        }
        ptx::mbar_init(tmem_ready, 1);
        ptx::fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) trace(p, 0);
    griddep_launch();  // let the next kernel in the stream start its prologue

    const int32_t xb = p.cuts[blockIdx.x], xe = p.cuts[blockIdx.x + 1];

    // Every role walks this CTA's work as the same sequence of (segment, chunk)
    // pairs; f(sg, ti, gc, cg) runs once per chunk and returns false to stop.
    auto for_chunks = [&](auto&& f) {
        for (int32_t x = xb; x < xe;) {
            const Seg sg = seg_at(p, x, xe);
            x += sg.g1 - sg.g0;
            const TileInfo ti = tile_info(p, sg.tile);
            const int gps = ti.is8 ? C::GPS8 : GPS;
            for (int gc = sg.g0; gc < sg.g1; gc += gps) {
                const int cg = (sg.g1 - gc) < gps ? (sg.g1 - gc) : gps;
                if (!f(sg, ti, gc, cg)) return;
            }
        }
    };

    if (warp == 0) {
        // ============================== producer ==============================
        if (elect_one()) {
            ptx::prefetch_tmap(&tmap_act);
            if (kSa) ptx::prefetch_tmap(&tmap_sa);
        }
        const uint64_t pol_w = ptx::policy_evict_first();
        const uint64_t pol_a = ptx::policy_evict_last();
        constexpr uint32_t kBBytes = GPS * BN * 128;  // full boxes (OOB rows / groups zero-filled)
        constexpr uint32_t kSaBytes = kSa ? GPS * BN * 4 : 0;
        // pass 0: weights of the first NS chunks (independent of the previous
        // kernel); pass 1: activations/scales + everything else.
        for (int pass = 0; pass < 2; ++pass) {
            if (pass == 1) {
                if (lane == 0) trace(p, 1);
                griddep_wait();
                if (lane == 0) trace(p, 2);
            }
            Ring rr;
            int n = 0;
            for_chunks([&](const Seg& sg, const TileInfo& ti, int gc, int cg) {
                const bool pre = n < NS;
                if (pass == 0 && !pre) return false;
                uint8_t* st = stage(rr.idx);
                if (pass == 0 || !pre) {
                    if (pass == 1) ptx::mbar_wait(&empty[rr.idx], rr.ph ^ 1u);
                    if (lane == 0) trace_chunk(p, 0, n);
                    const uint32_t wbytes = uint32_t(cg * ti.blk);
                    if (elect_one()) {
                        ptx::mbar_arrive_expect_tx(&full[rr.idx], wbytes + kBBytes + kSaBytes);
                        ptx::bulk_g2s(st, p.wq + ti.off + int64_t(gc) * ti.blk, wbytes, &full[rr.idx], pol_w);
                    }
                    __syncwarp();
                }
                if (pass == 1) {
                    if (elect_one()) {
                        ptx::tma_load_3d(st + C::kOffB, &tmap_act, 0, sg.tb * BN, gc, &full[rr.idx], pol_a);
                        if (kSa) ptx::tma_load_2d(st + C::kOffSa, &tmap_sa, sg.tb * BN, gc, &full[rr.idx], pol_a);
                    }
                    __syncwarp();
                }
                rr.next<NS>();
                ++n;
                return true;
            });
        }
    } else if (warp == 1) {
        // ======================= TMEM allocation + MMA issuer ==================
        ptx::tmem_alloc<C::kTmemCols>(tmem_holder);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tmem_ready);
        ptx::tc_fence_after();
        const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_holder);
        const uint32_t idesc4 = idesc_i8(BN, true, true);
        const uint32_t idesc8 = p.idesc8 | ((uint32_t(BN) >> 3) << 17);
        Ring rs, ra, rt;
        int nch = 0;
        for_chunks([&](const Seg& sg, const TileInfo& ti, int gc, int cg) {
            ptx::mbar_wait(&full[rs.idx], rs.ph);
            ptx::mbar_wait(&afull[ra.idx], ra.ph);
            ptx::mbar_wait(&tempty[rt.idx], rt.ph ^ 1u);
            ptx::tc_fence_after();
            if (lane == 0) trace_chunk(p, 1, nch);
            const uint32_t st = ptx::smem_u32(stage(rs.idx));
            if (elect_one()) {
                if (!(p.dbg & 4)) {
                    for (int j = 0; j < cg; ++j) {
                        const uint32_t d_tmem = tmem_base + uint32_t((rt.idx * GPS + j) * BN);
                        const uint32_t b_addr = st + C::kOffB + j * (BN * 128);
                        if (ti.is8) {
                            const uint32_t a_addr = st + j * kBlock8Bytes;
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                ptx::mma_i8_ss(d_tmem, ptx::umma_desc_sw128(a_addr + 32 * k),
                                               ptx::umma_desc_sw128(b_addr + 32 * k), idesc8, k > 0);
                        } else {
                            const uint32_t a_tmem = tmem_base + C::kACol0 + uint32_t((ra.idx * GPS + j) * 32);
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                ptx::mma_i8_ts(d_tmem, a_tmem + 8 * k, ptx::umma_desc_sw128(b_addr + 32 * k), idesc4,
                                               k > 0);
                        }
                    }
                }
                ptx::tc_commit(&tfull[rt.idx]);
                ptx::tc_commit(&aempty[ra.idx]);
                ptx::tc_commit(&empty[rs.idx]);
            }
            __syncwarp();
            if (lane == 0) trace_chunk(p, 2, nch++);
            ra.next<NA>();
            rt.next<NT>();
            rs.next<NS>();
            return true;
        });
    } else if (warp >= 4 && warp < 4 + 4 * NC) {
        // =================== converter (sub4 -> int8 A tiles in TMEM) ===================
        const int wg = (warp - 4) >> 2;   // converter warpgroup: takes groups j = wg, wg+NC, ...
        const int r = (warp & 3) * 32 + lane;  // weight row = TMEM lane
        ptx::mbar_wait(tmem_ready, 0);
        ptx::tc_fence_after();
        const uint32_t tmem_row = *reinterpret_cast<volatile uint32_t*>(tmem_holder) + (uint32_t((warp & 3) * 32) << 16);
        Ring rs, ra, rt;
        int nch = 0;
        for_chunks([&](const Seg& sg, const TileInfo& ti, int gc, int cg) {
            // every chunk (sub8 too): wait for the stage, a free A slot and a free
            // meta slot, then (sub4) convert codes into TMEM and (all) copy the
            // chunk's weight / activation scales into the meta ring, so the stage
            // is released by the converter + MMA, never by the epilogue.
            ptx::mbar_wait(&full[rs.idx], rs.ph);
            if (threadIdx.x == 128) trace_chunk(p, 5, nch);
            ptx::mbar_wait(&aempty[ra.idx], ra.ph ^ 1u);
            ptx::mbar_wait(&tempty[rt.idx], rt.ph ^ 1u);
            if (threadIdx.x == 128) trace_chunk(p, 6, nch);
            const uint8_t* st = stage(rs.idx);
            float* msw = meta + rt.idx * (C::kMetaSlot / 4);
            for (int j = wg; j < cg; j += NC) {
                if (!ti.is8) {
                    const uint8_t* raw = st + j * kBlock4Bytes;
                    const uint32_t kk = uint32_t(128 - raw[kCodes4Bytes + 512 + r]) * 0x01010101u;
                    uint32_t v[32];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint4 w = *reinterpret_cast<const uint4*>(raw + q * 2048 + r * 16);
                        unpack_word(w.x, kk, v[q * 8 + 0], v[q * 8 + 1]);
                        unpack_word(w.y, kk, v[q * 8 + 2], v[q * 8 + 3]);
                        unpack_word(w.z, kk, v[q * 8 + 4], v[q * 8 + 5]);
                        unpack_word(w.w, kk, v[q * 8 + 6], v[q * 8 + 7]);
                    }
                    if (!(p.dbg & 2)) ptx::tmem_st32(tmem_row + C::kACol0 + uint32_t((ra.idx * GPS + j) * 32), v);
                    msw[j * 128 + r] = reinterpret_cast<const float*>(raw + kCodes4Bytes)[r];
                } else {
                    msw[j * 128 + r] = reinterpret_cast<const float*>(st + j * kBlock8Bytes + kCodes8Bytes)[r];
                }
            }
            if (kSa && wg == 0 && r < cg * BN)
                msw[GPS * 128 + r] = reinterpret_cast<const float*>(st + C::kOffSa)[r];
            if (!ti.is8) ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                ptx::mbar_arrive(&mfull[rt.idx]);
                ptx::mbar_arrive(&afull[ra.idx]);
                ptx::mbar_arrive(&empty[rs.idx]);
            }
            if (threadIdx.x == 128) trace_chunk(p, 3, nch);
            ++nch;
            ra.next<NA>();
            rt.next<NT>();
            rs.next<NS>();
            return true;
        });
    } else if (int(threadIdx.x) >= C::kEpiThread0) {
        // ============================== epilogue ==============================
        const int et = threadIdx.x - C::kEpiThread0;  // 0 .. 128*NE-1
        const int e = et >> 7;                        // epilogue warpgroup
        const int wq = warp & 3;                      // TMEM lane quarter this warp may access
        const int r = wq * 32 + lane;                 // tile row (= TMEM lane)
        const int c0 = e * BNE;                       // first token column of this warpgroup
        ptx::mbar_wait(tmem_ready, 0);
        ptx::tc_fence_after();
        const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_holder);
        griddep_wait();  // workspace / scales / output of this launch are ours now
        Ring rt;
        bool first_group = true;
        float acc[BNE];
        float sat[MODE == kExactToken ? BNE : 1];  // per-token s_a of this warpgroup's tokens
        int nch = 0;
        for_chunks([&](const Seg& sg, const TileInfo& ti, int gc, int cg) {
            if (gc == sg.g0) {
#pragma unroll
                for (int j = 0; j < BNE; ++j) acc[j] = 0.0f;
                if constexpr (MODE == kExactToken) {
                    const int64_t mb = int64_t(sg.tb) * BN + c0;
#pragma unroll
                    for (int j = 0; j < BNE; ++j) sat[j] = mb + j < p.M ? __ldg(p.sa + mb + j) : 0.0f;
                }
            }
            ptx::mbar_wait(&mfull[rt.idx], rt.ph);
            ptx::mbar_wait(&tfull[rt.idx], rt.ph);
            ptx::tc_fence_after();
            if (first_group && et == 0) trace(p, 3);
            first_group = false;
            const float* msw = meta + rt.idx * (C::kMetaSlot / 4);
            const int64_t m0 = int64_t(sg.tb) * BN + c0;  // first token of this warpgroup
            for (int j = 0; j < cg; ++j) {
                const float sw = msw[j * 128 + r];
                const float* sav = msw + GPS * 128 + j * BN + c0;
                const uint32_t tcol = uint32_t((rt.idx * GPS + j) * BN + c0);
#pragma unroll
                for (int ch = 0; ch < BNE / 16; ++ch) {
                    if (p.dbg & 1) break;
                    uint32_t v[16];
                    ptx::tmem_ld16(tmem_base + (uint32_t(wq * 32) << 16) + tcol + ch * 16, v);
                    ptx::tmem_wait_ld();
                    if constexpr (MODE == kDumpPartials) {
                        if (r < ti.rows) {
#pragma unroll
                            for (int i = 0; i < 16; ++i) {
                                const int64_t m = m0 + ch * 16 + i;
                                if (m < p.M)
                                    p.partials[(int64_t(gc + j) * p.M + m) * p.partial_rows + ti.first + r] = int32_t(v[i]);
                            }
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const float gs = __int2float_rn(int32_t(v[i]));  // exact: |S| < 2^22
                            const int jj = ch * 16 + i;
                            if constexpr (MODE == kExactGroup) {
                                // gemm.cpp:81 — out += gs * (s_a * s_w), no contraction
                                acc[jj] = __fadd_rn(acc[jj], __fmul_rn(gs, __fmul_rn(sav[jj], sw)));
                            } else if constexpr (MODE == kExactToken) {
                                acc[jj] = __fadd_rn(acc[jj], __fmul_rn(gs, __fmul_rn(sat[jj], sw)));
                            } else if constexpr (MODE == kFastGroup) {
                                acc[jj] = __fmaf_rn(gs, __fmul_rn(sav[jj], sw), acc[jj]);
                            } else {
                                acc[jj] = __fmaf_rn(gs, sw, acc[jj]);
                            }
                        }
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[rt.idx]);
            if (et == 0) trace_chunk(p, 4, nch);
            ++nch;
            rt.next<NT>();
            if (gc + cg < sg.g1) return true;  // the segment continues in the next chunk

            // ---------------- end of segment: output or stream-K partial
            if constexpr (MODE == kDumpPartials) return true;
            if (et == 0) trace(p, 4);
            const int col = r < ti.rows ? __ldg(p.colmap + sg.tile * kTileRows + r) : -1;
            bool do_store = true;
            const int32_t xs = sg.item * p.G;  // the item's linear group range [xs, xs + G)
            if (p.split && !(xb <= xs && xe >= xs + p.G)) {
                // this CTA holds only part of the item: publish the partial tile to
                // slot 2*c + (first segment of this CTA ? 0 : 1); the last arriving
                // CTA sums the item's partials in CTA order (deterministic).
                const int slot = 2 * int(blockIdx.x) + (sg.x0 == xb ? 0 : 1);
                float* part = p.ws + (int64_t(slot) * 128 + r) * BN + c0;
#pragma unroll
                for (int j = 0; j < BNE; j += 4)
                    __stcg(reinterpret_cast<float4*>(part + j), make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]));
                __threadfence();
                named_bar_sync(3, 128 * NE);
                const int ca = cta_owner(p, xs), cz = cta_owner(p, xs + p.G - 1);
                if (et == 0) {
                    const uint32_t prev = atomicAdd(p.counters + sg.item, 1u);
                    *reinterpret_cast<volatile int*>(last_flag) = (prev == uint32_t(cz - ca));
                }
                named_bar_sync(3, 128 * NE);
                do_store = *reinterpret_cast<volatile int*>(last_flag) != 0;
                if (do_store) {
                    __threadfence();
                    const bool ca_first = p.cuts[ca] == xs;
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
            return true;
        });
    }

    if (threadIdx.x == C::kEpiThread0) trace(p, 5);
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) trace(p, 6);
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<C::kTmemCols>(*reinterpret_cast<volatile uint32_t*>(tmem_holder));
    }
}

template <int BN, int MODE>
cudaError_t launch_bn_mode(const GemmParams& p, const void* tmap, const void* tmap_sa, bool pdl, cudaStream_t stream) {
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
    return cudaLaunchKernelEx(&cfg, kern, *static_cast<const CUtensorMap*>(tmap),
                              *static_cast<const CUtensorMap*>(tmap_sa), p);
}

template <int BN>
cudaError_t launch_bn(const GemmParams& p, const void* tmap, const void* tmap_sa, int mode, bool pdl, cudaStream_t s) {
    switch (mode) {
        case kExactGroup: return launch_bn_mode<BN, kExactGroup>(p, tmap, tmap_sa, pdl, s);
        case kFastGroup: return launch_bn_mode<BN, kFastGroup>(p, tmap, tmap_sa, pdl, s);
        case kFastToken: return launch_bn_mode<BN, kFastToken>(p, tmap, tmap_sa, pdl, s);
        case kExactToken: return launch_bn_mode<BN, kExactToken>(p, tmap, tmap_sa, pdl, s);
        default: return launch_bn_mode<BN, kDumpPartials>(p, tmap, tmap_sa, pdl, s);
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

cudaError_t launch_mixed_gemm_tc(const GemmParams& p, const void* tmap, const void* tmap_sa, int token_tile, int mode,
                                 bool pdl, cudaStream_t stream) {
    switch (token_tile) {
        case 16: return launch_bn<16>(p, tmap, tmap_sa, mode, pdl, stream);
        case 32: return launch_bn<32>(p, tmap, tmap_sa, mode, pdl, stream);
        case 64: return launch_bn<64>(p, tmap, tmap_sa, mode, pdl, stream);
        case 128: return launch_bn<128>(p, tmap, tmap_sa, mode, pdl, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace mq

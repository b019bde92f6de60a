// mixed_gemm_sm100.cuh — K2: the MixLLM W4/W8-A8 mixed-precision group GEMM on
// 5th-generation tensor cores (tcgen05.mma kind::i8, TMEM accumulators).
//
// Reference semantics (proj/src/gemm.cpp:51-85, the emulated kernel): for every
// output element and every K-group g in ascending order,
//   step 1  S_g = sum_i a[m, i] * (w[r, i] - z[r, g])        (int32, exact)
//   step 2  out += float(S_g) * (s_a[m, g] * s_w[r, g])     (f32 mul, f32 add)
// and the two sub-problems (8-bit / 4-bit output features) are scattered back
// to their original columns (proj/src/mixed.cpp:83-120).
//
// B200 design. One launch covers both sub-problems (the paper's "parallel
// sub-problems"). Each CTA owns one (128-row weight tile,
// token tile, K-slice) — see work_of() in mq_kernels.hpp; the K-slices of a
// split tile are reduced in slice order by the last one to finish
// (deterministic). Work moves in CHUNKS of up to GPS consecutive groups (GPS/2 for
// sub8, whose groups are twice the bytes); roles are warp-specialised and hand
// off per chunk through mbarriers:
//   warp 0      producer: per chunk one cp.async.bulk of the merged code+meta
//               blocks (L2 evict-first) and one bulk copy each of the chunk's
//               activation tiles / scales, which K1 already wrote in the
//               engine activation layout (EAL, pre-swizzled SW128 images). The
//               first NS weight copies issue BEFORE griddepcontrol.wait, so under
//               PDL they overlap the previous kernel;
//   converter   one thread per weight row: sub4 nibbles -> int8 (c - z) with the
//               carry-free bias trick ((x & 0x0F0F0F0F) + (128 - z)*0x01010101) ^
//               0x80808080 (the paper's step-1 zero-point subtraction,
//               PAPER.md:344-353), tcgen05.st of the row into a TMEM A-operand
//               ring; for every chunk it also copies the weight / activation
//               scales into a small meta ring, so a stage is released as soon as
//               the converter and the MMA are done with it;
//   warp 1      TMEM allocation, then MMA issue (elected lane): 4 x tcgen05.mma
//               (K = 32) per group, A from TMEM (sub4) or from the pre-swizzled
//               SMEM block (sub8), each group into a fresh int32 TMEM accumulator;
//   epilogue    tcgen05.ld the group sums, exact int->float, rescale and
//               accumulate in f32 registers (step 2); at the end scatter to the
//               original output columns (f32/f16/bf16), through the split-K
//               partial workspace when the tile is split along K.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "mq_kernels.hpp"
#include "mq_ptx.cuh"

namespace mq {
namespace {

constexpr int kSmemMax = 232448;  // 227 KB opt-in dynamic shared memory per CTA

template <int BN>
struct TcCfg {
    // Decode token tiles (<= 32 tokens) size a CTA for TWO per SM (half the
    // shared memory, registers and TMEM): the next launch's CTAs then become
    // resident while this launch's CTAs finish (split-K join, scattered output
    // stores), so under PDL the next projection's weights stream into its
    // rings during this one's tail. Token-tiled (prefill) launches own the SM.
#ifndef MQ_DEC2
#define MQ_DEC2 0
#endif
    static constexpr bool kDec = MQ_DEC2 && BN <= 32;
    static constexpr int kMinBlocks = kDec ? 2 : 1;
    static constexpr int kSmemBudget = kDec ? 113 * 1024 : kSmemMax;
    static constexpr uint32_t kTmemBudget = kDec ? 256u : 512u;
    static constexpr int GPS = gemm_gps(BN);                // sub4 groups per chunk
    static constexpr int GPS8 = GPS / 2 > 0 ? GPS / 2 : 1;  // sub8 groups per chunk
    static constexpr int kRaw0 = GPS * kBlock4Bytes > GPS8 * kBlock8Bytes ? GPS * kBlock4Bytes : GPS8 * kBlock8Bytes;
    // weight stage: one chunk's code+meta blocks; activation stage (separate
    // ring, so a sub4 weight stage is free as soon as the converter has read it):
    // the chunk's [GPS][BN][128] SW128 activation tiles + [GPS][BN] f32 scales
    static constexpr int kStageBytes = (kRaw0 + 1023) / 1024 * 1024;
    // decode token tiles apply the sub4 zero point in the epilogue
    // (sum a(c - z) = sum a c - z sum a, sum a from K1), so the converter only
    // widens nibbles to bytes and the MMA reads the codes as u8
    static constexpr bool kZpEpi = BN <= 32;
    // decode: the epilogue reads the activation scales / code sums straight from
    // the activation stage (released by the epilogue, not the MMA), so the
    // converter never waits for the activations and runs ahead on the weights
#ifndef MQ_SA_DIRECT
#define MQ_SA_DIRECT 1
#endif
    static constexpr bool kSaDirect = BN <= 32 && MQ_SA_DIRECT;
    static constexpr int kOffSa = GPS * BN * 128;
    static constexpr int kOffAs = kOffSa + GPS * BN * 4;
    static constexpr int kXStageBytes = ((kOffAs + (kZpEpi ? GPS * BN * 4 : 0)) + 1023) / 1024 * 1024;
    // activation stages: a prefill tile needs a fresh 16 KB activation tile per
    // group (from L2), so its ring is as deep as the weight ring
    #ifndef MQ_NX16
#define MQ_NX16 8
#endif
#ifndef MQ_NX32
#define MQ_NX32 4
#endif
    // (16-token tiles: 8 activation stages and 3 weight stages beat 3 + 5 — the
    // activations come from L2 under full HBM streaming, so their ring needs the
    // depth; M <= 16 stack -2%. 32-token tiles, 4-group chunks: 4 — 3 and 5 were
    // 8% slower)
#ifndef MQ_NX64
#define MQ_NX64 6
#endif
#ifndef MQ_NX128
#define MQ_NX128 8
#endif
    static constexpr int NX = BN >= 128 ? MQ_NX128 : BN >= 64 ? MQ_NX64 : BN == 16 ? MQ_NX16 : MQ_NX32;
    // TMEM rings: NT accumulator chunk slots of GPS x BN int32 columns, NA
    // A-operand chunk slots of GPS x 32 columns (128 int8 K per row).
    static constexpr uint32_t kAccPerChunk = GPS * BN, kAPerChunk = GPS * 32;
#ifndef MQ_NT16
#define MQ_NT16 2
#endif
    static constexpr int NT = BN >= 128 ? 3 : BN == 16 ? MQ_NT16 : 2;
    static constexpr int NA0 = int((kTmemBudget - NT * kAccPerChunk) / kAPerChunk);
    static constexpr int NA = NA0 > 4 ? 4 : NA0;
    static constexpr uint32_t kAccCols = NT * kAccPerChunk;
    static constexpr uint32_t kACol0 = kAccCols;
    static constexpr uint32_t kTmemNeed = kAccCols + NA * kAPerChunk;
    static constexpr uint32_t kTmemCols = kTmemNeed <= 32 ? 32 : kTmemNeed <= 64 ? 64 : kTmemNeed <= 128 ? 128 : kTmemNeed <= 256 ? 256 : 512;
    static_assert(kTmemCols <= kTmemBudget && NA >= 2, "TMEM budget");
    // meta ring (per accumulator slot): weight scales [GPS][128] | (kZpEpi) zero
    // points [GPS][128] | act scales [GPS][BN] | (kZpEpi) code sums [GPS][BN]
    static constexpr int kMetaZp = GPS * 128, kMetaSa = GPS * 128 * (kZpEpi ? 2 : 1), kMetaAs = kMetaSa + GPS * BN;
    static constexpr int kMetaSlot = (kMetaAs + (kZpEpi ? GPS * BN : 0)) * 4;
    // the meta ring is deeper than the accumulator ring and has its own
    // barriers, so the converter never waits on the epilogue of chunk n - NT
    static constexpr int NM = 4;
    static constexpr int kMetaBytes = NM * kMetaSlot;
    static constexpr int kFixed = 1024 /*alignment slack*/ + 1024 /*barriers*/ + kMetaBytes + NX * kXStageBytes;
    static constexpr int NS0 = (kSmemBudget - kFixed) / kStageBytes;
#ifndef MQ_NS_MAX
#define MQ_NS_MAX 8
#endif
    static constexpr int NS = NS0 > MQ_NS_MAX ? MQ_NS_MAX : NS0;
    // epilogue warpgroups: two for 128-token tiles (one warp per SMSP leaves
    // the TMEM-load / rescale chain latency-bound), one at 64 tokens (a second
    // measured ~2% slower) and at decode (two CTAs per SM share the SMSPs)
    #ifndef MQ_NE16
#define MQ_NE16 2
#endif
#ifndef MQ_NC16
#define MQ_NC16 2
#endif
    static constexpr int NE = BN == 16 ? (kDec ? 1 : MQ_NE16) : (BN == 64 || kDec) ? 1 : 2;
    // converter warpgroups: one (at decode the two co-resident CTAs provide the
    // second; from 32 tokens the rescale dominates)
    static constexpr int NC = (BN == 16 && !kDec) ? MQ_NC16 : 1;
    static constexpr int BNE = BN / NE;          // tokens per epilogue warpgroup
    static constexpr int kEpiThread0 = 128 * (1 + NC);
    static constexpr int kThreads = 128 * (1 + NC + NE);
    static constexpr int kSmem = kFixed + NS * kStageBytes;
    static_assert(NS >= 2, "pipeline needs at least two stages");
    static_assert(kSmem <= kSmemBudget, "shared memory budget");
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

// Development instrumentation (globaltimer / clock64 traces, MQ_DBG stage
// bypasses) is compiled only with -DMQ_DEV (tools/ builds it beside the
// product library): every check sits on the per-chunk hot path.
#ifdef MQ_DEV
constexpr bool kDev = true;
#else
constexpr bool kDev = false;
#endif
__device__ __forceinline__ int dbg_bits(const GemmParams& p) { return kDev ? p.dbg : 0; }
__device__ __forceinline__ void trace(const GemmParams& p, int ev) {
    if (kDev && p.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
        p.trace[blockIdx.x * 8 + ev] = t;
    }
}
// per-chunk event trace of one CTA (MQ_DBG & 64, CTA = MQ_DBG >> 8), in SM cycles
__device__ __forceinline__ void trace_chunk(const GemmParams& p, int ev, int n) {
    if (kDev && p.trace && (p.dbg & 64) && int(blockIdx.x) == (p.dbg >> 8) && n < 64)
        p.trace[148 * 8 + ev * 64 + n] = clock64();
}

// One thread's output row: tokens m0 .. m0 + BNE - 1 of original column col
// (col < 0: a padding row), the dtype switch and the bounds hoisted out of the
// per-token loop, the address advanced by one row stride per token (a
// per-element dtype switch and 64-bit index made the scatter ~20% of a prefill
// launch). The PEER kernel variant (the fused gather, mq_mixed_linear_peers,
// npeer > 1) also stores every element into each peer rank's copy of Y at the
// same (original) column, over NVLink — a separate instantiation
// (mixed_gemm_peers.cu): the peer loop costs the plain kernels ~20% at prefill.
template <typename T>
__device__ __forceinline__ T to_out(float v) {
    if constexpr (std::is_same<T, __half>::value) return __float2half_rn(v);
    else if constexpr (std::is_same<T, __nv_bfloat16>::value) return __float2bfloat16_rn(v);
    else return v;
}
template <typename T, int BNE, int MODE>
__device__ __forceinline__ void store_col(void* Y, int64_t ldy, int64_t m0, int col, int jn, const float* v,
                                          const float* sa) {
    T* y = static_cast<T*>(Y) + (m0 * ldy + col);
#pragma unroll
    for (int j = 0; j < BNE; ++j) {
        if (j < jn) {
            float x = v[j];
            if constexpr (MODE == kFastToken) x = __fmul_rn(x, __ldg(sa + m0 + j));
            *y = to_out<T>(x);
        }
        y += ldy;
    }
}
template <typename T, int BNE, int MODE, int PEER>
__device__ __forceinline__ void store_cols(const GemmParams& p, int64_t m0, int col, int jn, const float* v) {
    store_col<T, BNE, MODE>(p.Y, p.ldy, m0, col, jn, v, p.sa);
    if constexpr (PEER)
        for (int i = 1; i < p.npeer; ++i) store_col<T, BNE, MODE>(p.ypeer[i], p.ldy, m0, col, jn, v, p.sa);
}
template <int BNE, int MODE, int PEER>
__device__ __forceinline__ void store_tokens(const GemmParams& p, int64_t m0, int col, const float* v) {
    if (col < 0) return;
    const int64_t rem = p.M - m0;
    const int jn = rem < BNE ? int(rem) : BNE;
    if (p.out_dtype == 1) store_cols<__half, BNE, MODE, PEER>(p, m0, col, jn, v);
    else if (p.out_dtype == 2) store_cols<__nv_bfloat16, BNE, MODE, PEER>(p, m0, col, jn, v);
    else store_cols<float, BNE, MODE, PEER>(p, m0, col, jn, v);
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

// f32x2 (FFMA2 / FMUL2 on sm_100) through the float2 builtins, so the
// accumulator pairs stay in place (no register-pair moves). FAST modes only —
// the exact (reference op order) mode stays scalar.
__device__ __forceinline__ float2 pk2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// nibbles of one packed word -> two words of int8 (c - z): codes 0..3 and 4..7
__device__ __forceinline__ void unpack_word(uint32_t w, uint32_t kk, uint32_t& lo, uint32_t& hi) {
    lo = ((w & 0x0F0F0F0Fu) + kk) ^ 0x80808080u;
    hi = (((w >> 4) & 0x0F0F0F0Fu) + kk) ^ 0x80808080u;
}

// Stream-K: the CTA whose range [skb[b], skb[b+1]) holds position `key`
// (item << 8 | group); the plan's boundaries are strictly increasing.
__device__ __forceinline__ int sk_cta_of(const GemmParams& p, uint32_t key) {
    int lo = 0, hi = p.grid - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p.skb[mid] <= key) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Stream-K split piece epilogue. Every CTA's range covers at least one item's
// length (host plan), so an item is cut at most once: its HEAD (groups [0, g)) is the last
// piece of CTA b and its TAIL (groups [g, G)) the first piece of CTA b + 1.
// The two meet without any spin-wait (no co-residency assumption): boundary
// s = b + 1 owns flag cnt[s] and two partial slots ([slot][BN/4][128] float4,
// a warp's stores are 512 contiguous bytes), tails in p.part, heads in
// p.part2. The tail publishes its partial and arrives; the head (which almost
// always runs later) first checks the flag: if the tail is done it adds the
// tail's partial without publishing its own; otherwise it publishes and
// arrives. Whoever arrives second sums head + tail (one f32 add: commutative,
// so the result is the same bit pattern either way) and returns true so the
// caller scatters; it also re-arms the flag for the next launch.
template <int BN, int BNE, int NE>
__device__ __noinline__ bool sk_piece_done(const GemmParams& p, const Work& wk, float* acc, int r, int c0, int et,
                                           volatile int* s_last) {
    constexpr int V = BNE / 4;
    const bool tail = wk.g0 > 0;
    const int s = int(blockIdx.x) + (tail ? 0 : 1);
    float4* mine = reinterpret_cast<float4*>(tail ? p.part : p.part2) + (int64_t(s) * (BN / 4) + c0 / 4) * 128 + r;
    const float4* other = reinterpret_cast<const float4*>(tail ? p.part2 : p.part) + (int64_t(s) * (BN / 4) + c0 / 4) * 128 + r;
    int mode = 0;  // 0: publish and arrive, 2: head that found the tail done
    if (!tail) {
        if (et == 0) {
            uint32_t f;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(p.cnt + s) : "memory");
            if (f) p.cnt[s] = 0u;  // both pieces are here: re-arm
            *s_last = f ? 2 : 0;
        }
        named_bar_sync(2, 128 * NE);  // orders the acquire before every thread's ld.cg below
        mode = *s_last;
        named_bar_sync(2, 128 * NE);  // s_last is rewritten below
    }
    bool last = mode == 2;
    if (!last) {
#pragma unroll
        for (int j = 0; j < V; ++j)
            __stcg(mine + j * 128, make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]));
        named_bar_sync(2, 128 * NE);
        if (et == 0) {  // release our partial (ordered before by bar.sync) / acquire the other's
            uint32_t prev;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.cnt + s) : "memory");
            if (prev == 1u) p.cnt[s] = 0u;  // second arrival: re-arm
            *s_last = prev == 1u;
        }
        named_bar_sync(2, 128 * NE);
        last = *s_last != 0;
        named_bar_sync(2, 128 * NE);  // s_last is reused by the next unit
        if (!last) return false;
    }
    constexpr int VB = V < 8 ? V : 8;  // float4 loads in flight per batch
#pragma unroll
    for (int j0 = 0; j0 < V; j0 += VB) {
        float4 t[VB];
#pragma unroll
        for (int q = 0; q < VB; ++q) t[q] = __ldcg(other + (j0 + q) * 128);
#pragma unroll
        for (int q = 0; q < VB; ++q) {
            acc[4 * (j0 + q) + 0] = __fadd_rn(acc[4 * (j0 + q) + 0], t[q].x);
            acc[4 * (j0 + q) + 1] = __fadd_rn(acc[4 * (j0 + q) + 1], t[q].y);
            acc[4 * (j0 + q) + 2] = __fadd_rn(acc[4 * (j0 + q) + 2], t[q].z);
            acc[4 * (j0 + q) + 3] = __fadd_rn(acc[4 * (j0 + q) + 3], t[q].w);
        }
    }
    return true;
}

// K-split join for wide token tiles (BN >= 64, one token block, MQ_FAST): the
// S slices of an item publish their partial tiles to slot = unit
// ([slot][BN/4][128] float4, coalesced). When every unit runs in one round of
// the persistent grid (all slices co-resident) the slices meet at a per-item
// barrier (arrivals then departures on one counter) and each one sums and
// scatters only ITS BN/S tokens — the scattered stores drain at ~25 cycles per
// warp instruction, so one CTA storing the whole tile would be the launch's
// tail. Otherwise the last arrival sums and scatters the whole tile. Sums run
// in slice order (deterministic). Out of line: its registers would push the
// 64-accumulator epilogue loop into spills.
template <int BN, int BNE, int NE, int MODE, int PEER>
__device__ __noinline__ void split_join_wide(const GemmParams& p, const Work& wk, int slot, float* acc, int r,
                                             int c0, int et, volatile int* s_last, int col, int64_t m0) {
    constexpr int V = BNE / 4;
    float4* part4 = reinterpret_cast<float4*>(p.part);
    float4* mine = part4 + (int64_t(slot) * (BN / 4) + c0 / 4) * 128 + r;
#pragma unroll
    for (int j = 0; j < V; ++j)
        __stcg(mine + j * 128, make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]));
    named_bar_sync(2, 128 * NE);
    // the per-item barrier assumes every slice is resident: only when all units
    // run in one round and the caller did not declare concurrent launches
    const bool together = p.units <= int(gridDim.x) && !p.no_spin;
    if (et == 0) {
        if (together) {
            // arrivals count to S, departures to 2S; the last departure re-arms
            // the counter (every slice has seen >= S by then), so it is zero
            // again at launch end and no generation word is needed
            uint32_t* c = p.cnt + wk.item;
            uint32_t prev, v;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(c) : "memory");
            for (v = prev + 1; v < uint32_t(wk.S);) {
                __nanosleep(20);
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
            }
            asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(c) : "memory");
            if (prev == uint32_t(2 * wk.S - 1)) *c = 0u;
        } else {  // release our partial / acquire the others' (see the decode join)
            uint32_t prev;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.cnt + wk.item) : "memory");
            *s_last = prev == uint32_t(wk.S - 1);
            if (prev == uint32_t(wk.S - 1)) p.cnt[wk.item] = 0u;  // re-arm for the next launch
        }
    }
    named_bar_sync(2, 128 * NE);
    // token range this CTA sums and scatters: its slice's share, or the whole tile
    int j0 = 0, j1 = BNE;
    if (together) {
        const int t0 = wk.sl * (BN / wk.S), t1 = t0 + BN / wk.S;
        j0 = (t0 > c0 ? t0 : c0) - c0;
        j1 = (t1 < c0 + BNE ? t1 : c0 + BNE) - c0;
        if (j1 <= j0) return;
    } else {
        const bool last = *s_last != 0;
        named_bar_sync(2, 128 * NE);  // s_last is reused by the next unit
        if (!last) return;
    }
    for (int j = j0; j < j1; j += 4) {  // float4 of tokens j..j+3 (BN/S is a multiple of 4)
        float4 sum = __ldcg(part4 + (int64_t(wk.cta0) * (BN / 4) + (c0 + j) / 4) * 128 + r);
        for (int sl = 1; sl < wk.S; ++sl) {
            const float4 t = __ldcg(part4 + (int64_t(wk.cta0 + sl) * (BN / 4) + (c0 + j) / 4) * 128 + r);
            sum.x = __fadd_rn(sum.x, t.x);
            sum.y = __fadd_rn(sum.y, t.y);
            sum.z = __fadd_rn(sum.z, t.z);
            sum.w = __fadd_rn(sum.w, t.w);
        }
        const float v4[4] = {sum.x, sum.y, sum.z, sum.w};
        store_tokens<4, MODE, PEER>(p, m0 + j, col, v4);
    }
}

// SPL = 1: for 64/128-token tiles the wide-tile K-split join is compiled in
// (launched only for split unit schedules; its out-of-line call costs the other
// wide launches ~4% in the accumulation loop's register allocation); for decode
// tiles the stream-K piece decoding (launched only for schedule = 2)
template <int BN, int MODE, int SPL, int PEER>
__global__ void __launch_bounds__(TcCfg<BN>::kThreads, TcCfg<BN>::kMinBlocks) mixed_gemm_tc_kernel(const __grid_constant__ GemmParams p) {
    using C = TcCfg<BN>;
    constexpr int NS = C::NS, NE = C::NE, BNE = C::BNE, GPS = C::GPS, NA = C::NA, NT = C::NT, NC = C::NC;
    constexpr bool kSa = (MODE == kExactGroup || MODE == kFastGroup);
    constexpr bool kSkPath = BN >= 64 || SPL;  // stream-K piece decoding compiled in
    extern __shared__ uint8_t smem_raw[];
    // 1024-B aligned base (SWIZZLE_128B atoms), derived from smem_raw so the
    // compiler keeps shared-space provenance (LDS/STS, not generic LD/ST)
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* stages = smem;                            // [NS][kStageBytes] weights
    uint8_t* xstages = stages + NS * C::kStageBytes;   // [NX][kXStageBytes] activations
    float* meta = reinterpret_cast<float*>(xstages + C::NX * C::kXStageBytes);  // [NT] x (sw [GPS][128] | sa [GPS][BN])
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(meta) + C::kMetaBytes);
    uint64_t* full = bars;                 // [NS] producer (expect_tx)
    uint64_t* empty = full + NS;           // [NS] converter warps + (sub8: MMA commit, sub4: converter)
    uint64_t* xfull = empty + NS;          // [NX] producer (activation tiles + scales, expect_tx)
    uint64_t* xempty = xfull + C::NX;      // [NX] MMA commit
    uint64_t* afull = xempty + C::NX;      // [NA] converter -> MMA (TMEM A tiles + meta written)
    uint64_t* aempty = afull + NA;         // [NA] MMA commit -> converter
    uint64_t* tfull = aempty + NA;         // [NT] MMA commit -> epilogue
    uint64_t* tempty = tfull + NT;         // [NT] epilogue -> MMA / converter (acc + meta slot free)
    uint64_t* mfull = tempty + NT;         // [NM] converter -> epilogue (meta slot written)
    uint64_t* mempty = mfull + C::NM;      // [NM] epilogue -> converter (meta slot read)
    uint64_t* tmem_ready = mempty + C::NM; // warp 1 -> everyone using TMEM
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_ready + 1);
    volatile int* s_last = reinterpret_cast<volatile int*>(tmem_holder + 1);  // split-K: this CTA reduces

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto stage = [&](int s) { return stages + s * C::kStageBytes; };
    auto xstage = [&](int s) { return xstages + s * C::kXStageBytes; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1 + 4 * NC);
        }
        for (int s = 0; s < C::NX; ++s) {
            ptx::mbar_init(&xfull[s], 1);
            ptx::mbar_init(&xempty[s], C::kSaDirect ? 4 * NE : 1);
        }
        for (int i = 0; i < NA; ++i) {
            ptx::mbar_init(&afull[i], 4 * NC);
            ptx::mbar_init(&aempty[i], 1);
        }
        for (int i = 0; i < NT; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 4 * NE);
        }
        for (int i = 0; i < C::NM; ++i) {
            ptx::mbar_init(&mfull[i], 4 * NC);
            ptx::mbar_init(&mempty[i], 4 * NE);
        }
        ptx::mbar_init(tmem_ready, 1);
        ptx::fence_barrier_init();
    }
    if constexpr (C::kSaDirect) {
        // the decode epilogue runs every group of a chunk and reads a short
        // chunk's unused activation-scale slots (times a zero weight scale):
        // they must hold finite values before the first copy lands
        if (warp == 3)
            for (int i = lane; i < C::NX * GPS * BN; i += 32)
                reinterpret_cast<float*>(xstage(i / (GPS * BN)) + C::kOffSa)[i % (GPS * BN)] = 0.0f;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        trace(p, 0);
        trace_chunk(p, 14, 0);
    }
    griddep_launch();  // let the next kernel in the stream start its prologue

    // Persistent: CTA b walks work units b, b + grid, b + 2 grid, ... (each unit
    // = one (tile, token block, K-slice), mq_kernels.hpp); every role walks the
    // same (unit, chunk) sequence, so the rings run on across units and the next
    // unit's weights stream while the current unit's epilogue finishes.
    struct Unit {
        Work wk;
        TileInfo ti;
        int gps, nch, rot, key;
    };
    auto unit_of = [&](const Work& w, int u) {
        Unit U;
        U.wk = w;
        U.key = u;
        U.ti = tile_info(p, U.wk.tile);
        U.gps = U.ti.is8 ? C::GPS8 : GPS;
        // gps is a power of two: shifts, not divisions (see work_of)
        const int lgg = U.gps == 4 ? 2 : U.gps == 2 ? 1 : 0;
        U.nch = (dbg_bits(p) & 8) ? 0 : (U.wk.g1 - U.wk.g0 + U.gps - 1) >> lgg;  // dbg&8: launch-floor probe
        // FAST modes start each unit at a different chunk of its K-slice so the
        // CTAs do not all read the same activation lines at the same time
        // (multiply-shift hash into [0, nch), no division)
        U.rot = (p.rotate && U.nch > 1) ? int(((uint32_t(u) * 2654435761u >> 16) * uint32_t(U.nch)) >> 16) : 0;
        return U;
    };
    const int u0 = blockIdx.x, ustep = gridDim.x;
    // k-th piece of work of this CTA. Unit schedule: units u0, u0 + grid, ...
    // Stream-K schedule (p.sk): the CTA's contiguous range [skb[b], skb[b+1])
    // of (item, group) positions, cut into one piece per item it touches; a
    // piece that is not a whole item is "split" (S = 2; see sk_piece_done).
    auto piece = [&](int k, Unit& U) -> bool {
        // decode token tiles compile the stream-K decoding only into their SPL = 1
        // variant (schedule = 2): every role decodes a piece per unit, and the
        // extra path costs the default decode launches a few percent
        if (!(kSkPath && p.sk)) {
            const int u = u0 + k * ustep;
            if (u >= p.units) return false;
            U = unit_of(work_of(p, u), u);
            return true;
        }
        const uint32_t a = p.skb[blockIdx.x], e = p.skb[blockIdx.x + 1];
        const int it = int(a >> 8) + k, ie = int(e >> 8);
        if (it > ie || (it == ie && (e & 255u) == 0u)) return false;
        Work w;
        w.item = it;
        w.tb = p.TB == 1 ? 0 : it / p.T;
        w.tile = it - w.tb * p.T;
        w.g0 = k == 0 ? int(a & 255u) : 0;
        w.g1 = it == ie ? int(e & 255u) : p.G;
        w.S = (w.g0 == 0 && w.g1 == p.G) ? 1 : 2;
        w.sl = 0;
        w.cta0 = 0;
        U = unit_of(w, it);
        return true;
    };
    auto chunk_at = [&](const Unit& U, int i, int& gc, int& cg) {
        int c = i + U.rot;
        if (c >= U.nch) c -= U.nch;
        gc = U.wk.g0 + c * U.gps;
        cg = (U.wk.g1 - gc) < U.gps ? (U.wk.g1 - gc) : U.gps;
    };

    if (warp == 0) {
        // ============================== producer ==============================
        if (lane == 0) trace(p, 2);
        if (lane == 0) trace_chunk(p, 15, 1);
        const uint64_t pol_w = ptx::policy_evict_first();
        if (lane == 0) trace_chunk(p, 15, 2);
        // weights are immutable: this warp never waits on the previous kernel
        // (griddepcontrol), so under PDL the first NS stages fill while it runs
        Ring rr;
        int n = 0;  // chunk counter across units
        for (int pk = 0;; ++pk) {
            Unit U;
            if (!piece(pk, U)) break;
            if (lane == 0 && pk == 0) trace_chunk(p, 15, 3);
            for (int i = 0; i < U.nch; ++i, ++n) {
                int gc, cg;
                chunk_at(U, i, gc, cg);
                uint8_t* st = stage(rr.idx);
                if (lane == 0 && n == 0) trace_chunk(p, 15, 4);
                ptx::mbar_wait(&empty[rr.idx], rr.ph ^ 1u);
                if (lane == 0 && n == 0) trace_chunk(p, 15, 5);
                if (lane == 0) trace_chunk(p, 0, n);
                if (n == 0 && lane == 0) trace(p, 7);
                const uint32_t wbytes = uint32_t(cg * U.ti.blk);
                if (elect_one()) {
                    ptx::mbar_arrive_expect_tx(&full[rr.idx], wbytes);
                    ptx::bulk_g2s(st, p.wq + U.ti.off + int64_t(gc) * U.ti.blk, wbytes, &full[rr.idx], pol_w);
                }
                __syncwarp();
                rr.next<NS>();
            }
        }
        // every weight read of this launch is issued: warm L2 with the next
        // layer's weights (its first-byte latency and this launch's tail overlap)
        if (p.pf_bytes > 0 && elect_one()) {
            const int64_t per = ((p.pf_bytes + gridDim.x - 1) / gridDim.x + 255) / 256 * 256;
            int64_t a = int64_t(blockIdx.x) * per;
            const int64_t e = a + per < p.pf_bytes ? a + per : p.pf_bytes;
            for (; a < e; a += 32768) ptx::bulk_prefetch_l2(p.pf + a, uint32_t(e - a < 32768 ? e - a : 32768));
        }
        __syncwarp();
        if (lane == 0) trace(p, 1);
    } else if (warp == 2) {
        // ===================== activation producer (EAL tiles) =====================
        // its own warp, so the weight stream never waits behind the activation ring
        const uint64_t pol_a = ptx::policy_evict_last();
        const bool contig = p.Mpad == BN;  // one token tile: a chunk's act tiles are contiguous
        griddep_wait();  // K1's output
        Ring rx;
        int n = 0;
        for (int pk = 0;; ++pk) {
            Unit U;
            if (!piece(pk, U)) break;
            for (int i = 0; i < U.nch; ++i, ++n) {
                int gc, cg;
                chunk_at(U, i, gc, cg);
                uint8_t* xs = xstage(rx.idx);
                ptx::mbar_wait(&xempty[rx.idx], rx.ph ^ 1u);
                if (lane == 0) trace_chunk(p, 10, n);
                if (elect_one()) {
                    ptx::mbar_arrive_expect_tx(&xfull[rx.idx], uint32_t(cg * BN * 128 + (kSa ? cg * BN * 4 : 0) +
                                                                        (C::kZpEpi ? cg * BN * 4 : 0)));
                    const int64_t row0 = int64_t(U.wk.tb) * BN;
                    if (contig) {
                        ptx::bulk_g2s(xs, p.acts + int64_t(gc) * p.Mpad * 128, uint32_t(cg * BN * 128), &xfull[rx.idx], pol_a);
                        if (kSa)
                            ptx::bulk_g2s(xs + C::kOffSa, p.sa + int64_t(gc) * p.Mpad, uint32_t(cg * BN * 4), &xfull[rx.idx],
                                          pol_a);
                        if (C::kZpEpi)
                            ptx::bulk_g2s(xs + C::kOffAs, p.asum + int64_t(gc) * p.Mpad, uint32_t(cg * BN * 4),
                                          &xfull[rx.idx], pol_a);
                    } else {
                        for (int j = 0; j < cg; ++j) {
                            ptx::bulk_g2s(xs + j * BN * 128, p.acts + (int64_t(gc + j) * p.Mpad + row0) * 128,
                                          uint32_t(BN * 128), &xfull[rx.idx], pol_a);
                            if (kSa)
                                ptx::bulk_g2s(xs + C::kOffSa + j * BN * 4, p.sa + int64_t(gc + j) * p.Mpad + row0,
                                              uint32_t(BN * 4), &xfull[rx.idx], pol_a);
                            if (C::kZpEpi)
                                ptx::bulk_g2s(xs + C::kOffAs + j * BN * 4, p.asum + int64_t(gc + j) * p.Mpad + row0,
                                              uint32_t(BN * 4), &xfull[rx.idx], pol_a);
                        }
                    }
                }
                __syncwarp();
                rx.next<C::NX>();
            }
        }
    } else if (warp == 1) {
        // ======================= TMEM allocation + MMA issuer ==================
        if (!(dbg_bits(p) & 16)) ptx::tmem_alloc<C::kTmemCols>(tmem_holder);  // dbg&16 (with &8): launch-floor probe
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tmem_ready);
        ptx::tc_fence_after();
        const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_holder);
        const uint32_t idesc4 = idesc_i8(BN, !C::kZpEpi, true);  // kZpEpi: raw u4 codes as u8
        const uint32_t idesc8 = p.idesc8 | ((uint32_t(BN) >> 3) << 17);
        Ring rs, ra, rt, rx;
        int n = 0;
        for (int pk = 0;; ++pk) {
            Unit U;
            if (!piece(pk, U)) break;
            for (int i = 0; i < U.nch; ++i, ++n) {
                int gc, cg;
                chunk_at(U, i, gc, cg);
                // the weight stage is read here only for sub8 chunks (A in SMEM);
                // sub4 weight stages are released by the converter alone
                if (U.ti.is8) ptx::mbar_wait(&full[rs.idx], rs.ph);
                if (lane == 0) trace_chunk(p, 7, n);
                ptx::mbar_wait(&xfull[rx.idx], rx.ph);
                if (lane == 0) trace_chunk(p, 8, n);
                ptx::mbar_wait(&afull[ra.idx], ra.ph);
                if (lane == 0) trace_chunk(p, 9, n);
                ptx::mbar_wait(&tempty[rt.idx], rt.ph ^ 1u);
                ptx::tc_fence_after();
                if (lane == 0) trace_chunk(p, 1, n);
                const uint32_t st = ptx::smem_u32(stage(rs.idx));
                const uint32_t xs = ptx::smem_u32(xstage(rx.idx));
                if (elect_one()) {
                    if (!(dbg_bits(p) & 4)) {
                        for (int j = 0; j < cg; ++j) {
                            const uint32_t d_tmem = tmem_base + uint32_t((rt.idx * GPS + j) * BN);
                            const uint32_t b_addr = xs + j * (BN * 128);
                            if (U.ti.is8) {
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
                    if (!C::kSaDirect) ptx::tc_commit(&xempty[rx.idx]);
                    if (U.ti.is8) ptx::tc_commit(&empty[rs.idx]);
                }
                __syncwarp();
                if (lane == 0) trace_chunk(p, 2, n);
                ra.next<NA>();
                rt.next<NT>();
                rs.next<NS>();
                rx.next<C::NX>();
            }
        }
    } else if (warp >= 4 && warp < 4 + 4 * NC) {
        // ============ converter (sub4 -> int8 A tiles in TMEM; scales -> meta ring) ============
        const int wg = (warp - 4) >> 2;        // converter warpgroup: takes groups j = wg, wg+NC, ...
        const int r = (warp & 3) * 32 + lane;  // weight row = TMEM lane
        ptx::mbar_wait(tmem_ready, 0);
        ptx::tc_fence_after();
        const uint32_t tmem_row = *reinterpret_cast<volatile uint32_t*>(tmem_holder) + (uint32_t((warp & 3) * 32) << 16);
        Ring rs, ra, rm, rx;
        int n = 0;
        for (int pk = 0;; ++pk) {
            Unit U;
            if (!piece(pk, U)) break;
            for (int i = 0; i < U.nch; ++i, ++n) {
                int gc, cg;
                chunk_at(U, i, gc, cg);
                // (1) every chunk (sub8 too — a role that skipped chunks could run two
                // phases ahead of a barrier and read an older phase's parity as
                // complete): pull this thread's codes / zero point / scale out of the
                // weight stage into registers and release the stage at once, so the
                // weight stream never waits for the TMEM rings or the epilogue
                constexpr int JPW = (GPS + NC - 1) / NC;  // groups per converter warpgroup
                ptx::mbar_wait(&full[rs.idx], rs.ph);
                if (threadIdx.x == 128) trace_chunk(p, 5, n);
                const uint8_t* st = stage(rs.idx);
                uint4 raw[JPW][4];
                uint32_t kk[JPW];
                float swv[JPW];
#pragma unroll
                for (int jj = 0; jj < JPW; ++jj) {
                    const int j = wg + jj * NC;
                    if (j >= cg) break;
                    if (!U.ti.is8) {
                        const uint8_t* blk = st + j * kBlock4Bytes;
#pragma unroll
                        for (int q = 0; q < 4; ++q) raw[jj][q] = *reinterpret_cast<const uint4*>(blk + q * 2048 + r * 16);
                        kk[jj] = C::kZpEpi ? uint32_t(blk[kCodes4Bytes + 512 + r])
                                           : uint32_t(128 - blk[kCodes4Bytes + 512 + r]) * 0x01010101u;
                        swv[jj] = reinterpret_cast<const float*>(blk + kCodes4Bytes)[r];
                    } else {
                        swv[jj] = reinterpret_cast<const float*>(st + j * kBlock8Bytes + kCodes8Bytes)[r];
                        kk[jj] = 0u;
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(&empty[rs.idx]);
                    // sub4: the weight stage has no other reader — stand in for the MMA's arrival
                    if (!U.ti.is8 && threadIdx.x == 128) ptx::mbar_arrive(&empty[rs.idx]);
                }
                // (2) convert into a free TMEM A slot, scales into a free meta slot
                ptx::mbar_wait(&aempty[ra.idx], ra.ph ^ 1u);
                ptx::mbar_wait(&mempty[rm.idx], rm.ph ^ 1u);
                if (threadIdx.x == 128) trace_chunk(p, 6, n);
                float* msw = meta + rm.idx * (C::kMetaSlot / 4);
#pragma unroll
                for (int jj = 0; jj < JPW; ++jj) {
                    const int j = wg + jj * NC;
                    if (j >= cg) break;
                    if (!U.ti.is8) {
                        uint32_t v[32];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t w4[4] = {raw[jj][q].x, raw[jj][q].y, raw[jj][q].z, raw[jj][q].w};
#pragma unroll
                            for (int e2 = 0; e2 < 4; ++e2) {
                                if constexpr (C::kZpEpi) {  // widen only: bytes c (zero point applied in the epilogue)
                                    v[q * 8 + 2 * e2] = w4[e2] & 0x0F0F0F0Fu;
                                    v[q * 8 + 2 * e2 + 1] = (w4[e2] >> 4) & 0x0F0F0F0Fu;
                                } else {
                                    unpack_word(w4[e2], kk[jj], v[q * 8 + 2 * e2], v[q * 8 + 2 * e2 + 1]);
                                }
                            }
                        }
                        if (!(dbg_bits(p) & 2)) ptx::tmem_st32(tmem_row + C::kACol0 + uint32_t((ra.idx * GPS + j) * 32), v);
                    }
                    msw[j * 128 + r] = swv[jj];
                    if constexpr (C::kZpEpi) reinterpret_cast<int32_t*>(msw)[C::kMetaZp + j * 128 + r] = -int32_t(kk[jj]);  // -z
                }
                if constexpr (C::kZpEpi) {
                    // a short last chunk: zero the unused groups' scales, so the decode
                    // epilogue runs all GPS groups without branches (their terms are
                    // exactly +0: finite int -> f32 times a zero scale)
#pragma unroll
                    for (int jj = 0; jj < JPW; ++jj) {
                        const int j = wg + jj * NC;
                        if (j >= cg && j < GPS) {
                            msw[j * 128 + r] = 0.0f;
                            reinterpret_cast<int32_t*>(msw)[C::kMetaZp + j * 128 + r] = 0;
                        }
                    }
                }
                if ((kSa || C::kZpEpi) && wg == 0 && !C::kSaDirect) {
                    ptx::mbar_wait(&xfull[rx.idx], rx.ph);
                    if (r < cg * BN) {
                        if (kSa) msw[C::kMetaSa + r] = reinterpret_cast<const float*>(xstage(rx.idx) + C::kOffSa)[r];
                        if constexpr (C::kZpEpi)
                            reinterpret_cast<int32_t*>(msw)[C::kMetaAs + r] =
                                reinterpret_cast<const int32_t*>(xstage(rx.idx) + C::kOffAs)[r];
                    } else if (C::kZpEpi && r < GPS * BN) {
                        if (kSa) msw[C::kMetaSa + r] = 0.0f;
                        reinterpret_cast<int32_t*>(msw)[C::kMetaAs + r] = 0;
                    }
                }
                if (!U.ti.is8) ptx::tmem_wait_st();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(&mfull[rm.idx]);
                    ptx::mbar_arrive(&afull[ra.idx]);
                }
                if (threadIdx.x == 128) trace_chunk(p, 3, n);
                ra.next<NA>();
                rm.next<C::NM>();
                rs.next<NS>();
                rx.next<C::NX>();
            }
        }
    } else if (int(threadIdx.x) >= C::kEpiThread0) {
        // ================================ epilogue ================================
        const int et = threadIdx.x - C::kEpiThread0;  // 0 .. 128*NE-1
        const int e = et >> 7;                        // epilogue warpgroup
        const int wq = warp & 3;                      // TMEM lane quarter this warp may access
        const int r = wq * 32 + lane;                 // tile row (= TMEM lane)
        const int c0 = e * BNE;                       // first token column of this warpgroup
        ptx::mbar_wait(tmem_ready, 0);
        ptx::tc_fence_after();
        const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_holder);
        griddep_wait();  // scales / output of this launch are ours now
        Ring rt, rm, rx;
        int n = 0;
        for (int pk = 0;; ++pk) {
            Unit U;
            if (!piece(pk, U)) break;
            const Work& wk = U.wk;
            const TileInfo& ti = U.ti;
            const int64_t m0 = int64_t(wk.tb) * BN + c0;  // first token of this warpgroup
            constexpr bool kPair = (MODE == kFastGroup || MODE == kFastToken);
            float acc[BNE];
            float2 acc2[kPair ? BNE / 2 : 1];  // FAST modes accumulate in f32x2 pairs
            if constexpr (kPair) {
#pragma unroll
                for (int j = 0; j < BNE / 2; ++j) acc2[j] = make_float2(0.0f, 0.0f);
            } else {
#pragma unroll
                for (int j = 0; j < BNE; ++j) acc[j] = 0.0f;
            }
            float sat[MODE == kExactToken ? BNE : 1];  // per-token s_a of this warpgroup's tokens
            if constexpr (MODE == kExactToken) {
#pragma unroll
                for (int j = 0; j < BNE; ++j) sat[j] = m0 + j < p.M ? __ldg(p.sa + m0 + j) : 0.0f;
            }
            for (int i = 0; i < U.nch; ++i, ++n) {
                int gc, cg;
                chunk_at(U, i, gc, cg);
                ptx::mbar_wait(&mfull[rm.idx], rm.ph);
                if constexpr (C::kSaDirect) ptx::mbar_wait(&xfull[rx.idx], rx.ph);  // (complete: the MMA waited it)
                // activation scales [GPS][BN] (+ code sums): the stage itself, or the meta copy
                const float* sa_base = C::kSaDirect ? reinterpret_cast<const float*>(xstage(rx.idx) + C::kOffSa)
                                                    : meta + rm.idx * (C::kMetaSlot / 4) + C::kMetaSa;
                const int32_t* as_base = C::kSaDirect ? reinterpret_cast<const int32_t*>(xstage(rx.idx) + C::kOffAs)
                                                      : reinterpret_cast<const int32_t*>(meta + rm.idx * (C::kMetaSlot / 4)) + C::kMetaAs;
                ptx::mbar_wait(&tfull[rt.idx], rt.ph);
                ptx::tc_fence_after();
                if (n == 0 && et == 0) trace(p, 3);
                if (et == 0) trace_chunk(p, 13, n);
                const float* msw = meta + rm.idx * (C::kMetaSlot / 4);
                if constexpr (kPair && (BNE == 16 || BNE == 8)) {
                    // decode: two groups' sums in flight per wait (register budget)
                    // every group of the chunk, no branches: a short chunk's unused
                    // groups carry zero scales (converter), so they add exactly +0
#pragma unroll
                    for (int j0 = 0; j0 < GPS; j0 += 2) {
                        if (dbg_bits(p) & 1) break;
                        uint32_t v[2][BNE];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint32_t ta = tmem_base + (uint32_t(wq * 32) << 16) + uint32_t((rt.idx * GPS + j0 + h) * BN + c0);
                            if constexpr (BNE == 16) ptx::tmem_ld16(ta, v[h]);
                            else ptx::tmem_ld8(ta, v[h]);
                        }
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int j = j0 + h;
                            const float sw = msw[j * 128 + r];
                            const float2 sw2 = pk2(sw, sw);
                            const float* sav = sa_base + j * BN + c0;
                            if constexpr (C::kZpEpi) {  // S = sum a c - z sum a (exact int32)
                                const int32_t zr = reinterpret_cast<const int32_t*>(msw)[C::kMetaZp + j * 128 + r];
                                const int32_t* asv = as_base + j * BN + c0;
#pragma unroll
                                for (int q = 0; q < BNE; ++q) v[h][q] = uint32_t(int32_t(v[h][q]) + zr * asv[q]);  // zr = -z
                            }
#pragma unroll
                            for (int q = 0; q < BNE; q += 2) {
                                const float2 g2 = pk2(__int2float_rn(int32_t(v[h][q])), __int2float_rn(int32_t(v[h][q + 1])));
                                if constexpr (MODE == kFastGroup)
                                    acc2[q / 2] = fma2(g2, mul2(*reinterpret_cast<const float2*>(sav + q), sw2), acc2[q / 2]);
                                else
                                    acc2[q / 2] = fma2(g2, sw2, acc2[q / 2]);
                            }
                        }
                    }
                } else
                for (int j = 0; j < cg; ++j) {
                    const float sw = msw[j * 128 + r];
                    const float* sav = sa_base + j * BN + c0;
                    const float2 sw2 = pk2(sw, sw);
                    const uint32_t tcol = uint32_t((rt.idx * GPS + j) * BN + c0);
#ifndef MQ_CW64
#define MQ_CW64 64
#endif
                    // TMEM columns per tcgen05.wait::ld: two 16-column loads in flight per wait
                    // for 128-token tiles (register budget: 32 keeps 128 registers without spills;
                    // M = 512 stack -5%, M = 256 -2.5%), MQ_CW64 for 64-token tiles (64: -0.7..2% at M 33-64)
                    constexpr int CW = BNE < 16 ? BNE : (BN == 64 ? MQ_CW64 : (BNE >= 32 ? 32 : 16));
#pragma unroll
                    for (int ch = 0; ch < BNE / CW; ++ch) {
                        if (dbg_bits(p) & 1) break;
                        uint32_t v[CW];
                        if constexpr (CW >= 16) {
#pragma unroll
                            for (int h = 0; h < CW / 16; ++h)
                                ptx::tmem_ld16(tmem_base + (uint32_t(wq * 32) << 16) + tcol + ch * CW + h * 16,
                                               *reinterpret_cast<uint32_t(*)[16]>(v + h * 16));
                        } else {
                            ptx::tmem_ld8(tmem_base + (uint32_t(wq * 32) << 16) + tcol + ch * CW, v);
                        }
                        ptx::tmem_wait_ld();
                        if constexpr (C::kZpEpi) {  // S = sum a c - z sum a (exact int32)
                            const int32_t zr = reinterpret_cast<const int32_t*>(msw)[C::kMetaZp + j * 128 + r];
                            const int32_t* asv = as_base + j * BN + c0 + ch * CW;
#pragma unroll
                            for (int q = 0; q < CW; ++q) v[q] = uint32_t(int32_t(v[q]) + zr * asv[q]);  // zr = -z
                        }
                        if constexpr (MODE == kDumpPartials) {
                            if (r < ti.rows) {
#pragma unroll
                                for (int q = 0; q < CW; ++q) {
                                    const int64_t m = m0 + ch * CW + q;
                                    if (m < p.M)
                                        p.partials[(int64_t(gc + j) * p.M + m) * p.partial_rows + ti.first + r] =
                                            int32_t(v[q]);
                                }
                            }
                        } else if constexpr (kPair) {
#pragma unroll
                            for (int q = 0; q < CW; q += 4) {
                                const int jj = ch * CW + q;
                                // exact int -> f32 (|S| < 2^22), two lanes per FFMA2; four
                                // activation scales per 16-byte shared load
                                const float2 g2a = pk2(__int2float_rn(int32_t(v[q])), __int2float_rn(int32_t(v[q + 1])));
                                const float2 g2b = pk2(__int2float_rn(int32_t(v[q + 2])), __int2float_rn(int32_t(v[q + 3])));
                                if constexpr (MODE == kFastGroup) {
                                    const float4 sa4 = *reinterpret_cast<const float4*>(sav + jj);
                                    acc2[jj / 2] = fma2(g2a, mul2(make_float2(sa4.x, sa4.y), sw2), acc2[jj / 2]);
                                    acc2[jj / 2 + 1] = fma2(g2b, mul2(make_float2(sa4.z, sa4.w), sw2), acc2[jj / 2 + 1]);
                                } else {
                                    acc2[jj / 2] = fma2(g2a, sw2, acc2[jj / 2]);
                                    acc2[jj / 2 + 1] = fma2(g2b, sw2, acc2[jj / 2 + 1]);
                                }
                            }
                        } else {
#pragma unroll
                            for (int q = 0; q < CW; ++q) {
                                const float gs = __int2float_rn(int32_t(v[q]));  // exact: |S| < 2^22
                                const int jj = ch * CW + q;
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
                if (lane == 0) {
                    ptx::mbar_arrive(&tempty[rt.idx]);
                    ptx::mbar_arrive(&mempty[rm.idx]);
                    if constexpr (C::kSaDirect) ptx::mbar_arrive(&xempty[rx.idx]);
                }
                if (et == 0) trace_chunk(p, 4, n);
                rt.next<NT>();
                rm.next<C::NM>();
                rx.next<C::NX>();
            }
            if (et == 0) trace(p, 4);
            if constexpr (kPair) {
#pragma unroll
                for (int j = 0; j < BNE / 2; ++j) {
                    acc[2 * j] = acc2[j].x;
                    acc[2 * j + 1] = acc2[j].y;
                }
            }
            if (MODE == kDumpPartials || U.nch == 0) continue;
            // scatter this thread's row to its original output column
            const int col = (r < ti.rows && !(dbg_bits(p) & 128)) ? __ldg(p.colmap + wk.tile * kTileRows + r) : -1;
            auto store_acc = [&]() { store_tokens<BNE, MODE, PEER>(p, m0, col, acc); };
            if (wk.S == 1) {  // whole-K tile
                if (et == 0) trace_chunk(p, 11, n);
                store_acc();
                if (et == 0) trace_chunk(p, 12, n);
                continue;
            }
            if constexpr (BN >= 64 && (MODE == kFastGroup || MODE == kFastToken)) {
                // a split piece of a wide tile, out of line (its registers would
                // push the 64-accumulator loop into spills): stream-K head / tail
                // (the head scatters the joined tile from registers here), or a
                // K-slice of the unit schedule
                float tmp[BNE];
#pragma unroll
                for (int j = 0; j < BNE; ++j) tmp[j] = acc[j];
                if constexpr (SPL) {
                    split_join_wide<BN, BNE, NE, MODE, PEER>(p, wk, U.key, tmp, r, c0, et, s_last, col, m0);
                } else {
                    if (!sk_piece_done<BN, BNE, NE>(p, wk, tmp, r, c0, et, s_last)) continue;
#pragma unroll
                    for (int j = 0; j < BNE; ++j) acc[j] = tmp[j];
                    store_acc();
                }
                continue;
            }
            // split item at decode (token tiles <= 32): publish this piece's
            // partial tile [128][BN] (a thread's tokens are contiguous -> float4),
            // count arrivals; the last piece sums all S partials in piece order
            // (deterministic) and scatters them. Unit schedule: the item's slices
            // are units cta0 .. cta0 + S - 1 (slot = unit). Decode stream-K: the
            // item's pieces lie on consecutive CTAs b_f .. b_l; CTA b's first
            // piece uses slot 2b, its last (a head cut at the range end) 2b + 1.
            if constexpr (BN <= 32) {
            int S = wk.S, my = U.key, b_f = wk.cta0;
            if (kSkPath && p.sk) {
                b_f = sk_cta_of(p, uint32_t(wk.item) << 8);
                S = sk_cta_of(p, (uint32_t(wk.item) << 8) | uint32_t(p.G - 1)) - b_f + 1;
                my = 2 * int(blockIdx.x) + (pk == 0 ? 0 : 1);
            }
            if (et == 0) trace_chunk(p, 11, n);
            float4* mine = reinterpret_cast<float4*>(p.part + int64_t(my) * (BN * 128) + r * BN + c0);
#pragma unroll
            for (int j = 0; j < BNE / 4; ++j)
                __stcg(mine + j, make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]));
            named_bar_sync(2, 128 * NE);
            if (et == 0) {
                // release: this CTA's partial (ordered before by bar.sync) is
                // visible at gpu scope before the count; acquire: the other
                // pieces' partials are visible to the reduction below (ordered
                // after by bar.sync; ld.cg reads L2) — no full fences
                uint32_t prev;
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.cnt + wk.item) : "memory");
                *s_last = prev == uint32_t(S - 1);
                if (prev == uint32_t(S - 1)) p.cnt[wk.item] = 0u;  // re-arm for the next launch
            }
            named_bar_sync(2, 128 * NE);
            const bool last = *s_last != 0;
            named_bar_sync(2, 128 * NE);  // s_last is reused by the next unit
            if (et == 0) trace_chunk(p, 12, n);
            if (last) {
                // slot of piece j of the item (in order)
                const bool first_own = kSkPath && p.sk && (p.skb[b_f] >> 8) == uint32_t(wk.item);
                auto slot_of = [&](int j) -> int64_t {
                    if (!(kSkPath && p.sk)) return int64_t(b_f) + j;
                    return int64_t(2 * (b_f + j)) + ((j == 0 && !first_own) ? 1 : 0);
                };
                constexpr int V = BNE / 4;      // float4s per piece
                constexpr int SB = 32 / BNE;    // pieces per batch: every load of a batch in flight
                float sum[BNE];
                for (int s0 = 0; s0 < S; s0 += SB) {
                    float4 t[SB][V];
#pragma unroll
                    for (int s2 = 0; s2 < SB; ++s2)
                        if (s0 + s2 < S) {
                            const float4* src = reinterpret_cast<const float4*>(p.part + slot_of(s0 + s2) * (BN * 128) + r * BN + c0);
#pragma unroll
                            for (int q = 0; q < V; ++q) t[s2][q] = __ldcg(src + q);
                        }
#pragma unroll
                    for (int s2 = 0; s2 < SB; ++s2) {
                        if (s0 + s2 >= S) break;
#pragma unroll
                        for (int q = 0; q < V; ++q) {
                            const float tv[4] = {t[s2][q].x, t[s2][q].y, t[s2][q].z, t[s2][q].w};
#pragma unroll
                            for (int e4 = 0; e4 < 4; ++e4)
                                sum[4 * q + e4] = (s0 + s2 == 0) ? tv[e4] : __fadd_rn(sum[4 * q + e4], tv[e4]);
                        }
                    }
                }
                if (et == 0) trace_chunk(p, 15, 8);
                store_tokens<BNE, MODE, PEER>(p, m0, col, sum);
            }
            }  // BN <= 32
        }
    }

    if (threadIdx.x == C::kEpiThread0) {
        trace(p, 5);
        trace_chunk(p, 15, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) trace(p, 6);
    if (warp == 1 && !(dbg_bits(p) & 16)) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<C::kTmemCols>(*reinterpret_cast<volatile uint32_t*>(tmem_holder));
    }
}

template <int BN, void (*KERN)(GemmParams)>
cudaError_t launch_kernel(const GemmParams& p, bool pdl, cudaStream_t stream) {
    using C = TcCfg<BN>;
    static thread_local uint64_t configured = 0;  // per kernel: device ordinal bitmask
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(configured >> dev & 1)) {
        cudaError_t e = cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        if (e != cudaSuccess) return e;
        configured |= uint64_t(1) << dev;
    }
    if (p.units <= 0 || p.grid <= 0) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(p.grid));
    cfg.blockDim = dim3(C::kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, KERN, p);
}

template <int BN, int MODE, int PEER>
cudaError_t launch_bn_mode(const GemmParams& p, bool pdl, cudaStream_t stream) {
    if constexpr (BN >= 64 && (MODE == kFastGroup || MODE == kFastToken)) {
        if (!p.sk && (p.S4 > 1 || p.S8 > 1))
            return launch_kernel<BN, mixed_gemm_tc_kernel<BN, MODE, 1, PEER>>(p, pdl, stream);
    }
    if constexpr (BN <= 32 && (MODE == kFastGroup || MODE == kFastToken)) {
        if (p.sk) return launch_kernel<BN, mixed_gemm_tc_kernel<BN, MODE, 1, PEER>>(p, pdl, stream);  // decode stream-K
    }
    return launch_kernel<BN, mixed_gemm_tc_kernel<BN, MODE, 0, PEER>>(p, pdl, stream);
}

template <int BN, int PEER>
cudaError_t launch_bn(const GemmParams& p, int mode, bool pdl, cudaStream_t s) {
    switch (mode) {
        case kExactGroup: return launch_bn_mode<BN, kExactGroup, PEER>(p, pdl, s);
        case kFastGroup: return launch_bn_mode<BN, kFastGroup, PEER>(p, pdl, s);
        case kFastToken: return launch_bn_mode<BN, kFastToken, PEER>(p, pdl, s);
        case kExactToken: return launch_bn_mode<BN, kExactToken, PEER>(p, pdl, s);
        default:
            if constexpr (PEER) return cudaErrorInvalidValue;  // partial dumps have no peers
            else return launch_bn_mode<BN, kDumpPartials, PEER>(p, pdl, s);
    }
}

// token-tile dispatch of the plain (PEER = 0) or fused-gather (PEER = 1) kernels
template <int PEER>
cudaError_t launch_tc(const GemmParams& p, int token_tile, int mode, bool pdl, cudaStream_t stream) {
    switch (token_tile) {
        case 16: return launch_bn<16, PEER>(p, mode, pdl, stream);
        case 32: return launch_bn<32, PEER>(p, mode, pdl, stream);
        case 64: return launch_bn<64, PEER>(p, mode, pdl, stream);
        case 128: return launch_bn<128, PEER>(p, mode, pdl, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace
}  // namespace mq

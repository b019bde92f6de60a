// mq_layer.cpp — device layer handle, the one-time packer into the engine's
// HBM layout (mq_layout.cuh), launch planning and the forward entry points of
// the C ABI.
//
// The reference re-prepacks both sub-problems on every forward call
// (proj/src/gemm.cpp:148-149, ~45% of its call time at M=16); here
// packing happens once in mq_layer_create and forwards only stream weights.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../kernels/mq_kernels.hpp"
#include "mq_internal.hpp"

using namespace mq;

struct mq_layer_s {
    int device = 0;
    int num_sms = 148;
    int64_t N = 0, K = 0;
    int group = 128;
    int G = 0;
    int64_t n8 = 0, n4 = 0;  // local (shard) rows
    int32_t rank = 0, world = 1;
    int64_t shard_cols = 0;
    int w8_mode = MQ_W8_REFERENCE;
    int64_t tiles8 = 0, tiles4 = 0;
    int split4[3] = {1, 1, 1};          // K-split chosen once at create (choose_split) for token
    int split8[3] = {1, 1, 1};          // tiles <= 32 (decode), 64 and 128 (one token block)
    double split_span[3] = {0, 0, 0};   // the chosen split's modelled busiest-CTA cost (sub4 groups)
    uint8_t* d_wq = nullptr;
    int32_t* d_colmap = nullptr;
    int32_t* d_colmap_orig = nullptr;   // sharded layers: original output column of every tile row
    int32_t* d_shard_colmap = nullptr;  // sharded layers: device copy of shard_colmap (gather permute)
    int64_t bytes_wq = 0, stream_bytes = 0;
    std::vector<TileDesc> tiles;        // host copy (packing / accounting)
    std::vector<int32_t> shard_colmap;  // [world * shard_cols]
    std::mutex mu;                      // guards the internal workspace
    void* d_ws = nullptr;               // internal scratch (workspace = NULL)
    size_t ws_bytes = 0;
    std::vector<void*> retired;         // outgrown internal workspaces: freed at destroy, never
                                        // while a launch queued by another caller may use them
};

namespace {

unsigned long long* g_trace_buf = nullptr;

mq_status cuda_fail(cudaError_t e, const char* what) {
    return fail(MQ_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CU_TRY(expr)                                        \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
    } while (0)

// Token tile per launch: 16 / 32 / 64 / 128 by M, except on a narrow, short-K
// layer (G <= 64, where K-splitting has little to split), which takes the
// smallest tile whose token blocks x tiles still fit one round of the SMs:
// more, smaller items instead of idle SMs (graph-timed launches, Llama-8B):
// qkv 6144x4096 at M = 48: 64 -> 16-token tiles (147 items) 17.0 -> 12.4 us;
// at M = 80-96: 32-token tiles 18.1 -> 15.9 us; o 4096x4096 at M = 64: 16-token
// tiles 13.7 -> 12.4 us, at M = 128: 32-token tiles 17.6 -> 15.8 us; qkv at
// M = 128: 64-token tiles 23.7 -> 18.2 us. Long-K layers split K instead (down
// 4096x14336 keeps its tile).
#ifndef MQ_TT64_MAX
#define MQ_TT64_MAX 256
#endif
int auto_token_tile(const mq_layer_s* L, int64_t M, bool per_layer) {
    if (M <= 16) return 16;
    if (M <= 32) return 32;
    static const int rule = [] {
        const char* v = std::getenv("MQ_TT_RULE");  // development A/B: 0 off, 1 64 only, 2 all
        return v ? std::atoi(v) : 2;
    }();
    const int64_t T = L->tiles8 + L->tiles4;
    if (per_layer && rule && L->G <= 64 && M <= int64_t(MQ_TT64_MAX))
        for (int bn = rule >= 2 ? 16 : 64; bn <= 64; bn *= 2)
            if ((M + bn - 1) / bn * T <= L->num_sms) return bn;
    return M <= 64 ? 64 : 128;
}

struct Plan {
    int bn, tb, mode, per_token, S4, S8, units, grid;
    int64_t Mpad;
    bool pdl, rotate, sk, no_spin, f16;
    const mq_layer_s* pf_layer;
    int64_t pf_bytes;
    std::vector<uint32_t> skb;  // stream-K boundaries [grid + 1]
};

// Stream-K plan (mq_kernels.hpp): equal cost per CTA over the item sequence,
// boundaries rounded down to the tile's chunk size. Used by FAST token-tiled
// launches when the unit schedule's last round would leave CTAs idle for
// longer than a cut item costs; every CTA range covers at least one item's
// length, so an item is cut at most once (head + tail, sk_piece_done).
// Prefill stream-K: a sub8 item's extra cost, in sub4 groups — its epilogue
// scatters to the sparse salient columns (~20 sectors per warp store instead
// of 2). Measured on the Llama-8B shapes at M = 512: 4 balances gate_up
// (142 -> 132 us); 8 pushes qkv below stream_k_pays' cover bound.
int sk_extra8() {
    static const int e = [] {
        const char* v = std::getenv("MQ_SK_E8");  // development override
        return v ? std::atoi(v) : 4;
    }();
    return e;
}

bool stream_k_pays(const mq_layer_s* L, const Plan* pl, bool force) {
    const int64_t G = L->G, items = int64_t(pl->tb) * (L->tiles8 + L->tiles4);
    const int grid = std::min<int>(L->num_sms, kSkMax);
    const int64_t E = sk_extra8();
    // groups per CTA (a sub8 item costs G + E sub4 groups: its scattered stores)
    const double per_cta = double(pl->tb * (L->tiles8 * (G + E) + L->tiles4 * G)) / grid;
    // every CTA range (less the chunk rounding of its ends) must cover a whole
    // item's length, so no item is cut twice (head + tail, sk_piece_done)
    if (per_cta * double(G) / double(G + E) < double(G + 2 * gemm_gps(pl->bn) + 1)) return false;
    if (force) return true;
    const int64_t rounds = (items + grid - 1) / grid;
    // measured (BN = 64 and 128): publish + join + tail of a cut item ~ 16 groups
    const double cut_cost = 16.0;
    return per_cta + cut_cost < double(rounds * G);
}

// Decode (token tiles <= 32, one token block) stream-K: every CTA streams the
// same bytes (a sub8 group costs two sub4 groups); an item cut across CTAs is
// joined by its last piece (any number of pieces, see the kernel). Measured on
// the Llama decode shapes it loses to the unit schedule even where it balances
// better (gate_up 28672x4096: 21.9 vs 18.6 us): a join in the middle of a
// CTA's range stalls its epilogue, and decode is bound by the per-SM pipeline.
// So the unit schedule stays the default and schedule = 2 forces stream-K.
bool decode_stream_k_pays(const mq_layer_s*, bool force) { return force; }

void plan_stream_k(const mq_layer_s* L, Plan* pl) {
    const int64_t G = L->G, T8 = L->tiles8, T4 = L->tiles4, T = T8 + T4;
    // cost of a sub8 / sub4 group: decode streams twice the bytes for a sub8
    // group; prefill spreads a sub8 item's extra cost E over its G groups
    const int64_t c8 = pl->bn <= 32 ? 2 : G + sk_extra8(), c4 = pl->bn <= 32 ? 1 : G;
    const int gps = gemm_gps(pl->bn), gps8 = gps / 2 > 0 ? gps / 2 : 1;
    const int64_t ctb = T8 * G * c8 + T4 * G * c4, total = ctb * pl->tb;
    const int64_t chunks = (T8 * ((G + gps8 - 1) / gps8) + T4 * ((G + gps - 1) / gps)) * pl->tb;
    const int grid = static_cast<int>(std::min<int64_t>({L->num_sms, kSkMax, chunks}));
    pl->skb.assign(size_t(grid) + 1, 0);
    for (int b = 0; b < grid; ++b) {
        const int64_t x = total * b / grid;
        const int64_t tb = x / ctb, rr = x - tb * ctb;
        int64_t t, g;
        if (rr < T8 * G * c8) {
            t = rr / (G * c8);
            g = (rr - t * G * c8) / c8;
            g = g / gps8 * gps8;
        } else {
            const int64_t r4 = rr - T8 * G * c8;
            t = T8 + r4 / (G * c4);
            g = (r4 - (t - T8) * G * c4) / c4;
            g = g / gps * gps;
        }
        pl->skb[b] = static_cast<uint32_t>(((tb * T + t) << 8) | g);
    }
    pl->skb[grid] = static_cast<uint32_t>((int64_t(pl->tb) * T) << 8);
    // chunk rounding can make neighbouring boundaries equal: drop the empty
    // ranges, so the boundaries are strictly increasing (the decode join finds
    // an item's pieces as the CTAs between two boundary searches)
    pl->skb.erase(std::unique(pl->skb.begin(), pl->skb.end()), pl->skb.end());
    pl->grid = static_cast<int>(pl->skb.size()) - 1;
    pl->sk = true;
}

// K-slices per item (mq_kernels.hpp schedule). Exact mode keeps the
// reference's ascending group order per output, so it never splits; token-
// tiled (prefill) launches use one tile per unit (and stream-K, below). Decode
// (best_split, once per layer: it is off the per-call host path) picks the
// power-of-two split (S4 for sub4 tiles, S8 in {S4, 2 S4} for sub8
// tiles, whose groups stream twice the bytes) that minimises the busiest CTA's
// streamed bytes under the persistent grid's round-robin unit assignment, plus
// a per-unit cost and a reduction cost for split items (cost model in sub4
// groups; constants measured on the Llama decode shapes).
// kind 0: decode token tiles, where a sub8 group streams twice a sub4 group's
// bytes; kind 1 / 2: 64 / 128-token tiles, where every group costs the same
// rescale work and a split join moves a 32 / 64 KB partial
void best_split(mq_layer_s* L, int kind) {
    const double kUnitCost = 2.0, kSplitCost = kind == 0 ? 4.0 : kind == 1 ? 8.0 : 16.0, k8 = kind == 0 ? 2.0 : 1.0;
    // (charging sub8 items their scatter cost here too, sk_extra8, moves the
    // 64-token launches' plans to S8 = 2 S4: 2.3 us faster over the four
    // projections launched alone, no faster inside the PDL-chained stack)
    const int64_t G = L->G, T8 = L->tiles8, T4 = L->tiles4;
    double best = 1e30;
    for (int S4 = 1; S4 <= 8; S4 *= 2) {
        for (int S8 = S4; S8 <= 2 * S4; S8 *= 2) {
            if (S4 > G || S8 > G) continue;
            const int64_t u8 = T8 * S8, units = u8 + T4 * S4;
            const int64_t grid = std::min<int64_t>(units, L->num_sms);
            // wide tiles: split items only when every slice runs in one round (the together-mode join)
            if (kind > 0 && S8 > 1 && units > L->num_sms) continue;
            const double c8 = k8 * double(G) / S8 + kUnitCost + (S8 > 1 ? kSplitCost : 0.0);
            const double c4 = double(G) / S4 + kUnitCost + (S4 > 1 ? kSplitCost : 0.0);
            double span = 0;
            for (int64_t b = 0; b < grid; ++b) {  // CTA b runs units b, b + grid, ...
                const int64_t n = (units - b + grid - 1) / grid;
                const int64_t n8 = u8 > b ? (u8 - b + grid - 1) / grid : 0;
                span = std::max(span, double(n8) * c8 + double(n - n8) * c4);
            }
            if (span < best - 1e-9) {
                best = span;
                L->split4[kind] = S4;
                L->split8[kind] = S8;
                L->split_span[kind] = span;
            }
        }
    }
}

// The same model for tb > 1 token blocks of wide tiles when there are fewer
// items than SMs (prefill on a narrow layer): explicit round-robin over the
// tb x (sub8 slices, sub4 slices) unit sequence (<= 8 x #SM units).
void best_split_blocks(const mq_layer_s* L, int kind, int tb, int* S4o, int* S8o) {
    const double kUnitCost = 2.0, kSplitCost = kind == 1 ? 8.0 : 16.0;
    const int64_t G = L->G, T8 = L->tiles8, T4 = L->tiles4;
    double best = 1e30;
    std::vector<double> cta(size_t(L->num_sms));
    for (int S = 1; S <= 8; S *= 2) {
        if (S > G) break;
        const int64_t per_tb = (T8 + T4) * S, units = per_tb * tb;
        const int64_t grid = std::min<int64_t>(units, L->num_sms);
        if (S > 1 && units > L->num_sms) break;  // split items only within one round (see choose_split)
        std::fill(cta.begin(), cta.end(), 0.0);
        const double c = double(G) / S + kUnitCost + (S > 1 ? kSplitCost : 0.0);
        for (int64_t u = 0; u < units; ++u) cta[size_t(u % grid)] += c;
        const double span = *std::max_element(cta.begin(), cta.begin() + grid);
        if (span < best - 1e-9) {
            best = span;
            *S4o = *S8o = S;
        }
    }
}

void choose_split(const mq_layer_s* L, Plan* pl, int ksplit) {
    pl->S4 = pl->S8 = 1;
    if (pl->mode == kExactGroup || pl->mode == kExactToken || ksplit == 1) return;
    if (pl->tb > 1) {
        const int64_t items = int64_t(pl->tb) * (L->tiles8 + L->tiles4);
        if (pl->bn > 32 && ksplit == 0 && items < L->num_sms)
            best_split_blocks(L, pl->bn == 64 ? 1 : 2, pl->tb, &pl->S4, &pl->S8);
        return;
    }
    if (ksplit >= 2) {
        int best = 1;
        while (best * 2 <= ksplit) best *= 2;  // powers of two
        pl->S4 = best;
        pl->S8 = 2 * best;
        while (pl->S8 > 1 && pl->S8 > L->G) pl->S8 >>= 1;
        // wide token tiles: the slices of an item must run in one round (the
        // together-mode join); a multi-round split of 64/128-token tiles joins
        // through one CTA per tile and measured 3-20x slower
        while (pl->bn > 32 && (pl->S4 > 1 || pl->S8 > 1) &&
               (int64_t(pl->S8) * L->tiles8 + int64_t(pl->S4) * L->tiles4) * pl->tb > L->num_sms) {
            pl->S4 = std::max(pl->S4 >> 1, 1);
            pl->S8 = std::max(pl->S8 >> 1, 1);
        }
        return;
    }
    const int kind = pl->bn <= 32 ? 0 : pl->bn == 64 ? 1 : 2;  // best_split, computed once per layer
    pl->S4 = L->split4[kind];
    pl->S8 = L->split8[kind];
}

// shared_acts: the split API (mq_quantize_act_ws + mq_mixed_linear_ws), where one
// quantized activation feeds several layers, so the token tile (hence the EAL
// layout) must depend on M only, not on the layer
mq_status make_plan(const mq_layer_s* L, int64_t M, const mq_exec_opts* o, Plan* pl, bool shared_acts = false) {
    mq_exec_opts d{};
    if (!o) o = &d;
    const int act_group = o->act_group ? o->act_group : L->group;
    if (act_group == L->group && act_group < L->K) pl->per_token = 0;
    else if (act_group >= L->K) pl->per_token = 1;
    else if (act_group < 1)
        return fail(MQ_USAGE, "act_group must be >= 1");
    else
        return fail(MQ_USAGE, "activations and weights must share group boundaries (act group " +
                                  std::to_string(act_group) + ", weight group " + std::to_string(L->group) +
                                  "); per-token activations use act_group = K");
    if (o->mode != MQ_EXACT && o->mode != MQ_FAST) return fail(MQ_USAGE, "unknown mode");
    if (pl->per_token && L->K > kPerTokenKMax)
        return fail(MQ_USAGE, "per-token activations support K <= " + std::to_string(kPerTokenKMax) + " (K = " +
                                  std::to_string(L->K) + "); use group-wise activations (act_group = group size)");
    pl->no_spin = o->concurrent != 0;
    pl->f16 = o->act_scale_f16 != 0;
    pl->pf_layer = o->prefetch_next;
    pl->pf_bytes = o->prefetch_bytes;
    if (pl->pf_bytes < 0) return fail(MQ_USAGE, "prefetch_bytes must be >= 0");
    if (o->ksplit < 0 || o->ksplit > 8) return fail(MQ_USAGE, "ksplit must be 0 (auto), 1 (none) or a split <= 8");
    pl->bn = o->token_tile ? o->token_tile : auto_token_tile(L, M, !shared_acts);
    if (pl->bn != 16 && pl->bn != 32 && pl->bn != 64 && pl->bn != 128)
        return fail(MQ_USAGE, "token_tile must be 16, 32, 64 or 128");
    pl->tb = static_cast<int>((M + pl->bn - 1) / pl->bn);
    pl->Mpad = int64_t(pl->tb) * pl->bn;
    pl->mode = o->mode == MQ_EXACT ? (pl->per_token ? kExactToken : kExactGroup) : (pl->per_token ? kFastToken : kFastGroup);
    pl->pdl = o->no_pdl == 0;
    pl->rotate = o->mode == MQ_FAST;  // stagger the CTAs' (shared, L2-resident) activation reads
    choose_split(L, pl, o->ksplit);
    pl->units = static_cast<int>((int64_t(pl->S8) * L->tiles8 + int64_t(pl->S4) * L->tiles4) * pl->tb);
    pl->grid = std::min(pl->units, L->num_sms);
    pl->sk = false;
    // stream-K when the unit schedule's last round would leave CTAs idle
    if (o->schedule < 0 || o->schedule > 2) return fail(MQ_USAGE, "schedule must be 0 (auto), 1 (units) or 2 (stream-K)");
    const int64_t items = int64_t(pl->tb) * (L->tiles8 + L->tiles4);
    if (o->mode == MQ_FAST && o->ksplit == 0 && pl->bn >= 64 && pl->S4 == 1 && pl->S8 == 1 && L->G < 256 &&
        items * 256 < (int64_t(1) << 32) &&
        o->schedule != 1 && stream_k_pays(L, pl, o->schedule == 2))
        plan_stream_k(L, pl);
    if (o->mode == MQ_FAST && o->ksplit == 0 && pl->bn <= 32 && pl->tb == 1 && L->G < 256 && o->schedule != 1 &&
        decode_stream_k_pays(L, o->schedule == 2))
        plan_stream_k(L, pl);
    static const bool plan_log = std::getenv("MQ_PLAN_LOG") != nullptr;  // development
    if (plan_log)
        std::fprintf(stderr, "mq plan: N=%lld K=%lld M=%lld bn=%d tb=%d S4=%d S8=%d units=%d grid=%d sk=%d\n",
                     (long long)L->N, (long long)L->K, (long long)M, pl->bn, pl->tb, pl->S4, pl->S8, pl->units, pl->grid,
                     pl->sk ? 1 : 0);
    return MQ_OK;
}

// Forward workspace. [0, 32 KiB): arrival counters (kCntWords; every launch
// leaves them zero) | EAL codes [G][Mpad][128] | EAL scales [Ga][Mpad] | EAL
// code sums [G][Mpad] int32 | split-K / stream-K partial tiles. The counter
// region is the same for every layer and M, and the EAL offsets depend only on
// (K, Mpad, per_token): one workspace serves any sequence of launches (any M)
// and one quantized activation feeds several layers (mq_quantize_act_ws).
struct EalWs {
    size_t off_acts, off_sa, off_asum, off_part, off_part2, total;
};
EalWs eal_ws_layout(const mq_layer_s* L, const Plan& pl) {
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    EalWs w;
    w.off_acts = size_t(kCntWords) * 4;
    w.off_sa = w.off_acts + al(size_t(L->G) * size_t(pl.Mpad) * 128);
    const int64_t Ga = pl.per_token ? 1 : L->G;
    w.off_asum = w.off_sa + al(size_t(Ga) * size_t(pl.Mpad) * 4);
    w.off_part = w.off_asum + al(size_t(L->G) * size_t(pl.Mpad) * 4);
    const bool split = pl.S4 > 1 || pl.S8 > 1;
    const size_t tile = 128 * size_t(pl.bn) * 4;
    // decode stream-K: two slots per CTA (its first and last piece); prefill
    // stream-K: tail partials [grid + 1] then head partials [grid + 1]
    const size_t slots = pl.sk ? (pl.bn <= 32 ? 2 * (size_t(pl.grid) + 1) : size_t(pl.grid) + 1)
                               : split ? size_t(pl.units) : 0;
    w.off_part2 = w.off_part + al(slots * tile);
    w.total = w.off_part2 + (pl.sk && pl.bn > 32 ? al(slots * tile) : 0);
    return w;
}

void gemm_params(const mq_layer_s* L, const Plan& pl, int64_t M, void* Y, mq_dtype out_dtype, GemmParams* p) {
    std::memset(p, 0, sizeof(*p));
    p->T8 = static_cast<int32_t>(L->tiles8);
    p->T4 = static_cast<int32_t>(L->tiles4);
    p->n8 = L->n8;
    p->n4 = L->n4;
    p->G = L->G;
    p->TB = pl.tb;
    p->K = L->K;
    p->wq = L->d_wq;
    p->colmap = L->d_colmap;
    p->Mpad = pl.Mpad;
    p->M = M;
    p->Y = Y;
    p->out_dtype = out_dtype;
    p->ldy = L->world > 1 ? L->shard_cols : L->N;
    p->S4 = pl.S4;
    p->S8 = pl.S8;
    auto lg2 = [](int x) { int l = 0; while ((1 << l) < x) ++l; return l; };
    p->lgS4 = lg2(pl.S4);
    p->lgS8 = lg2(pl.S8);
    p->units = pl.units;
    p->grid = pl.grid;
    p->rotate = pl.rotate ? 1 : 0;
    p->T = static_cast<int32_t>(L->tiles8 + L->tiles4);
    p->sk = pl.sk ? 1 : 0;
    if (pl.sk) std::copy(pl.skb.begin(), pl.skb.end(), p->skb);
    p->idesc8 = idesc_i8(0, L->w8_mode == MQ_W8_SIGNED, true);
    if (pl.pf_layer && pl.pf_layer != L && pl.pf_layer->device == L->device) {
        // auto: the whole next layer, up to a third of L2 (the weight stream of
        // this launch is read evict-first, so prefetched lines survive it)
        const int64_t cap = pl.pf_bytes ? pl.pf_bytes : int64_t(40) << 20;
        p->pf = pl.pf_layer->d_wq;
        p->pf_bytes = std::min<int64_t>(cap, pl.pf_layer->bytes_wq) / 256 * 256;
    }
#ifdef MQ_DEV
    static const int dbg = [] {  // development builds: pipeline-stage bypass / trace bits
        const char* e = std::getenv("MQ_DBG");
        return e ? std::atoi(e) : 0;
    }();
#else
    constexpr int dbg = 0;
#endif
    p->dbg = dbg;
    if (dbg & 32) {
        static unsigned long long* tr = [] {
            unsigned long long* t = nullptr;
            cudaMalloc(&t, (148 * 8 + 1024) * sizeof(unsigned long long));
            cudaMemset(t, 0, (148 * 8 + 1024) * sizeof(unsigned long long));
            return t;
        }();
        p->trace = tr;
        g_trace_buf = tr;
    }
}

mq_status ensure_internal_ws(mq_layer_s* L, size_t bytes, cudaStream_t stream, void** ws) {
    std::lock_guard<std::mutex> lk(L->mu);
    if (L->ws_bytes < bytes) {
        cudaStreamCaptureStatus cs;
        if (stream && cudaStreamIsCapturing(stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
            return fail(MQ_USAGE, "internal workspace cannot grow during graph capture; pass a workspace");
        // the outgrown buffer may still be referenced by launches queued on other
        // streams: keep it until the layer is destroyed
        if (L->d_ws) L->retired.push_back(L->d_ws);
        L->d_ws = nullptr;
        L->ws_bytes = 0;
        void* buf = nullptr;
        CU_TRY(cudaMalloc(&buf, bytes));
        CU_TRY(cudaMemset(buf, 0, bytes));
        L->d_ws = buf;
        L->ws_bytes = bytes;
    }
    *ws = L->d_ws;
    return MQ_OK;
}

}  // namespace

namespace {
// Layer creation shared by the host packer (mq_layer_create: host reference
// layouts) and the device packer (mq_layer_create_device: reference layouts
// already in device memory, packed by wq_engine_kernel). Index maps are host
// arrays in both cases.
mq_status create_layer(const mq_layer_desc* d, const mq_layer_opts* opts, int device, bool dev_src,
                       cudaStream_t stream, mq_layer_t* out) {
    if (!out) return fail(MQ_USAGE, "out handle is null");
    if (mq_status st = dev_src ? validate_maps(d) : validate_desc(d)) return st;
    if (d->group_size != kGroupK)
        return fail(MQ_USAGE, "group size " + std::to_string(d->group_size) +
                                  " not supported by the sm_100a engine (tcgen05 tiles use group 128, the reference default)");
    mq_layer_opts o{MQ_W8_REFERENCE, 0, 1};
    if (opts) o = *opts;
    if (o.world < 1 || o.rank < 0 || o.rank >= o.world) return fail(MQ_USAGE, "bad rank/world");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(MQ_CUDA, "no CUDA device: the engine has no CPU fallback");
    if (device < 0 || device >= ndev) return fail(MQ_USAGE, "bad device ordinal");
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    if (major != 10) return fail(MQ_CUDA, "the engine is built for sm_100a (B200); device is sm_" + std::to_string(major) + "x");
    CU_TRY(cudaSetDevice(device));
    const int64_t G = num_groups(d->in_features, d->group_size);
    if (dev_src) {  // validate_quantized's metadata checks (quant.cpp:81-101), on device
        int32_t* flags = nullptr;
        CU_TRY(cudaMalloc(&flags, 8));
        int32_t h[2] = {0, 0};
        cudaError_t e = cudaMemsetAsync(flags, 0, 8, stream);
        if (e == cudaSuccess)
            e = launch_meta_check(d->scales8, d->n8 * G, d->scales4, d->n4 * G, d->zero_points4, flags, stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(h, flags, 8, cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        cudaFree(flags);
        if (e != cudaSuccess) return cuda_fail(e, "layer metadata check");
        if (h[0]) return fail(MQ_DATA, "quantized tensor has a non-positive scale");
        if (h[1]) return fail(MQ_DATA, "4-bit zero point out of [0, 15]");
    }

    auto* L = new mq_layer_s;
    L->device = device;
    cudaDeviceGetAttribute(&L->num_sms, cudaDevAttrMultiProcessorCount, device);
    L->N = d->out_features;
    L->K = d->in_features;
    L->group = d->group_size;
    L->G = static_cast<int>(G);
    L->rank = o.rank;
    L->world = o.world;
    L->w8_mode = o.w8_mode;
    const int64_t K = L->K;

    // Shard: rank r owns rows [r*n/W, (r+1)*n/W) of each sub-problem.
    auto lo = [&](int64_t n, int r) { return n * r / o.world; };
    const int64_t a8 = lo(d->n8, o.rank), b8 = lo(d->n8, o.rank + 1);
    const int64_t a4 = lo(d->n4, o.rank), b4 = lo(d->n4, o.rank + 1);
    L->n8 = b8 - a8;
    L->n4 = b4 - a4;
    L->tiles8 = (L->n8 + kTileRows - 1) / kTileRows;
    L->tiles4 = (L->n4 + kTileRows - 1) / kTileRows;
    if (L->tiles8 + L->tiles4 > kCntWords) {
        const int64_t T = L->tiles8 + L->tiles4;
        delete L;
        return fail(MQ_USAGE, "layer has " + std::to_string(T) + " 128-row tiles per rank; the engine supports " +
                                  std::to_string(kCntWords) + " (shard it over more ranks)");
    }
    for (int kind = 0; kind < 3; ++kind) best_split(L, kind);
    if (o.world > 1) {
        if (mq_status st = mq_shard_plan(d, o.world, &L->shard_cols, nullptr)) {
            delete L;
            return st;
        }
        L->shard_colmap.assign(size_t(o.world * L->shard_cols), -1);
        mq_shard_plan(d, o.world, &L->shard_cols, L->shard_colmap.data());
    } else {
        L->shard_cols = L->N;
    }

    // ---- tiles and the scatter column of every tile row
    const int64_t T = L->tiles8 + L->tiles4;
    L->bytes_wq = (L->tiles8 * kBlock8Bytes + L->tiles4 * kBlock4Bytes) * G;
    std::vector<int32_t> colmap(size_t(std::max<int64_t>(T * kTileRows, 1)), -1);
    std::vector<int32_t> colmap_orig(o.world > 1 ? colmap.size() : 0, -1);
    L->tiles.resize(size_t(T));
    int64_t coff = 0;
    for (int64_t t = 0; t < T; ++t) {
        const bool is8 = t < L->tiles8;
        const int64_t first = is8 ? t * kTileRows : (t - L->tiles8) * kTileRows;  // local sub row
        const int64_t nloc = is8 ? L->n8 : L->n4;
        const int rows = static_cast<int>(std::min<int64_t>(kTileRows, nloc - first));
        TileDesc& td = L->tiles[t];
        td.codes_off = coff;
        td.is8 = is8;
        td.rows = rows;
        td.first = static_cast<int32_t>(first);
        td.pad = 0;
        for (int r = 0; r < rows; ++r) {
            const int64_t srow = (is8 ? a8 : a4) + first + r;  // global sub-problem row
            const int64_t lcol = (is8 ? 0 : L->n8) + first + r;  // local gather column
            const int32_t orig = is8 ? d->index_map8[srow] : d->index_map4[srow];
            colmap[t * kTileRows + r] = o.world > 1 ? static_cast<int32_t>(lcol) : orig;
            if (o.world > 1) colmap_orig[t * kTileRows + r] = orig;
        }
        coff += (is8 ? kBlock8Bytes : kBlock4Bytes) * G;
        L->stream_bytes += int64_t(is8 ? kBlock8Bytes : kBlock4Bytes) * G;
    }

    auto upload = [&](void** dst, const void* src, size_t n) -> cudaError_t {
        cudaError_t e = cudaMalloc(dst, std::max<size_t>(n, 16));
        if (e != cudaSuccess) return e;
        return n ? cudaMemcpy(*dst, src, n, cudaMemcpyHostToDevice) : cudaSuccess;
    };
    cudaError_t e = cudaSuccess;
    if (dev_src) {  // pack on the GPU from the device reference layouts (weight_quant.cu)
        e = cudaMalloc(reinterpret_cast<void**>(&L->d_wq), std::max<size_t>(size_t(L->bytes_wq), 16));
        if (e == cudaSuccess)
            e = launch_engine_pack(static_cast<int32_t>(L->tiles8), static_cast<int32_t>(L->tiles4), L->n8, L->n4, a8,
                                   a4, L->G, K, d->payload8, d->scales8, d->payload4, d->scales4, d->zero_points4,
                                   L->d_wq, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    } else {  // pack on the host, upload once
        std::vector<uint8_t> wq(size_t(std::max<int64_t>(L->bytes_wq, 1)), 0);
        const int64_t stride4 = row_stride(4, K);
        for (int64_t t = 0; t < T; ++t) {
            const TileDesc& td = L->tiles[t];
            const bool is8 = td.is8 != 0;
            for (int64_t g = 0; g < G; ++g) {
                const int64_t k0 = g * kGroupK;
                uint8_t* cb = wq.data() + td.codes_off + g * (is8 ? kBlock8Bytes : kBlock4Bytes);
                uint8_t* mb = cb + (is8 ? kCodes8Bytes : kCodes4Bytes);  // scales | zero points
                for (int r = 0; r < td.rows; ++r) {
                    const int64_t srow = (is8 ? a8 : a4) + td.first + r;
                    float sc;
                    if (is8) {
                        const uint8_t* src = d->payload8 + srow * K;
                        for (int k = 0; k < kGroupK && k0 + k < K; ++k) cb[sw128_offset(r, k)] = src[k0 + k];
                        sc = d->scales8[srow * G + g];
                    } else {
                        const uint8_t* src = d->payload4 + srow * stride4;
                        for (int ch = 0; ch < 8; ++ch) {
                            uint8_t ev[16];
                            for (int j = 0; j < 16; ++j) {
                                const int64_t k = k0 + ch * 16 + j;
                                ev[j] = k < K ? ((k & 1) ? (src[k / 2] >> 4) : (src[k / 2] & 0x0F)) : 0;
                            }
                            uint32_t w0, w1;
                            pack_chunk4(ev, &w0, &w1);
                            std::memcpy(cb + sub4_chunk_offset(r, ch), &w0, 4);
                            std::memcpy(cb + sub4_chunk_offset(r, ch) + 4, &w1, 4);
                        }
                        sc = d->scales4[srow * G + g];
                        mb[512 + r] = d->zero_points4[srow * G + g];
                    }
                    std::memcpy(mb + 4 * r, &sc, 4);
                }
            }
        }
        e = upload(reinterpret_cast<void**>(&L->d_wq), wq.data(), size_t(L->bytes_wq));
    }
    if (e == cudaSuccess) e = upload(reinterpret_cast<void**>(&L->d_colmap), colmap.data(), colmap.size() * 4);
    if (e == cudaSuccess && o.world > 1)
        e = upload(reinterpret_cast<void**>(&L->d_colmap_orig), colmap_orig.data(), colmap_orig.size() * 4);
    if (e == cudaSuccess && o.world > 1)
        e = upload(reinterpret_cast<void**>(&L->d_shard_colmap), L->shard_colmap.data(), L->shard_colmap.size() * 4);
    if (e != cudaSuccess) {
        mq_layer_destroy(L);
        return cuda_fail(e, "layer upload");
    }
    *out = L;
    return MQ_OK;
}
}  // namespace

extern "C" {

mq_status mq_layer_create(const mq_layer_desc* d, const mq_layer_opts* opts, int device, mq_layer_t* out) {
    return create_layer(d, opts, device, false, nullptr, out);
}

mq_status mq_layer_create_device(const mq_layer_desc* d, const mq_layer_opts* opts, int device, void* stream,
                                 mq_layer_t* out) {
    return create_layer(d, opts, device, true, static_cast<cudaStream_t>(stream), out);
}

mq_status mq_layer_export_packed(mq_layer_t L, void* wq_host, size_t bytes, int32_t* colmap_host) {
    if (!L) return fail(MQ_USAGE, "layer handle is null");
    if (bytes != size_t(L->bytes_wq)) return fail(MQ_USAGE, "export buffer must be mq_layer_info.device_bytes bytes");
    cudaError_t e = cudaMemcpy(wq_host, L->d_wq, bytes, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && colmap_host)
        e = cudaMemcpy(colmap_host, L->d_colmap, size_t(L->tiles8 + L->tiles4) * kTileRows * 4,
                       cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "export packed layer");
    return MQ_OK;
}

// ------------------------------------------------- GPU partition_and_quantize
struct mq_device_qlayer_s {
    int device = 0;
    int64_t N = 0, K = 0;
    int group = 128;
    mq_scheme large{}, small{};
    std::vector<int32_t> map8, map4;
    uint8_t *p8 = nullptr, *p4 = nullptr, *z8 = nullptr, *z4 = nullptr;
    float *s8 = nullptr, *s4 = nullptr;
};

void mq_device_qlayer_destroy(mq_device_qlayer_t h) {
    if (!h) return;
    for (void* p : {static_cast<void*>(h->p8), static_cast<void*>(h->p4), static_cast<void*>(h->z8),
                    static_cast<void*>(h->z4), static_cast<void*>(h->s8), static_cast<void*>(h->s4)})
        if (p) cudaFree(p);
    delete h;
}

mq_status mq_partition_and_quantize_device(const double* W, int64_t N, int64_t K, const int32_t* promoted, int64_t np,
                                           const mq_scheme* large, const mq_scheme* small, int device, void* stream,
                                           mq_device_qlayer_t* out) {
    if (!out) return fail(MQ_USAGE, "out handle is null");
    if (!W && N * K > 0) return fail(MQ_USAGE, "weight matrix is null");
    if (mq_status st = check_scheme(large)) return st;
    if (mq_status st = check_scheme(small)) return st;
    if (large->group_size != small->group_size)
        return fail(MQ_DATA, "mixed layer: sub-problems must share group boundaries");
    for (const mq_scheme* sc : {large, small})
        if (sc->bit_width == 4 && sc->symmetric)
            return fail(MQ_USAGE, "quantize_tensor: 4-bit symmetric tensors are not supported");
    CU_TRY(cudaSetDevice(device));
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto* h = new mq_device_qlayer_s;
    h->device = device;
    h->N = N;
    h->K = K;
    h->group = large->group_size;
    h->large = *large;
    h->small = *small;
    if (mq_status st = partition_maps(N, promoted, np, h->map8, h->map4)) {
        delete h;
        return st;
    }
    const int64_t G = num_groups(K, h->group);
    int32_t* d_err = nullptr;
    int32_t* d_map = nullptr;
    uint8_t* d_codes = nullptr;
    int32_t herr[2] = {INT32_MAX, INT32_MAX};
    const int64_t n8 = int64_t(h->map8.size()), n4 = int64_t(h->map4.size());
    cudaError_t e = cudaMalloc(&d_err, 8);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_err, herr, 8, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMalloc(&d_map, size_t(std::max<int64_t>(N, 1)) * 4);
    // sub8 (large-bit) then sub4 (small-bit): gather + quantize in one pass per sub-problem
    for (int w = 0; w < 2 && e == cudaSuccess; ++w) {
        const mq_scheme* sc = w ? small : large;
        const std::vector<int32_t>& map = w ? h->map4 : h->map8;
        const int64_t rows = w ? n4 : n8;
        uint8_t*& pay = w ? h->p4 : h->p8;
        float*& scl = w ? h->s4 : h->s8;
        uint8_t*& zp = w ? h->z4 : h->z8;
        const int64_t stride = row_stride(sc->bit_width, K);
        e = cudaMalloc(&pay, size_t(std::max<int64_t>(rows * stride, 16)));
        if (e == cudaSuccess) e = cudaMalloc(&scl, size_t(std::max<int64_t>(rows * G, 4)) * 4);
        if (e == cudaSuccess && !sc->symmetric) e = cudaMalloc(&zp, size_t(std::max<int64_t>(rows * G, 16)));
        if (e == cudaSuccess && rows > 0)
            e = cudaMemcpyAsync(d_map, map.data(), size_t(rows) * 4, cudaMemcpyHostToDevice, s);
        uint8_t* codes = pay;
        if (e == cudaSuccess && sc->bit_width == 4) {  // one byte per code, then the nibble packer
            if (d_codes) cudaFree(d_codes);
            d_codes = nullptr;
            e = cudaMalloc(&d_codes, size_t(std::max<int64_t>(rows * K, 16)));
            codes = d_codes;
        }
        if (e == cudaSuccess)
            e = launch_weight_quant(W, K, d_map, rows, h->group, sc->bit_width, sc->symmetric, sc->scale_f16_storage,
                                    codes, scl, zp, d_err + w, s);
        if (e == cudaSuccess && sc->bit_width == 4) e = launch_pack_nibbles(codes, rows, K, pay, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // d_map / d_codes are reused
    }
    if (e == cudaSuccess) e = cudaMemcpy(herr, d_err, 8, cudaMemcpyDeviceToHost);
    cudaFree(d_err);
    cudaFree(d_map);
    if (d_codes) cudaFree(d_codes);
    if (e != cudaSuccess) {
        mq_device_qlayer_destroy(h);
        return cuda_fail(e, "device partition_and_quantize");
    }
    for (int w = 0; w < 2; ++w)
        if (herr[w] != INT32_MAX) {  // the reference throws at the first failing group (sub8 first)
            const int64_t r = herr[w] / G, g = herr[w] % G;
            mq_device_qlayer_destroy(h);
            return fail(MQ_DATA, "row " + std::to_string(r) + ", group " + std::to_string(g) +
                                     ": quantize: non-finite input value");
        }
    *out = h;
    return MQ_OK;
}

mq_status mq_device_qlayer_desc(mq_device_qlayer_t h, mq_layer_desc* d) {
    if (!h || !d) return fail(MQ_USAGE, "null device layer");
    if (h->large.bit_width != 8 || !h->large.symmetric || h->small.bit_width != 4 || h->small.symmetric)
        return fail(MQ_USAGE, "engine requires 8-bit symmetric / 4-bit asymmetric sub-problems");
    d->out_features = h->N;
    d->in_features = h->K;
    d->group_size = h->group;
    d->n8 = static_cast<int64_t>(h->map8.size());
    d->n4 = static_cast<int64_t>(h->map4.size());
    d->index_map8 = h->map8.data();
    d->index_map4 = h->map4.data();
    d->payload8 = h->p8;
    d->scales8 = h->s8;
    d->payload4 = h->p4;
    d->scales4 = h->s4;
    d->zero_points4 = h->z4;
    return MQ_OK;
}

void mq_layer_destroy(mq_layer_t L) {
    if (!L) return;
    cudaFree(L->d_wq);
    cudaFree(L->d_colmap);
    if (L->d_colmap_orig) cudaFree(L->d_colmap_orig);
    if (L->d_shard_colmap) cudaFree(L->d_shard_colmap);
    if (L->d_ws) cudaFree(L->d_ws);
    for (void* b : L->retired) cudaFree(b);
    delete L;
}

mq_status mq_layer_get_info(mq_layer_t L, mq_layer_info* info) {
    if (!L) return fail(MQ_USAGE, "layer handle is null");
    info->out_features = L->N;
    info->in_features = L->K;
    info->group_size = L->group;
    info->n8 = L->n8;
    info->n4 = L->n4;
    info->tiles8 = L->tiles8;
    info->tiles4 = L->tiles4;
    info->device_bytes = L->bytes_wq;
    info->weight_stream_bytes = L->stream_bytes;
    info->rank = L->rank;
    info->world = L->world;
    info->shard_cols = L->shard_cols;
    return MQ_OK;
}

mq_status mq_layer_shard_colmap(mq_layer_t L, int32_t* out) {
    if (!L) return fail(MQ_USAGE, "layer handle is null");
    if (L->world == 1) return fail(MQ_USAGE, "layer is not sharded");
    std::copy(L->shard_colmap.begin(), L->shard_colmap.end(), out);
    return MQ_OK;
}

mq_status mq_quantize_act(const void* A, mq_dtype dt, int64_t M, int64_t K, int64_t lda, int32_t group, int8_t* codes,
                          int64_t ldc, float* scales, int64_t lds, int32_t* err, void* stream) {
    if (M < 0 || K < 1) return fail(MQ_USAGE, "bad activation shape");
    if (group < 1) return fail(MQ_USAGE, "group_size must be >= 1");
    if (lda < K || ldc < K) return fail(MQ_USAGE, "leading dimension smaller than K");
    if (group < K && lds < M) return fail(MQ_USAGE, "scales leading dimension smaller than M");
    if (dt != MQ_F32 && dt != MQ_F16 && dt != MQ_BF16) return fail(MQ_USAGE, "bad activation dtype");
    cudaError_t e = launch_act_quant(A, dt, M, K, lda, group >= K ? int(K) : group, 0, codes, ldc, scales, lds, err,
                                     true, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "act_quant launch");
    return MQ_OK;
}

mq_status mq_quantize_act_scheme(const void* A, mq_dtype dt, int64_t M, int64_t K, int64_t lda, const mq_scheme* sc,
                                 int8_t* codes, int64_t ldc, float* scales, int64_t lds, int32_t* err, void* stream) {
    if (!sc) return fail(MQ_USAGE, "scheme is null");
    // check_engine_inputs (gemm.cpp:43-45): activations must be 8-bit symmetric
    if (sc->bit_width != 8 || !sc->symmetric) return fail(MQ_USAGE, "activation scheme must be 8-bit symmetric");
    if (M < 0 || K < 1) return fail(MQ_USAGE, "bad activation shape");
    if (sc->group_size < 1) return fail(MQ_USAGE, "group_size must be >= 1");
    if (lda < K || ldc < K) return fail(MQ_USAGE, "leading dimension smaller than K");
    if (sc->group_size < K && lds < M) return fail(MQ_USAGE, "scales leading dimension smaller than M");
    if (dt != MQ_F32 && dt != MQ_F16 && dt != MQ_BF16) return fail(MQ_USAGE, "bad activation dtype");
    const int group = sc->group_size >= K ? int(K) : sc->group_size;
    cudaError_t e = launch_act_quant(A, dt, M, K, lda, group, sc->scale_f16_storage ? 1 : 0, codes, ldc, scales, lds,
                                     err, true, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "act_quant launch");
    return MQ_OK;
}

size_t mq_forward_workspace_bytes(mq_layer_t L, int64_t M, const mq_exec_opts* o) {
    Plan pl, ps;  // a workspace serves the fused forward and the split API
    if (!L || M <= 0 || make_plan(L, M, o, &pl) != MQ_OK || make_plan(L, M, o, &ps, true) != MQ_OK) return 0;
    return std::max(eal_ws_layout(L, pl).total, eal_ws_layout(L, ps).total);
}

namespace {
mq_status launch_k2(mq_layer_s* L, const Plan& pl, const void* ws, int64_t M, void* Y, mq_dtype out_dtype,
                    cudaStream_t s, void* const* peers = nullptr, int npeer = 0) {
    const EalWs w = eal_ws_layout(L, pl);
    uint8_t* base = static_cast<uint8_t*>(const_cast<void*>(ws));
    GemmParams p;
    gemm_params(L, pl, M, Y, out_dtype, &p);
    if (npeer > 0) {  // fused gather: every rank's full Y at the original columns
        p.npeer = npeer;
        for (int i = 0; i < npeer; ++i) p.ypeer[i] = peers[i];
        p.Y = peers[0];
        p.ldy = L->N;
        if (L->world > 1) p.colmap = L->d_colmap_orig;
    }
    p.cnt = reinterpret_cast<uint32_t*>(base);
    p.part = reinterpret_cast<float*>(base + w.off_part);
    p.part2 = reinterpret_cast<float*>(base + w.off_part2);
    p.no_spin = pl.no_spin ? 1 : 0;
    p.acts = base + w.off_acts;
    p.sa = reinterpret_cast<const float*>(base + w.off_sa);
    p.asum = reinterpret_cast<const int32_t*>(base + w.off_asum);
    cudaError_t e = launch_mixed_gemm_tc(p, pl.bn, pl.mode, pl.pdl, s);
    if (e != cudaSuccess) return cuda_fail(e, "mixed_gemm launch");
    return MQ_OK;
}
}  // namespace

mq_status mq_mixed_linear_codes(mq_layer_t L, const int8_t* codes, int64_t ldc, const float* scales, int64_t lds,
                                int64_t M, void* Y, mq_dtype out_dtype, const mq_exec_opts* o, void* ws,
                                void* stream) {
    if (!L) return fail(MQ_USAGE, "layer handle is null");
    if (M < 0) return fail(MQ_USAGE, "M must be >= 0");
    if (M == 0) return MQ_OK;
    if (ldc < L->K) return fail(MQ_USAGE, "ldc must be >= K");
    if (out_dtype != MQ_F32 && out_dtype != MQ_F16 && out_dtype != MQ_BF16) return fail(MQ_USAGE, "bad output dtype");
    Plan pl;
    if (mq_status st = make_plan(L, M, o, &pl)) return st;
    if (!pl.per_token && lds < M) return fail(MQ_USAGE, "group-wise scales need lds >= M (group-major layout)");
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (o && o->gemm_impl == 1) {
        GemmParams p;
        gemm_params(L, pl, M, Y, out_dtype, &p);
        p.sa_rm = scales;
        p.sa_gstride = pl.per_token ? 0 : lds;
        cudaError_t e = launch_mixed_gemm_simt(p, codes, ldc, pl.mode == kFastToken ? kFastToken : kExactGroup,
                                               L->w8_mode == MQ_W8_REFERENCE, s);
        if (e != cudaSuccess) return cuda_fail(e, "simt launch");
        return MQ_OK;
    }
    const EalWs w = eal_ws_layout(L, pl);
    if (!ws) {
        if (mq_status st = ensure_internal_ws(L, w.total, s, &ws)) return st;
    }
    uint8_t* acts = static_cast<uint8_t*>(ws) + w.off_acts;
    float* sa = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + w.off_sa);
    int32_t* asum = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + w.off_asum);
    cudaError_t e = launch_repack_eal(codes, ldc, scales, lds, pl.per_token, M, L->K, pl.Mpad, acts, sa, asum, s);
    if (e != cudaSuccess) return cuda_fail(e, "repack launch");
    return launch_k2(L, pl, ws, M, Y, out_dtype, s);
}

size_t mq_mixed_linear_workspace_bytes(mq_layer_t L, int64_t M, const mq_exec_opts* o) {
    return mq_forward_workspace_bytes(L, M, o);
}

mq_status mq_mixed_linear(mq_layer_t L, const void* A, mq_dtype a_dtype, int64_t M, void* Y, mq_dtype out_dtype,
                          const mq_exec_opts* o, void* ws, int32_t* err, void* stream) {
    if (!L) return fail(MQ_USAGE, "layer handle is null");
    if (M < 0) return fail(MQ_USAGE, "M must be >= 0");
    if (M == 0) return MQ_OK;
    if (a_dtype != MQ_F32 && a_dtype != MQ_F16 && a_dtype != MQ_BF16) return fail(MQ_USAGE, "bad activation dtype");
    if (out_dtype != MQ_F32 && out_dtype != MQ_F16 && out_dtype != MQ_BF16) return fail(MQ_USAGE, "bad output dtype");
    Plan pl;
    if (mq_status st = make_plan(L, M, o, &pl)) return st;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const EalWs w = eal_ws_layout(L, pl);
    if (!ws) {
        if (mq_status st = ensure_internal_ws(L, w.total, s, &ws)) return st;
    }
    uint8_t* acts = static_cast<uint8_t*>(ws) + w.off_acts;
    float* sa = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + w.off_sa);
    if (o && o->gemm_impl == 1) return fail(MQ_USAGE, "the SIMT debug kernel takes quantized codes (mq_mixed_linear_codes)");
    int32_t* asum = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + w.off_asum);
    cudaError_t e = launch_act_quant_eal(A, a_dtype, M, L->K, L->K, pl.per_token ? int(L->K) : L->group, pl.Mpad, acts,
                                         sa, asum, err, pl.f16 ? 1 : 0, pl.pdl, s);
    if (e != cudaSuccess) return cuda_fail(e, "act_quant launch");
    return launch_k2(L, pl, ws, M, Y, out_dtype, s);
}

mq_status mq_quantize_act_ws(mq_layer_t L, const void* A, mq_dtype a_dtype, int64_t M, const mq_exec_opts* o, void* ws,
                             int32_t* err, void* stream) {
    if (!L || !ws) return fail(MQ_USAGE, "layer handle / workspace is null");
    if (M < 0) return fail(MQ_USAGE, "M must be >= 0");
    if (M == 0) return MQ_OK;
    if (a_dtype != MQ_F32 && a_dtype != MQ_F16 && a_dtype != MQ_BF16) return fail(MQ_USAGE, "bad activation dtype");
    Plan pl;
    if (mq_status st = make_plan(L, M, o, &pl, true)) return st;
    const EalWs w = eal_ws_layout(L, pl);
    uint8_t* base = static_cast<uint8_t*>(ws);
    cudaError_t e = launch_act_quant_eal(A, a_dtype, M, L->K, L->K, pl.per_token ? int(L->K) : L->group, pl.Mpad,
                                         base + w.off_acts, reinterpret_cast<float*>(base + w.off_sa),
                                         reinterpret_cast<int32_t*>(base + w.off_asum), err, pl.f16 ? 1 : 0, pl.pdl,
                                         static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "act_quant launch");
    return MQ_OK;
}

mq_status mq_mixed_linear_ws(mq_layer_t L, int64_t M, const void* ws, void* Y, mq_dtype out_dtype,
                             const mq_exec_opts* o, void* stream) {
    if (!L || !ws) return fail(MQ_USAGE, "layer handle / workspace is null");
    if (M < 0) return fail(MQ_USAGE, "M must be >= 0");
    if (M == 0) return MQ_OK;
    if (out_dtype != MQ_F32 && out_dtype != MQ_F16 && out_dtype != MQ_BF16) return fail(MQ_USAGE, "bad output dtype");
    Plan pl;
    if (mq_status st = make_plan(L, M, o, &pl, true)) return st;
    return launch_k2(L, pl, ws, M, Y, out_dtype, static_cast<cudaStream_t>(stream));
}

// ------------------------------------------------ column-sharded forwards
namespace {
size_t out_size(mq_dtype dt) { return dt == MQ_F32 ? 4 : 2; }
size_t al256(size_t x) { return (x + 255) / 256 * 256; }
}  // namespace

size_t mq_mixed_linear_allgather_workspace_bytes(mq_layer_t L, int64_t M, const mq_exec_opts* o, mq_dtype out_dtype) {
    const size_t fw = mq_forward_workspace_bytes(L, M, o);
    if (!fw) return 0;
    const size_t blk = size_t(M) * size_t(L->shard_cols) * out_size(out_dtype);
    return al256(fw) + al256(blk) + (L->world > 1 ? al256(blk * size_t(L->world)) : 0);
}

mq_status mq_mixed_linear_allgather(mq_layer_t L, const void* A, mq_dtype a_dtype, int64_t M, void* Y,
                                    mq_dtype out_dtype, const mq_exec_opts* o, void* ws, int32_t* err, void* comm,
                                    void* stream) {
    if (!L) return fail(MQ_USAGE, "layer handle is null");
    if (!ws) return fail(MQ_USAGE, "the gathered forward needs a workspace (mq_mixed_linear_allgather_workspace_bytes)");
    if (mq_status st = nccl_check_comm(comm, L->world, L->rank)) return st;
    if (M == 0) return MQ_OK;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t fw = al256(mq_forward_workspace_bytes(L, M, o));
    if (fw == 0) return fail(MQ_USAGE, "bad forward options");
    const size_t blk = size_t(M) * size_t(L->shard_cols);
    uint8_t* local = static_cast<uint8_t*>(ws) + fw;
    // this rank's block in gather order, then the gather of every rank's block
    if (mq_status st = mq_mixed_linear(L, A, a_dtype, M, local, out_dtype, o, ws, err, stream)) return st;
    if (L->world == 1) return nccl_all_gather(local, Y, blk, out_dtype, comm, s);
    uint8_t* gathered = local + al256(blk * out_size(out_dtype));
    if (mq_status st = nccl_all_gather(local, gathered, blk, out_dtype, comm, s)) return st;
    cudaError_t e = launch_permute(gathered, L->d_shard_colmap, L->world, L->shard_cols, M, L->N, Y, out_dtype, s);
    if (e != cudaSuccess) return cuda_fail(e, "permute launch");
    return MQ_OK;
}

mq_status mq_mixed_linear_peers(mq_layer_t L, const void* A, mq_dtype a_dtype, int64_t M, void* const* y_peers,
                                int32_t n_peers, mq_dtype out_dtype, const mq_exec_opts* o, void* ws, int32_t* err,
                                void* stream) {
    if (!L) return fail(MQ_USAGE, "layer handle is null");
    if (!y_peers || n_peers < 1 || n_peers > kMaxPeers)
        return fail(MQ_USAGE, "y_peers must list 1.." + std::to_string(kMaxPeers) + " output buffers");
    for (int i = 0; i < n_peers; ++i)
        if (!y_peers[i]) return fail(MQ_USAGE, "null peer output buffer");
    if (M < 0) return fail(MQ_USAGE, "M must be >= 0");
    if (M == 0) return MQ_OK;
    if (a_dtype != MQ_F32 && a_dtype != MQ_F16 && a_dtype != MQ_BF16) return fail(MQ_USAGE, "bad activation dtype");
    if (out_dtype != MQ_F32 && out_dtype != MQ_F16 && out_dtype != MQ_BF16) return fail(MQ_USAGE, "bad output dtype");
    Plan pl;
    if (mq_status st = make_plan(L, M, o, &pl)) return st;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const EalWs w = eal_ws_layout(L, pl);
    if (!ws) {
        if (mq_status st = ensure_internal_ws(L, w.total, s, &ws)) return st;
    }
    uint8_t* base = static_cast<uint8_t*>(ws);
    cudaError_t e = launch_act_quant_eal(A, a_dtype, M, L->K, L->K, pl.per_token ? int(L->K) : L->group, pl.Mpad,
                                         base + w.off_acts, reinterpret_cast<float*>(base + w.off_sa),
                                         reinterpret_cast<int32_t*>(base + w.off_asum), err, pl.f16 ? 1 : 0, pl.pdl, s);
    if (e != cudaSuccess) return cuda_fail(e, "act_quant launch");
    return launch_k2(L, pl, ws, M, y_peers[0], out_dtype, s, y_peers, n_peers);
}

mq_status mq_peer_barrier(uint32_t* const* flags, int32_t world, int32_t rank, uint32_t epoch, void* stream) {
    if (!flags || world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
        return fail(MQ_USAGE, "bad peer barrier arguments");
    cudaError_t e = launch_peer_barrier(flags, world, rank, epoch, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "peer barrier launch");
    return MQ_OK;
}

mq_status mq_gemm_partials(mq_layer_t L, const int8_t* codes, int64_t ldc, int64_t M, int32_t which, int32_t* partials,
                           void* stream) {
    if (!L) return fail(MQ_USAGE, "layer handle is null");
    if (which != 0 && which != 1) return fail(MQ_USAGE, "which must be 0 (sub8) or 1 (sub4)");
    if (ldc < L->K) return fail(MQ_USAGE, "ldc must be >= K");
    if (M == 0) return MQ_OK;
    mq_exec_opts o{};
    o.mode = MQ_EXACT;
    o.ksplit = 1;
    Plan pl;
    if (mq_status st = make_plan(L, M, &o, &pl)) return st;
    pl.mode = kDumpPartials;
    pl.rotate = false;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const EalWs w = eal_ws_layout(L, pl);
    void* ws = nullptr;
    if (mq_status st = ensure_internal_ws(L, w.total, s, &ws)) return st;
    uint8_t* acts = static_cast<uint8_t*>(ws) + w.off_acts;
    float* sa = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + w.off_sa);
    // scales are unused by the dump: repack with zero scales from a null-free buffer
    cudaError_t e = cudaMemsetAsync(sa, 0, w.total - w.off_sa, s);
    int32_t* asum = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + w.off_asum);
    if (e == cudaSuccess) e = launch_repack_eal(codes, ldc, sa, 0, 1, M, L->K, pl.Mpad, acts, sa, asum, s);
    if (e != cudaSuccess) return cuda_fail(e, "repack launch");
    GemmParams p;
    gemm_params(L, pl, M, nullptr, MQ_F32, &p);
    p.acts = acts;
    p.sa = sa;
    p.asum = asum;
    // restrict the launch to one sub-problem: its tiles, offsets and rows
    if (which == 0) {
        p.T4 = 0;
        p.n4 = 0;
    } else {
        p.wq += L->tiles8 * L->G * kBlock8Bytes;
        p.colmap += L->tiles8 * kTileRows;
        p.T8 = 0;
        p.n8 = 0;
    }
    if (p.T8 + p.T4 == 0) return MQ_OK;
    p.S4 = p.S8 = 1;
    p.lgS4 = p.lgS8 = 0;
    p.units = (p.T8 + p.T4) * pl.tb;
    p.grid = std::min(p.units, L->num_sms);
    p.partials = partials;
    p.partial_rows = static_cast<int32_t>(which == 0 ? L->n8 : L->n4);
    e = launch_mixed_gemm_tc(p, pl.bn, kDumpPartials, false, s);
    if (e != cudaSuccess) return cuda_fail(e, "partials launch");
    return MQ_OK;
}

#ifdef MQ_DEV
// development builds only (-DMQ_DEV, tools/trace_k2.py): copy the last traced
// launch's per-CTA timestamps (MQ_DBG & 32); not part of the C ABI
int mq_debug_trace(unsigned long long* out) {
    if (!g_trace_buf) return 0;
    cudaDeviceSynchronize();
    cudaMemcpy(out, g_trace_buf, (148 * 8 + 1024) * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    return 148;
}
#endif

mq_status mq_permute_gathered(const void* gathered, const int32_t* colmap, int32_t world, int64_t sc, int64_t M,
                              int64_t N, void* Y, mq_dtype dt, void* stream) {
    if (world < 1 || sc < 0 || M < 0) return fail(MQ_USAGE, "bad permute shape");
    cudaError_t e = launch_permute(gathered, colmap, world, sc, M, N, Y, dt, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "permute launch");
    return MQ_OK;
}

}  // extern "C"

// mq_layer.cpp — device layer handle, the one-time packer into the engine's
// HBM layout (mq_layout.cuh), launch planning and the forward entry points of
// the C ABI.
//
// The reference re-prepacks both sub-problems on every forward call
// (proj/src/gemm.cpp:148-149, ~45% of its call time at M=16); here
// packing happens once in mq_layer_create and forwards only stream weights.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cmath>
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
    uint8_t* d_wq = nullptr;
    int32_t* d_colmap = nullptr;
    int64_t bytes_wq = 0, stream_bytes = 0;
    std::vector<TileDesc> tiles;        // host copy (packing / accounting)
    std::vector<int32_t> shard_colmap;  // [world * shard_cols]
    std::mutex mu;                      // guards the internal workspace
    void* d_ws = nullptr;               // internal scratch (workspace = NULL)
    size_t ws_bytes = 0;
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

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

int auto_token_tile(int64_t M) {
    if (M <= 16) return 16;
    if (M <= 32) return 32;
    if (M <= 64) return 64;
    return 128;
}

struct Plan {
    int bn, tb, mode, per_token;
    bool split, pdl;
};

mq_status make_plan(const mq_layer_s* L, int64_t M, const mq_exec_opts* o, Plan* pl) {
    mq_exec_opts d{};
    if (!o) o = &d;
    const int act_group = o->act_group ? o->act_group : L->group;
    if (act_group == L->group && act_group < L->K) pl->per_token = 0;
    else if (act_group >= L->K) pl->per_token = 1;
    else
        return fail(MQ_USAGE, "activations and weights must share group boundaries (act group " +
                                  std::to_string(act_group) + ", weight group " + std::to_string(L->group) +
                                  "); per-token activations use act_group = K");
    if (o->mode != MQ_EXACT && o->mode != MQ_FAST) return fail(MQ_USAGE, "unknown mode");
    pl->bn = o->token_tile ? o->token_tile : auto_token_tile(M);
    if (pl->bn != 16 && pl->bn != 32 && pl->bn != 64 && pl->bn != 128)
        return fail(MQ_USAGE, "token_tile must be 16, 32, 64 or 128");
    pl->tb = static_cast<int>((M + pl->bn - 1) / pl->bn);
    pl->split = o->mode == MQ_FAST && o->ksplit != 1;
    pl->mode = o->mode == MQ_EXACT ? (pl->per_token ? kExactToken : kExactGroup) : (pl->per_token ? kFastToken : kFastGroup);
    pl->pdl = o->no_pdl == 0;
    return MQ_OK;
}

// Every CTA must own at least one group: an empty range inside an item would
// never arrive on the item's stream-K counter (the reduction counts the CTAs
// ca..cz that overlap it). P <= X, so strictly increasing cuts always exist.
void fill_cuts(GemmParams* p) {
    const Schedule S(*p);
    const int32_t X = static_cast<int32_t>(S.X);
    for (int c = 0; c <= p->P; ++c) p->cuts[c] = static_cast<int32_t>(S.cut(c));
    for (int c = 1; c < p->P; ++c) p->cuts[c] = std::max(p->cuts[c], p->cuts[c - 1] + 1);
    for (int c = p->P - 1; c >= 1; --c) p->cuts[c] = std::min(p->cuts[c], p->cuts[c + 1] - 1);
    p->cuts[0] = 0;
    p->cuts[p->P] = X;
}

// The launch grid and the stream-K cost weights (bytes streamed per group,
// incl. the activation tile and a fixed per-group pipeline cost).
void fill_schedule(const mq_layer_s* L, const Plan& pl, int sms, GemmParams* p) {
    const int64_t items = (L->tiles8 + L->tiles4) * pl.tb;
    const int64_t X = items * L->G;
    p->split = pl.split ? 1 : 0;
    p->P = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>({int64_t(sms), int64_t(kMaxCtas), pl.split ? X : items})));
    p->c8 = (kBlock8Bytes + 128 * pl.bn + 1024) / 64;
    p->c4 = (kBlock4Bytes + 128 * pl.bn + 1024) / 64;
    fill_cuts(p);
}

size_t ws_bytes_for(const mq_layer_s* L, const Plan& pl, int sms) {
    const int64_t items = (L->tiles8 + L->tiles4) * pl.tb;
    const int64_t X = items * L->G;
    const int64_t P = std::max<int64_t>(1, std::min<int64_t>(sms, pl.split ? X : items));
    const size_t counters = ((size_t(items) * 4 + 255) / 256) * 256;
    return counters + (pl.split ? size_t(2 * P) * 128 * pl.bn * 4 : 0);
}

// Activation codes as a 3-D tensor {128 (k in group), M, G} with byte strides
// {ldc, 128}: one box {128, BN, GPS} lands GPS per-group [BN][128] SW128 tiles.
// Scales (group-major [G][lds] f32) as 2-D {M, G}: box {BN, GPS}.
mq_status encode_maps(CUtensorMap* amap, CUtensorMap* smap, const int8_t* codes, int64_t ldc, const float* scales,
                      int64_t lds, int64_t M, int G, int bn, bool with_scales) {
    auto fn = encode_fn();
    if (!fn) return fail(MQ_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
    const int gps = gemm_gps(bn);
    {
        const cuuint64_t dims[3] = {128u, static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(G)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ldc), 128u};
        const cuuint32_t box[3] = {128u, static_cast<cuuint32_t>(bn), static_cast<cuuint32_t>(gps)};
        const cuuint32_t estr[3] = {1u, 1u, 1u};
        CUresult r = fn(amap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(codes), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(MQ_CUDA, "cuTensorMapEncodeTiled(codes) failed: " + std::to_string(int(r)));
    }
    std::memset(smap, 0, sizeof(*smap));
    if (with_scales) {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(G)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(lds) * 4u};
        const cuuint32_t box[2] = {static_cast<cuuint32_t>(bn), static_cast<cuuint32_t>(gps)};
        const cuuint32_t estr[2] = {1u, 1u};
        CUresult r = fn(smap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(scales), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(MQ_CUDA, "cuTensorMapEncodeTiled(scales) failed: " + std::to_string(int(r)));
    }
    return MQ_OK;
}

void gemm_params(const mq_layer_s* L, const Plan& pl, const float* sa, int64_t lds, int64_t M, void* Y,
                 mq_dtype out_dtype, void* ws, GemmParams* p) {
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
    p->sa = sa;
    p->sa_gstride = pl.per_token ? 0 : lds;
    p->M = M;
    p->Y = Y;
    p->out_dtype = out_dtype;
    p->ldy = L->world > 1 ? L->shard_cols : L->N;
    fill_schedule(L, pl, L->num_sms, p);
    if (ws) {
        const int64_t items = (L->tiles8 + L->tiles4) * pl.tb;
        uint8_t* w = static_cast<uint8_t*>(ws);
        p->counters = reinterpret_cast<uint32_t*>(w);
        p->ws = reinterpret_cast<float*>(w + ((size_t(items) * 4 + 255) / 256) * 256);
    }
    p->idesc8 = idesc_i8(0, L->w8_mode == MQ_W8_SIGNED, true);
    static const int dbg = [] {
        const char* e = std::getenv("MQ_DBG");
        return e ? std::atoi(e) : 0;
    }();
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
        if (L->d_ws) cudaFree(L->d_ws);
        L->d_ws = nullptr;
        L->ws_bytes = 0;
        CU_TRY(cudaMalloc(&L->d_ws, bytes));
        CU_TRY(cudaMemset(L->d_ws, 0, bytes));
        L->ws_bytes = bytes;
    }
    *ws = L->d_ws;
    return MQ_OK;
}

int64_t lds_for(int64_t M) { return (M + 3) / 4 * 4; }

// workspace of the full dynamic path: codes [M, ldc] | scales [Ga, lds] | gemm
struct FullWs {
    int64_t ldc, lds;
    size_t off_scales, off_gemm, total;
};
FullWs full_ws_layout(const mq_layer_s* L, int64_t M, int per_token, size_t gemm_bytes) {
    FullWs f;
    f.ldc = (L->K + 127) / 128 * 128;
    f.lds = lds_for(M);
    const int64_t Ga = per_token ? 1 : L->G;
    f.off_scales = size_t((M * f.ldc + 255) / 256 * 256);
    f.off_gemm = f.off_scales + size_t((Ga * f.lds * 4 + 255) / 256 * 256);
    f.total = f.off_gemm + gemm_bytes;
    return f;
}

}  // namespace

extern "C" {

mq_status mq_layer_create(const mq_layer_desc* d, const mq_layer_opts* opts, int device, mq_layer_t* out) {
    if (!out) return fail(MQ_USAGE, "out handle is null");
    if (mq_status st = validate_desc(d)) return st;
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

    auto* L = new mq_layer_s;
    L->device = device;
    cudaDeviceGetAttribute(&L->num_sms, cudaDevAttrMultiProcessorCount, device);
    L->N = d->out_features;
    L->K = d->in_features;
    L->group = d->group_size;
    L->G = static_cast<int>(num_groups(L->K, L->group));
    L->rank = o.rank;
    L->world = o.world;
    L->w8_mode = o.w8_mode;
    const int64_t K = L->K, G = L->G;

    // Shard: rank r owns rows [r*n/W, (r+1)*n/W) of each sub-problem.
    auto lo = [&](int64_t n, int r) { return n * r / o.world; };
    const int64_t a8 = lo(d->n8, o.rank), b8 = lo(d->n8, o.rank + 1);
    const int64_t a4 = lo(d->n4, o.rank), b4 = lo(d->n4, o.rank + 1);
    L->n8 = b8 - a8;
    L->n4 = b4 - a4;
    L->tiles8 = (L->n8 + kTileRows - 1) / kTileRows;
    L->tiles4 = (L->n4 + kTileRows - 1) / kTileRows;
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

    // ---- pack (host), then upload once
    const int64_t T = L->tiles8 + L->tiles4;
    L->bytes_wq = (L->tiles8 * kBlock8Bytes + L->tiles4 * kBlock4Bytes) * G;
    std::vector<uint8_t> wq(size_t(std::max<int64_t>(L->bytes_wq, 1)), 0);
    std::vector<int32_t> colmap(size_t(std::max<int64_t>(T * kTileRows, 1)), -1);
    L->tiles.resize(size_t(T));
    int64_t coff = 0;
    const int64_t stride4 = row_stride(4, K);
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
            colmap[t * kTileRows + r] = o.world > 1 ? static_cast<int32_t>(lcol)
                                                    : (is8 ? d->index_map8[srow] : d->index_map4[srow]);
        }
        for (int64_t g = 0; g < G; ++g) {
            const int64_t k0 = g * kGroupK;
            uint8_t* cb = wq.data() + coff + g * (is8 ? kBlock8Bytes : kBlock4Bytes);
            uint8_t* mb = cb + (is8 ? kCodes8Bytes : kCodes4Bytes);  // scales | zero points
            for (int r = 0; r < rows; ++r) {
                const int64_t srow = (is8 ? a8 : a4) + first + r;
                float sc;
                if (is8) {
                    const uint8_t* src = d->payload8 + srow * K;
                    for (int k = 0; k < kGroupK && k0 + k < K; ++k) cb[sw128_offset(r, k)] = src[k0 + k];
                    sc = d->scales8[srow * G + g];
                } else {
                    const uint8_t* src = d->payload4 + srow * stride4;
                    for (int ch = 0; ch < 8; ++ch) {
                        uint8_t e[16];
                        for (int j = 0; j < 16; ++j) {
                            const int64_t k = k0 + ch * 16 + j;
                            e[j] = k < K ? ((k & 1) ? (src[k / 2] >> 4) : (src[k / 2] & 0x0F)) : 0;
                        }
                        uint32_t w0, w1;
                        pack_chunk4(e, &w0, &w1);
                        std::memcpy(cb + sub4_chunk_offset(r, ch), &w0, 4);
                        std::memcpy(cb + sub4_chunk_offset(r, ch) + 4, &w1, 4);
                    }
                    sc = d->scales4[srow * G + g];
                    mb[512 + r] = d->zero_points4[srow * G + g];
                }
                std::memcpy(mb + 4 * r, &sc, 4);
            }
        }
        coff += (is8 ? kBlock8Bytes : kBlock4Bytes) * G;
        L->stream_bytes += int64_t(is8 ? kBlock8Bytes : kBlock4Bytes) * G;
    }

    auto upload = [&](void** dst, const void* src, size_t n) -> cudaError_t {
        cudaError_t e = cudaMalloc(dst, std::max<size_t>(n, 16));
        if (e != cudaSuccess) return e;
        return n ? cudaMemcpy(*dst, src, n, cudaMemcpyHostToDevice) : cudaSuccess;
    };
    cudaError_t e = upload(reinterpret_cast<void**>(&L->d_wq), wq.data(), size_t(L->bytes_wq));
    if (e == cudaSuccess) e = upload(reinterpret_cast<void**>(&L->d_colmap), colmap.data(), colmap.size() * 4);
    if (e != cudaSuccess) {
        mq_layer_destroy(L);
        return cuda_fail(e, "layer upload");
    }
    *out = L;
    return MQ_OK;
}


void mq_layer_destroy(mq_layer_t L) {
    if (!L) return;
    cudaFree(L->d_wq);
    cudaFree(L->d_colmap);
    if (L->d_ws) cudaFree(L->d_ws);
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

size_t mq_forward_workspace_bytes(mq_layer_t L, int64_t M, const mq_exec_opts* o) {
    Plan pl;
    if (!L || M <= 0 || make_plan(L, M, o, &pl) != MQ_OK) return 0;
    return ws_bytes_for(L, pl, L->num_sms);
}

mq_status mq_mixed_linear_codes(mq_layer_t L, const int8_t* codes, int64_t ldc, const float* scales, int64_t lds,
                                int64_t M, void* Y, mq_dtype out_dtype, const mq_exec_opts* o, void* ws,
                                void* stream) {
    if (!L) return fail(MQ_USAGE, "layer handle is null");
    if (M < 0) return fail(MQ_USAGE, "M must be >= 0");
    if (M == 0) return MQ_OK;
    if (ldc < int64_t(L->G) * kGroupK || ldc % 16 != 0)
        return fail(MQ_USAGE, "ldc must be >= ceil(K/128)*128 (zero-padded columns) and a multiple of 16");
    if (reinterpret_cast<uintptr_t>(codes) % 16 != 0) return fail(MQ_USAGE, "codes must be 16-byte aligned");
    if (reinterpret_cast<uintptr_t>(scales) % 16 != 0) return fail(MQ_USAGE, "scales must be 16-byte aligned");
    if (out_dtype != MQ_F32 && out_dtype != MQ_F16 && out_dtype != MQ_BF16) return fail(MQ_USAGE, "bad output dtype");
    Plan pl;
    if (mq_status st = make_plan(L, M, o, &pl)) return st;
    if (!pl.per_token && (lds < M || lds % 4 != 0))
        return fail(MQ_USAGE, "group-wise scales need lds >= M and lds % 4 == 0 (group-major layout)");
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (o && o->gemm_impl == 1) {
        GemmParams p;
        gemm_params(L, pl, scales, lds, M, Y, out_dtype, nullptr, &p);
        cudaError_t e = launch_mixed_gemm_simt(p, codes, ldc, pl.mode == kFastToken ? kFastToken : kExactGroup,
                                               L->w8_mode == MQ_W8_REFERENCE, s);
        if (e != cudaSuccess) return cuda_fail(e, "simt launch");
        return MQ_OK;
    }
    const size_t need = ws_bytes_for(L, pl, L->num_sms);
    if (!ws) {
        if (mq_status st = ensure_internal_ws(L, need, s, &ws)) return st;
    }
    GemmParams p;
    gemm_params(L, pl, scales, lds, M, Y, out_dtype, ws, &p);
    alignas(64) CUtensorMap amap, smap;
    if (mq_status st = encode_maps(&amap, &smap, codes, ldc, scales, lds, M, L->G, pl.bn, !pl.per_token)) return st;
    cudaError_t e = launch_mixed_gemm_tc(p, &amap, &smap, pl.bn, pl.mode, pl.pdl, s);
    if (e != cudaSuccess) return cuda_fail(e, "mixed_gemm launch");
    return MQ_OK;
}

size_t mq_mixed_linear_workspace_bytes(mq_layer_t L, int64_t M, const mq_exec_opts* o) {
    Plan pl;
    if (!L || M <= 0 || make_plan(L, M, o, &pl) != MQ_OK) return 0;
    return full_ws_layout(L, M, pl.per_token, mq_forward_workspace_bytes(L, M, o)).total;
}

mq_status mq_mixed_linear(mq_layer_t L, const void* A, mq_dtype a_dtype, int64_t M, void* Y, mq_dtype out_dtype,
                          const mq_exec_opts* o, void* ws, int32_t* err, void* stream) {
    if (!L) return fail(MQ_USAGE, "layer handle is null");
    if (M == 0) return MQ_OK;
    Plan pl;
    if (mq_status st = make_plan(L, M, o, &pl)) return st;
    const FullWs f = full_ws_layout(L, M, pl.per_token, mq_forward_workspace_bytes(L, M, o));
    if (!ws) {
        if (mq_status st = ensure_internal_ws(L, f.total, static_cast<cudaStream_t>(stream), &ws)) return st;
    }
    uint8_t* w = static_cast<uint8_t*>(ws);
    int8_t* codes = reinterpret_cast<int8_t*>(w);
    float* scales = reinterpret_cast<float*>(w + f.off_scales);
    const int32_t ag = pl.per_token ? int32_t(L->K) : int32_t(L->group);
    if (a_dtype != MQ_F32 && a_dtype != MQ_F16 && a_dtype != MQ_BF16) return fail(MQ_USAGE, "bad activation dtype");
    cudaError_t e = launch_act_quant(A, a_dtype, M, L->K, L->K, ag, 0, codes, f.ldc, scales, f.lds, err, pl.pdl,
                                     static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "act_quant launch");
    return mq_mixed_linear_codes(L, codes, f.ldc, scales, f.lds, M, Y, out_dtype, o, w + f.off_gemm, stream);
}

mq_status mq_gemm_partials(mq_layer_t L, const int8_t* codes, int64_t ldc, int64_t M, int32_t which, int32_t* partials,
                           void* stream) {
    if (!L) return fail(MQ_USAGE, "layer handle is null");
    if (which != 0 && which != 1) return fail(MQ_USAGE, "which must be 0 (sub8) or 1 (sub4)");
    if (ldc < int64_t(L->G) * kGroupK || ldc % 16 != 0)
        return fail(MQ_USAGE, "ldc must be >= ceil(K/128)*128 (zero-padded columns) and a multiple of 16");
    if (M == 0) return MQ_OK;
    Plan pl;
    if (mq_status st = make_plan(L, M, nullptr, &pl)) return st;
    pl.split = false;
    GemmParams p;
    gemm_params(L, pl, nullptr, 0, M, nullptr, MQ_F32, nullptr, &p);
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
    p.P = static_cast<int32_t>(std::min<int64_t>({int64_t(L->num_sms), int64_t(kMaxCtas), int64_t(p.T8 + p.T4) * pl.tb}));
    fill_cuts(&p);
    p.partials = partials;
    p.partial_rows = static_cast<int32_t>(which == 0 ? L->n8 : L->n4);
    alignas(64) CUtensorMap amap, smap;
    if (mq_status st = encode_maps(&amap, &smap, codes, ldc, nullptr, 0, M, L->G, pl.bn, false)) return st;
    cudaError_t e = launch_mixed_gemm_tc(p, &amap, &smap, pl.bn, kDumpPartials, false, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "partials launch");
    return MQ_OK;
}

// development: copy the last traced launch's per-CTA timestamps (MQ_DBG & 32)
int mq_debug_trace(unsigned long long* out) {
    if (!g_trace_buf) return 0;
    cudaDeviceSynchronize();
    cudaMemcpy(out, g_trace_buf, (148 * 8 + 1024) * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    return 148;
}

mq_status mq_permute_gathered(const void* gathered, const int32_t* colmap, int32_t world, int64_t sc, int64_t M,
                              int64_t N, void* Y, mq_dtype dt, void* stream) {
    if (world < 1 || sc < 0 || M < 0) return fail(MQ_USAGE, "bad permute shape");
    cudaError_t e = launch_permute(gathered, colmap, world, sc, M, N, Y, dt, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "permute launch");
    return MQ_OK;
}

}  // extern "C"

/*
 * mixllm/capi.h — C ABI of the B200-native MixLLM W4/W8-A8 mixed-precision
 * linear engine (libmixllm_b200.so).
 *
 * Drop-in boundary for the reference's hot path (/root/reference/proj). Every
 * entry cites the reference interface it replaces. All types are POD; device
 * buffers are caller-allocated (cudaMalloc / torch) unless stated; calls that
 * take a stream are stream-ordered and asynchronous. No torch types cross this
 * boundary. There is no CPU fallback: device entry points return MQ_CUDA when
 * no sm_100 device is present.
 *
 * Status codes mirror the reference CLI exit codes (proj/src/cli.cpp:501-510):
 * UsageError -> MQ_USAGE (1), DataError -> MQ_DATA (2), other -> MQ_INTERNAL (3),
 * plus MQ_CUDA (4) for device/runtime failures. Errors are reported BEFORE any
 * launch, as the reference throws before any compute (gemm.cpp:14-46).
 */
#ifndef MIXLLM_CAPI_H
#define MIXLLM_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MQ_OK = 0,
    MQ_USAGE = 1,    /* mixquant::UsageError  (proj/include/mixquant/errors.hpp:9-12) */
    MQ_DATA = 2,     /* mixquant::DataError   (errors.hpp:14-19) */
    MQ_INTERNAL = 3,
    MQ_CUDA = 4
} mq_status;

typedef enum { MQ_F32 = 0, MQ_F16 = 1, MQ_BF16 = 2 } mq_dtype;

/* Thread-local message of the last non-OK status on this thread. */
const char* mq_last_error(void);
const char* mq_version(void);

/* QuantScheme (proj/include/mixquant/quant.hpp:25-36). */
typedef struct {
    int32_t bit_width;         /* 4 or 8 */
    int32_t symmetric;         /* bool */
    int32_t group_size;        /* along K (in-features) */
    int32_t scale_f16_storage; /* bool */
} mq_scheme;

/* ===================================================================== */
/* Host packing — bit-exact with the reference layouts (synchronous, CPU). */
/* ===================================================================== */

/* quantize_tensor<float|double> (quant.hpp:183-243). payload: rows*row_stride
 * bytes (4-bit: nibbles low-first, stride ceil(cols/2); 8-bit: stride cols);
 * scales f32 [rows, G]; zero_points u8 [rows, G] (asymmetric only, else NULL).
 * On MQ_DATA, *err_row / *err_group (nullable) receive the failing group. */
mq_status mq_quantize_tensor_f32(const float* m, int64_t rows, int64_t cols,
                                 const mq_scheme* scheme, uint8_t* payload, float* scales,
                                 uint8_t* zero_points, int64_t* err_row, int64_t* err_group);
mq_status mq_quantize_tensor_f64(const double* m, int64_t rows, int64_t cols,
                                 const mq_scheme* scheme, uint8_t* payload, float* scales,
                                 uint8_t* zero_points, int64_t* err_row, int64_t* err_group);

/* pack_nibbles / unpack_nibbles (proj/src/tensor.cpp:63-94). */
mq_status mq_pack_nibbles(const uint8_t* values, int64_t count, uint8_t* out /* (count+1)/2 */);
mq_status mq_unpack_nibbles(const uint8_t* bytes, int64_t nbytes, int64_t count, uint8_t* out);

/* round_scale_f16 (proj/src/quant.cpp:81-86) and fast_i2f (gemm.hpp:27-31). */
float mq_round_scale_f16(float scale);
float mq_fast_i2f(int32_t x);

/* A quantized mixed layer in the reference layouts (MixedLinearLayer,
 * proj/include/mixquant/mixed.hpp:16-24). Host pointers. */
typedef struct {
    int64_t out_features;        /* N */
    int64_t in_features;         /* K */
    int32_t group_size;          /* shared by sub8 / sub4 */
    int64_t n8, n4;              /* rows of sub8 / sub4 */
    const int32_t* index_map8;   /* [n8] ascending original channels */
    const int32_t* index_map4;   /* [n4] */
    const uint8_t* payload8;     /* [n8, K] int8 codes ({8, sym, g}) */
    const float* scales8;        /* [n8, G] */
    const uint8_t* payload4;     /* [n4, ceil(K/2)] packed u4 ({4, asym, g}) */
    const float* scales4;        /* [n4, G] */
    const uint8_t* zero_points4; /* [n4, G] */
} mq_layer_desc;

/* partition_and_quantize (proj/src/mixed.cpp:46-81): splits W f64 [N, K] by the
 * promoted output channels into sub8 = {8, sym, g} and sub4 = {4, asym, g}.
 * The result is owned by the returned host layer; mq_host_layer_desc exposes
 * pointers into it (valid until mq_host_layer_destroy). */
typedef struct mq_host_layer_s* mq_host_layer_t;
mq_status mq_partition_and_quantize(const double* W, int64_t N, int64_t K,
                                    const int32_t* promoted, int64_t n_promoted,
                                    const mq_scheme* largebit, const mq_scheme* smallbit,
                                    mq_host_layer_t* out);
mq_status mq_host_layer_desc(mq_host_layer_t layer, mq_layer_desc* desc);
void mq_host_layer_destroy(mq_host_layer_t layer);

/* validate_mixed_layer (mixed.cpp:14-44) + validate_quantized (quant.cpp:81-101). */
mq_status mq_validate_layer(const mq_layer_desc* desc);

/* prepack_weights (gemm.cpp:89-108): the reference's group-major one-byte-per-
 * code layout, exported for parity only (the engine packs its own layout once
 * at mq_layer_create). which: 0 = sub8, 1 = sub4. out: rows*K bytes. */
mq_status mq_prepack_reference(const mq_layer_desc* desc, int32_t which, uint8_t* out);

/* reassemble_output (mixed.cpp:83-120) on host f32 buffers. */
mq_status mq_reassemble_output(const float* y8, int64_t n8, const float* y4, int64_t n4,
                               const int32_t* map8, const int32_t* map4, int64_t M,
                               int64_t out_features, float* out);

/* run_bench's synthetic inputs (gemm.cpp:211-227), byte-for-byte: W f64 [n,k],
 * A f32 [m,k], promoted [llround(percent*n)] (caller sizes it n). Returns the
 * promoted count. */
int64_t mq_bench_inputs(int64_t m, int64_t n, int64_t k, double percent, uint64_t seed,
                        double* W, float* A, int32_t* promoted);

/* Output-feature column-sharding plan (no reference counterpart —
 * the reference is single-process). Host only, no device needed. Rank r of
 * world W owns sub8 rows [r*n8/W, (r+1)*n8/W) and sub4 rows [r*n4/W, (r+1)*n4/W)
 * and writes its outputs in gather order: local column j of rank r is
 * original output column colmap[r*shard_cols + j] (sub8 rows first, then
 * sub4; -1 marks padding up to shard_cols = max over ranks). colmap may be
 * NULL (query shard_cols first); else it holds world*shard_cols entries. */
mq_status mq_shard_plan(const mq_layer_desc* desc, int32_t world, int64_t* shard_cols, int32_t* colmap);

/* fnv1a_hex (gemm.cpp:194-204) as a 64-bit value. */
uint64_t mq_fnv1a(const void* data, uint64_t nbytes);

/* ===================================================================== */
/* Device engine                                                          */
/* ===================================================================== */

typedef struct mq_layer_s* mq_layer_t;

/* 8-bit weight semantics. The reference stores 8-bit codes as uint8_t in
 * prepack_weights (gemm.cpp:103) and widens them UNSIGNED in gemm_block
 * (gemm.cpp:62,73-74): a code c < 0 contributes c + 256. MQ_W8_REFERENCE
 * reproduces that bit-for-bit (default: results identical to the reference);
 * MQ_W8_SIGNED follows SPEC.md:425 (codes used directly, signed). Same cost:
 * one bit of the tcgen05 instruction descriptor. */
typedef enum { MQ_W8_REFERENCE = 0, MQ_W8_SIGNED = 1 } mq_w8_mode;

typedef struct {
    int32_t w8_mode;  /* mq_w8_mode */
    int32_t rank;     /* output-feature column sharding: this rank ... */
    int32_t world;    /* ... of world (1 = unsharded) */
} mq_layer_opts;

/* Uploads a layer and packs the engine's device layout once (the reference
 * re-prepacks on every call, gemm.cpp:148-149). Immutable afterwards: safe to
 * use from several streams/threads. opts may be NULL (defaults). With world>1
 * the rank owns sub4 rows [r*n4/W, (r+1)*n4/W) and the same slice of sub8 rows
 * and writes its outputs in gather order (see mq_layer_info). */
mq_status mq_layer_create(const mq_layer_desc* desc, const mq_layer_opts* opts, int device,
                          mq_layer_t* out);
void mq_layer_destroy(mq_layer_t layer);

typedef struct {
    int64_t out_features, in_features;
    int32_t group_size;
    int64_t n8, n4;                /* rows owned by this handle (shard) */
    int64_t tiles8, tiles4;        /* 128-row tiles */
    int64_t device_bytes;          /* packed weights + metadata on device */
    int64_t weight_stream_bytes;   /* algorithmic weight bytes read per forward */
    int32_t rank, world;
    int64_t shard_cols;            /* columns per rank in gather order (padded) */
} mq_layer_info;
mq_status mq_layer_get_info(mq_layer_t layer, mq_layer_info* info);

/* ===================================================================== */
/* Offline quantization and prepack on the GPU        */
/* ===================================================================== */

/* partition_and_quantize (proj/src/mixed.cpp:46-81) on the GPU, bit-exact with
 * mq_partition_and_quantize: W is a DEVICE f64 [N, K] row-major matrix,
 * promoted a HOST list of output channels. The row gather and
 * quantize_group_{sym,asym}<double> (quant.hpp:84-140) run as one kernel per
 * sub-problem (a warp per (row, group), IEEE double throughout). The reference
 * layouts are kept in device memory, owned by the returned handle; errors
 * (non-finite input -> MQ_DATA with the first failing row/group, sub8 first)
 * are reported before returning, like the reference's DataError. Synchronous
 * w.r.t. `stream`. */
typedef struct mq_device_qlayer_s* mq_device_qlayer_t;
mq_status mq_partition_and_quantize_device(const double* W, int64_t N, int64_t K,
                                           const int32_t* promoted, int64_t n_promoted,
                                           const mq_scheme* largebit, const mq_scheme* smallbit,
                                           int device, void* stream, mq_device_qlayer_t* out);
/* Descriptor of a device-quantized layer: index maps are HOST pointers,
 * payloads / scales / zero points DEVICE pointers (valid until destroy). */
mq_status mq_device_qlayer_desc(mq_device_qlayer_t layer, mq_layer_desc* desc);
void mq_device_qlayer_destroy(mq_device_qlayer_t layer);

/* mq_layer_create from reference layouts already in device memory (desc:
 * HOST index maps, DEVICE payload8 / scales8 / payload4 / scales4 /
 * zero_points4, e.g. from mq_device_qlayer_desc): the engine layout is packed
 * on the GPU (same bytes as the host packer). validate_quantized's scale and
 * zero-point checks run on the device; synchronous w.r.t. `stream`. */
mq_status mq_layer_create_device(const mq_layer_desc* desc, const mq_layer_opts* opts, int device,
                                 void* stream, mq_layer_t* out);

/* Parity / debugging: copy a layer's packed device layout (device_bytes bytes)
 * and its tile-row column map ((tiles8 + tiles4) * 128 int32, nullable) to host. */
mq_status mq_layer_export_packed(mq_layer_t layer, void* wq_host, size_t bytes, int32_t* colmap_host);

/* Gather-order column map of a sharded layer: out[r*shard_cols + j] = original
 * output column of rank r's local column j, or -1 for padding. [world*shard_cols]. */
mq_status mq_layer_shard_colmap(mq_layer_t layer, int32_t* out);

/* Activation quantization (quant.hpp:117-140 via gemm.cpp:190), symmetric int8.
 * A: device [M, K] (row stride lda elements) in a_dtype. group_size == the
 * layer group (reference, group-wise) or == K (per-token, north_star). codes:
 * device int8 [M, ldc] (ldc >= K, multiple of 16; columns K..ldc are zeroed);
 * scales: device f32, group-major [G, lds] (group-wise) or [M] (per-token).
 * err (nullable, device int32, caller initialises to INT32_MAX): receives the
 * smallest m*G+g whose group held a non-finite value (the reference's
 * DataError, quant.hpp:56-64). Bit-exact with the reference for f32 input.
 * Scales are written GROUP-MAJOR, scales[g * lds + m] (lds >= M), so each
 * K-group's token scales are one contiguous run the GEMM producer streams
 * with a bulk copy (the reference keeps [M, G]; the values are identical).
 * Per-token: scales[m]. */
mq_status mq_quantize_act(const void* A, mq_dtype a_dtype, int64_t M, int64_t K, int64_t lda,
                          int32_t group_size, int8_t* codes, int64_t ldc, float* scales,
                          int64_t lds, int32_t* err, void* stream);
/* The same with the reference's full activation scheme (quantize_tensor<float>
 * with a QuantScheme, quant.hpp:183-185): scheme must be {8, symmetric,
 * group_size, scale_f16_storage}; scale_f16_storage rounds each scale to the
 * binary16 grid (round_scale_f16, quant.cpp:81-86). */
mq_status mq_quantize_act_scheme(const void* A, mq_dtype a_dtype, int64_t M, int64_t K, int64_t lda,
                                 const mq_scheme* scheme, int8_t* codes, int64_t ldc, float* scales,
                                 int64_t lds, int32_t* err, void* stream);

/* Forward modes.
 * MQ_EXACT: per output element the K-groups run in ascending order with an f32
 *   multiply then an f32 add (gemm.cpp:81), no split-K: bit-identical to the
 *   reference for group-wise activations.
 * MQ_FAST: FFMA/FFMA2 rescale and, at decode sizes, split-K over groups with a
 *   deterministic slice-order reduction; within the north_star tolerance
 *   (<= 1e-3 relative) and bit-reproducible run to run. */
typedef enum { MQ_EXACT = 0, MQ_FAST = 1 } mq_mode;

typedef struct {
    int32_t mode;        /* mq_mode */
    int32_t act_group;   /* group size the activation scales use (g or K) */
    int32_t ksplit;      /* MQ_FAST: 0 = auto, 1 = no K splitting, 2..8 = K-slices per sub4 tile (64/128-token
                            tiles: reduced until every slice runs in one round of the grid) */
    int32_t token_tile;  /* 0 = auto; else 16/32/64/128 */
    int32_t gemm_impl;   /* 0 = tcgen05 (product); 1 = SIMT debug kernel */
    int32_t no_pdl;      /* 1 = plain launches (default: programmatic dependent launch) */
    int32_t schedule;    /* MQ_FAST: 0 = auto (prefill: stream-K where the unit rounds leave SMs idle;
                            decode: unit schedule), 1 = unit rounds, 2 = stream-K wherever it applies,
                            decode included (equal work per SM; a cut item is joined by its last piece) */
    int32_t concurrent;  /* 1 = other kernels may hold SMs during this launch (multi-stream use,
                            overlapped collectives): never use a schedule whose CTAs wait on each
                            other (the one-round wide-tile barrier join); 0 = the launch owns the
                            device while it runs (default, fastest) */
    int32_t act_scale_f16; /* the activation scheme's scale_f16_storage (quant.hpp:70-76,
                              quant.cpp:81-86): round activation scales to binary16 */
    const struct mq_layer_s* prefetch_next; /* optional: the layer the caller runs NEXT on this
                            stream; once this launch has issued its own weight reads, its CTAs
                            prefetch the head of that layer's packed weights into L2 (weights
                            are immutable, so this is safe under any data dependency) */
    int64_t prefetch_bytes; /* bytes of prefetch_next to prefetch (0 = auto) */
} mq_exec_opts;

/* Bytes of scratch a forward needs: split-K arrival counters + partial tiles
 * and the engine-layout activations (K1 output, or the repacked codes). */
size_t mq_forward_workspace_bytes(mq_layer_t layer, int64_t M, const mq_exec_opts* opts);

/* The mixed-precision linear on quantized activations
 * (execute_mixed_on_codes, gemm.cpp:140-181): both sub-problems in one
 * persistent launch, scatter fused into the epilogue. The codes are first
 * repacked into the engine activation layout (one small kernel);
 * mq_mixed_linear / mq_quantize_act_ws write that layout directly.
 * codes: device int8 [M, ldc] (ldc >= K); scales as mq_quantize_act wrote them
 * (group-major [G, lds], lds >= M; per-token: [M]);
 * Y: device [M, out_features] row-major in out_dtype (sharded layers: the
 * rank's [M, shard_cols] block in gather order).
 * workspace: device, >= mq_forward_workspace_bytes, zero-initialised once
 * before first use. Its first 64 KiB are split-K arrival counters that every
 * launch leaves at zero, so one workspace can serve any M, any layer and any
 * options, as long as launches that share it are stream-ordered. NULL uses the
 * layer's own (then calls on one layer must be stream-serialised). */
mq_status mq_mixed_linear_codes(mq_layer_t layer, const int8_t* codes, int64_t ldc,
                                const float* scales, int64_t lds, int64_t M, void* Y,
                                mq_dtype out_dtype, const mq_exec_opts* opts, void* workspace,
                                void* stream);

/* The full dynamic path (execute_mixed_linear, gemm.cpp:183-192): activation
 * quantization + mixed GEMM + scatter. A: device [M, K] f32/f16/bf16.
 * err: as in mq_quantize_act (nullable). */
mq_status mq_mixed_linear(mq_layer_t layer, const void* A, mq_dtype a_dtype, int64_t M,
                          void* Y, mq_dtype out_dtype, const mq_exec_opts* opts,
                          void* workspace, int32_t* err, void* stream);
size_t mq_mixed_linear_workspace_bytes(mq_layer_t layer, int64_t M, const mq_exec_opts* opts);

/* Split form of mq_mixed_linear for callers that feed ONE quantized activation
 * to several layers with the same K, M and options (e.g. separate q/k/v or
 * gate/up layers): mq_quantize_act_ws runs K1 into the engine activation layout
 * (EAL) inside `workspace`; then any number of mq_mixed_linear_ws calls, on
 * any of those layers, run K2 on it. The EAL sits at an offset that depends
 * only on (K, M, options); each layer's split-K partials follow it, so the
 * workspace must be >= the MAXIMUM of mq_mixed_linear_workspace_bytes over the
 * layers that share it. The token tile depends on M only here (the EAL is
 * shared); the fused mq_mixed_linear may pick a per-layer tile for a narrow,
 * short-K layer. Same results as mq_mixed_linear: bit-identical in MQ_EXACT
 * mode and whenever opts.token_tile is set; otherwise, in MQ_FAST mode, equal
 * within its rounding (a different tile changes the K-split and summation
 * order). */
mq_status mq_quantize_act_ws(mq_layer_t layer, const void* A, mq_dtype a_dtype, int64_t M,
                             const mq_exec_opts* opts, void* workspace, int32_t* err, void* stream);
mq_status mq_mixed_linear_ws(mq_layer_t layer, int64_t M, const void* workspace, void* Y,
                             mq_dtype out_dtype, const mq_exec_opts* opts, void* stream);

/* Debug / parity: the int32 group partial sums S[g, m, r] = sum_i a*(w - z)
 * (the step-1 integer accumulator, gemm.cpp:64-75) of one sub-problem,
 * computed by the same tcgen05 pipeline. which: 0 = sub8, 1 = sub4.
 * partials: device int32 [G, M, rows]. */
mq_status mq_gemm_partials(mq_layer_t layer, const int8_t* codes, int64_t ldc, int64_t M,
                           int32_t which, int32_t* partials, void* stream);

/* Gathered sharded outputs -> original order: gathered [world, M, shard_cols]
 * (the all-gather of every rank's Y block), colmap from mq_layer_shard_colmap
 * (device copy), Y [M, out_features]. */
mq_status mq_permute_gathered(const void* gathered, const int32_t* colmap_dev, int32_t world,
                              int64_t shard_cols, int64_t M, int64_t out_features, void* Y,
                              mq_dtype dtype, void* stream);

/* ===================================================================== */
/* Multi-GPU: output-feature column sharding (no reference     */
/* counterpart — the reference is single-process). Layers are created with */
/* mq_layer_opts {rank, world}: rank r owns sub8 rows [r*n8/W, (r+1)*n8/W)  */
/* and the same slice of sub4 rows; activations are replicated.            */
/* ===================================================================== */

/* NCCL communicators. The library binds NCCL at run time (dlopen): the NCCL
 * already loaded in the process is used first (e.g. PyTorch's, so a
 * ProcessGroupNCCL communicator can be passed as `comm`), else libnccl.so.2.
 * id: NCCL_UNIQUE_ID_BYTES (128) bytes, created on one rank and shared. */
mq_status mq_nccl_unique_id(uint8_t* id);
mq_status mq_nccl_comm_init(const uint8_t* id, int32_t world, int32_t rank, int device, void** comm);
mq_status mq_nccl_comm_destroy(void* comm);

/* Gathered forward of one shard (north_star: NCCL all-gather over NVLink for
 * the gathered output only): K1 + K2 into this rank's [M, shard_cols] block in
 * gather order, ncclAllGather of the blocks on `comm` (an ncclComm_t whose rank
 * and size must match the layer's), then the permute to original column order
 * into Y [M, out_features]. Stream-ordered on `stream`; the workspace
 * (mq_mixed_linear_allgather_workspace_bytes) holds the forward scratch, the
 * local block and the gathered blocks. Equal, bit for bit, to the unsharded
 * layer's mq_mixed_linear under the same options. */
size_t mq_mixed_linear_allgather_workspace_bytes(mq_layer_t layer, int64_t M, const mq_exec_opts* opts,
                                                 mq_dtype out_dtype);
mq_status mq_mixed_linear_allgather(mq_layer_t layer, const void* A, mq_dtype a_dtype, int64_t M, void* Y,
                                    mq_dtype out_dtype, const mq_exec_opts* opts, void* workspace,
                                    int32_t* err, void* comm, void* stream);

/* Fused gather: the K2 epilogue scatters every output
 * element of this shard straight into ALL ranks' full outputs at the original
 * column — y_peers[i] is rank i's Y [M, out_features], peer-mapped into this
 * process (cudaIpcOpenMemHandle / NVLink UVA, or an NCCL window's LSA
 * pointer); y_peers[0] may be any rank's. No gather buffer, no permute: once
 * every rank's launch is complete (mq_peer_barrier) each Y is whole. n_peers
 * <= 8 (one NVLink domain). Workspace as mq_mixed_linear. */
mq_status mq_mixed_linear_peers(mq_layer_t layer, const void* A, mq_dtype a_dtype, int64_t M,
                                void* const* y_peers, int32_t n_peers, mq_dtype out_dtype,
                                const mq_exec_opts* opts, void* workspace, int32_t* err, void* stream);

/* Cross-rank completion barrier for the fused gather: flags[i] is rank i's
 * uint32 flag array [world] (peer-mapped, zero-initialised); rank `rank`
 * release-stores `epoch` into flags[i][rank] for every i, then waits until its
 * own flags[rank][0..world) all reached `epoch` (system-scope acquire). Use a
 * new epoch per call. One tiny kernel on `stream`. */
mq_status mq_peer_barrier(uint32_t* const* flags, int32_t world, int32_t rank, uint32_t epoch, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MIXLLM_CAPI_H */

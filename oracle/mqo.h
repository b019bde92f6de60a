/*
 * mqo.h — CPU ORACLE for the MixLLM W4/W8-A8 mixed-precision linear path.
 *
 * TEST INFRASTRUCTURE ONLY. This is a plain-C restatement of the reference
 * (`/root/reference/proj`, the C++20 `mixquant` toolkit) used as the parity
 * checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
 * The product path (paper_2412_14590_b200/) never links or calls it.
 *
 * Parity is PINNED: the restatement is checked bit-for-bit against the
 * reference's own code compiled from its sources (oracle/_ref, see
 * oracle/Makefile.ref) and against the reference tests' known-answer vectors
 * (proj/tests/test_quant_core.cpp, proj/tests/test_tensor_store.cpp) and the
 * SPEC examples, see tests/test_oracle_golden.py.
 *
 * Arithmetic contract: compile with -ffp-contract=off and
 * no -march (the reference's own flags, proj/src/CMakeLists.txt:14), IEEE
 * division, half-away-from-zero rounding (roundf/round + lround), no FTZ.
 */
#ifndef MQO_H
#define MQO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the CLI exit codes (proj/src/cli.cpp:501-510) */
enum { MQO_OK = 0, MQO_USAGE = 1, MQO_DATA = 2 };

/* ---- PRNG: proj/include/mixquant/rng.hpp:16-82 ---- */
typedef struct {
    uint64_t s[4];
    int has_spare;
    double spare;
} mqo_rng;

void mqo_rng_seed(mqo_rng* r, uint64_t seed);
uint64_t mqo_rng_next(mqo_rng* r);
double mqo_rng_uniform(mqo_rng* r);
int64_t mqo_rng_uniform_int(mqo_rng* r, int64_t lo, int64_t hi);
double mqo_rng_normal(mqo_rng* r);

/* ---- I2F: proj/include/mixquant/gemm.hpp:18-31 ---- */
float mqo_fast_i2f(int32_t x);

/* ---- f16 scale rounding: proj/src/quant.cpp:20-79 ---- */
float mqo_round_scale_f16(float s);

/* ---- nibble codec: proj/src/tensor.cpp:63-94 ---- */
int mqo_pack_nibbles(const uint8_t* v, int64_t n, uint8_t* out);           /* out: (n+1)/2 bytes */
int mqo_unpack_nibbles(const uint8_t* b, int64_t nbytes, int64_t count, uint8_t* out);

/* ---- group quantizers: proj/include/mixquant/quant.hpp:84-140 ----
 * One group of `len` values. sym: codes int8 in [-qmax,qmax]; asym: codes u8.
 * Returns MQO_DATA on a non-finite input, MQO_USAGE on bad bit width. */
int mqo_quant_group_sym_f32(const float* x, int64_t len, int bits, int f16,
                            int8_t* codes, float* scale);
int mqo_quant_group_sym_f64(const double* x, int64_t len, int bits, int f16,
                            int8_t* codes, float* scale);
int mqo_quant_group_asym_f32(const float* x, int64_t len, int bits, int f16,
                             uint8_t* codes, float* scale, uint8_t* zp);
int mqo_quant_group_asym_f64(const double* x, int64_t len, int bits, int f16,
                             uint8_t* codes, float* scale, uint8_t* zp);

/* ---- QuantizedTensor in reference layout (quant.hpp:146-243) ----
 * payload: rows*row_stride bytes (4-bit: packed low nibble first, stride
 * ceil(cols/2); 8-bit: stride cols); scales f32 [rows, G]; zps u8 [rows, G]
 * (asym only, may be NULL for sym). Returns status; on MQO_DATA err_row /
 * err_group (if non-NULL) receive the failing location. */
int64_t mqo_row_stride(int bits, int64_t cols);
int64_t mqo_num_groups(int64_t cols, int group);
int mqo_quantize_tensor_f32(const float* m, int64_t rows, int64_t cols, int bits, int sym,
                            int group, int f16, uint8_t* payload, float* scales,
                            uint8_t* zps, int64_t* err_row, int64_t* err_group);
int mqo_quantize_tensor_f64(const double* m, int64_t rows, int64_t cols, int bits, int sym,
                            int group, int f16, uint8_t* payload, float* scales,
                            uint8_t* zps, int64_t* err_row, int64_t* err_group);
/* raw code accessor QuantizedTensor::code (quant.hpp:165-175) */
int mqo_code(const uint8_t* payload, int bits, int sym, int64_t cols, int64_t r, int64_t c);

/* ---- partition (mixed.cpp:46-81): maps only; callers gather+quantize ----
 * promoted: n_promoted channel ids. map8 gets ascending promoted ids, map4 the
 * ascending remainder. Returns MQO_USAGE for out-of-range / duplicate ids. */
int mqo_partition_maps(int64_t out_features, const int32_t* promoted, int64_t n_promoted,
                       int32_t* map8, int64_t* n8, int32_t* map4, int64_t* n4);

/* ---- reference prepack (gemm.hpp:48-61, gemm.cpp:89-108) ----
 * codes[rows*begin_g + r*len_g + i] = (uint8_t)code(r, begin_g + i). */
void mqo_prepack(const uint8_t* payload, int bits, int sym, int64_t rows, int64_t cols,
                 int group, uint8_t* packed);

/* ---- emulated kernel (gemm.cpp:51-85) on one sub-problem ----
 * a_codes int8 [M,K]; a_scales f32 [M,G]; weights in reference layout;
 * out f32 [M, rows] is ACCUMULATED into (caller zero-initialises, gemm.cpp:122).
 * fast != 0 selects the fast-I2F mode. a_group_stride lets a per-token scale
 * array (G_a = 1) be broadcast: pass a_scale_cols = 1 for per-token.
 * w_u8 != 0 reproduces the reference's actual 8-bit behaviour: prepack stores
 * every code as uint8_t (gemm.cpp:103) and gemm_block widens that byte as
 * UNSIGNED (gemm.cpp:62,73-74), so a signed 8-bit code c < 0 enters the dot
 * product as c + 256. SPEC.md:425 says the 8-bit codes are used directly
 * (signed); w_u8 = 0 gives that. The reference's golden checksums (SURVEY
 * §8c) are produced with the unsigned reading. */
void mqo_gemm_sub(const int8_t* a_codes, const float* a_scales, int64_t a_scale_cols,
                  int64_t M, int64_t K, int group, const uint8_t* w_payload, int w_bits,
                  int w_sym, const float* w_scales, const uint8_t* w_zps, int64_t rows,
                  int fast, int w_u8, float* out);

/* int32 group partial sums S[g, m, r] = sum_i a[m,gG+i]*(w[r,gG+i]-z[r,g])
 * (the step-1 integer accumulator of gemm.cpp:64-75, without the I2F bias) */
void mqo_group_partials(const int8_t* a_codes, int64_t M, int64_t K, int group,
                        const uint8_t* w_payload, int w_bits, int w_sym,
                        const uint8_t* w_zps, int64_t rows, int w_u8, int32_t* partials);

/* ---- scatter (mixed.cpp:83-120) ---- */
int mqo_reassemble(const float* y8, int64_t n8, const float* y4, int64_t n4,
                   const int32_t* map8, const int32_t* map4, int64_t M, int64_t N, float* out);

/* ---- bench input generator, exactly run_bench (gemm.cpp:206-231) ----
 * W f64 [n,k], A f32 [m,k], promoted[llround(percent*n)] (caller sizes n). */
int64_t mqo_bench_inputs(int64_t m, int64_t n, int64_t k, double percent, uint64_t seed,
                         double* W, float* A, int32_t* promoted);

/* ---- the whole layer, oracle form of run_bench's timed region:
 * act quant {8,sym,group} (or per-token when act_group == K) + both GEMMs +
 * scatter. Weight payloads in reference layout. out f32 [M,N]. */
typedef struct {
    int64_t N, K;
    int group;
    int64_t n8, n4;
    const int32_t* map8; const int32_t* map4;
    const uint8_t* p8; const float* s8;                   /* sub8: 8-bit sym */
    const uint8_t* p4; const float* s4; const uint8_t* z4; /* sub4: 4-bit asym */
} mqo_layer;

int mqo_mixed_linear(const mqo_layer* L, const float* A, int64_t M, int act_group, int fast,
                     int w8_u8, int8_t* a_codes_out, float* a_scales_out, float* out);

/* ---- FNV-1a 64 (gemm.cpp:194-204) ---- */
uint64_t mqo_fnv1a(const void* data, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif

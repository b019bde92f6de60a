/*
 * mqo.c — CPU ORACLE (test infrastructure only; see mqo.h header).
 *
 * Plain-C restatement of the reference's hot path. Every function cites the
 * reference file:line it follows (paths relative to /root/reference).
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fPIC (no -march), oracle/Makefile.
 */
#include "mqo.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ PRNG */
/* proj/include/mixquant/rng.hpp:16-27 (SplitMix64) */
static uint64_t splitmix_next(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.hpp:31-34 */
void mqo_rng_seed(mqo_rng* r, uint64_t seed) {
    uint64_t st = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix_next(&st);
    r->has_spare = 0;
    r->spare = 0.0;
}

/* rng.hpp:36-46 (xoshiro256++, rotations 23/45, shift 17) */
uint64_t mqo_rng_next(mqo_rng* r) {
    uint64_t* s = r->s;
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

/* rng.hpp:49 */
double mqo_rng_uniform(mqo_rng* r) { return (double)(mqo_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:52-57 (fixed-point scaling, no modulo) */
int64_t mqo_rng_uniform_int(mqo_rng* r, int64_t lo, int64_t hi) {
    const uint64_t span = (uint64_t)(hi - lo);
    const uint64_t scaled = (uint64_t)(((unsigned __int128)mqo_rng_next(r) * span) >> 64);
    return lo + (int64_t)scaled;
}

/* rng.hpp:60-72 (Box-Muller, trigonometric form, cached spare) */
double mqo_rng_normal(mqo_rng* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    const double u1 = (double)((mqo_rng_next(r) >> 11) + 1) * 0x1.0p-53;
    const double u2 = mqo_rng_uniform(r);
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * M_PI * u2;
    r->spare = radius * sin(angle);
    r->has_spare = 1;
    return radius * cos(angle);
}

/* ------------------------------------------------------------------- I2F */
/* proj/include/mixquant/gemm.hpp:18-31 */
static const int32_t I2F_BIAS_INT = 0x4B400000;
static float bits_to_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t f32_to_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

float mqo_fast_i2f(int32_t x) {
    const int32_t tmp = (int32_t)((uint32_t)x + (uint32_t)I2F_BIAS_INT);
    return bits_to_f32((uint32_t)tmp) - bits_to_f32((uint32_t)I2F_BIAS_INT);
}

/* ------------------------------------------------------------ f16 scales */
/* proj/src/quant.cpp:20-51 */
static uint16_t f32_to_f16_bits(float f) {
    const uint32_t x = f32_to_bits(f);
    const uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
    const uint32_t exp = (x >> 23) & 0xFFu;
    uint32_t mant = x & 0x7FFFFFu;
    if (exp == 0xFFu) return (uint16_t)(sign | 0x7C00u | (mant ? 0x200u : 0));
    const int half_exp = (int)exp - 127 + 15;
    if (half_exp >= 0x1F) return (uint16_t)(sign | 0x7C00u);
    if (half_exp <= 0) {
        if (half_exp < -10) return sign;
        mant |= 0x800000u;
        const int shift = 14 - half_exp;
        uint32_t half_mant = mant >> shift;
        const uint32_t rem = mant & ((1u << shift) - 1);
        const uint32_t halfway = 1u << (shift - 1);
        if (rem > halfway || (rem == halfway && (half_mant & 1u))) ++half_mant;
        return (uint16_t)(sign | half_mant);
    }
    uint16_t h = (uint16_t)(sign | ((uint32_t)half_exp << 10) | (mant >> 13));
    const uint32_t rem = mant & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
    return h;
}

/* proj/src/quant.cpp:53-77 */
static float f16_bits_to_f32(uint16_t h) {
    const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    const uint32_t exp = (h >> 10) & 0x1Fu;
    uint32_t mant = h & 0x3FFu;
    uint32_t bits;
    if (exp == 0) {
        if (mant == 0) {
            bits = sign;
        } else {
            int e = -14;
            while ((mant & 0x400u) == 0) { mant <<= 1; --e; }
            mant &= 0x3FFu;
            bits = sign | ((uint32_t)(e + 127) << 23) | (mant << 13);
        }
    } else if (exp == 0x1Fu) {
        bits = sign | 0x7F800000u | (mant << 13);
    } else {
        bits = sign | ((exp + 127 - 15) << 23) | (mant << 13);
    }
    return bits_to_f32(bits);
}

/* proj/src/quant.cpp:81-86 */
float mqo_round_scale_f16(float s) {
    const float rounded = f16_bits_to_f32(f32_to_f16_bits(s));
    const float f16_min = 5.9604644775390625e-8f;
    return rounded > 0.0f ? rounded : f16_min;
}

/* ---------------------------------------------------------- nibble codec */
/* proj/src/tensor.cpp:63-78 */
int mqo_pack_nibbles(const uint8_t* v, int64_t n, uint8_t* out) {
    memset(out, 0, (size_t)((n + 1) / 2));
    for (int64_t i = 0; i < n; ++i) {
        if (v[i] > 15) return MQO_DATA;
        if (i % 2 == 0) out[i / 2] = v[i];
        else out[i / 2] |= (uint8_t)(v[i] << 4);
    }
    return MQO_OK;
}

/* proj/src/tensor.cpp:80-94 */
int mqo_unpack_nibbles(const uint8_t* b, int64_t nbytes, int64_t count, uint8_t* out) {
    if (count < 0 || count > nbytes * 2) return MQO_DATA;
    for (int64_t i = 0; i < count; ++i) {
        const uint8_t byte = b[i / 2];
        out[i] = (i % 2 == 0) ? (byte & 0x0F) : (byte >> 4);
    }
    return MQO_OK;
}

/* ------------------------------------------------------ group quantizers */
static long clampl(long v, long lo, long hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* quant.hpp:70-76 store_scale, Scalar = float */
static float store_scale_f32(float scale, float fallback, int f16) {
    float stored = scale;
    if (stored == 0.0f) stored = fallback;
    if (f16) stored = mqo_round_scale_f16(stored);
    return stored;
}
/* quant.hpp:70-76 store_scale, Scalar = double (scale rounded through f32) */
static double store_scale_f64(double scale, double fallback, int f16) {
    float stored = (float)scale;
    if (stored == 0.0f) stored = (float)fallback;
    if (f16) stored = mqo_round_scale_f16(stored);
    return (double)stored;
}

/* quant.hpp:117-140, Scalar = float (the activation path, gemm.cpp:190) */
int mqo_quant_group_sym_f32(const float* x, int64_t len, int bits, int f16,
                            int8_t* codes, float* scale_out) {
    if (bits != 4 && bits != 8) return MQO_USAGE;
    if (len <= 0) return MQO_USAGE;
    for (int64_t i = 0; i < len; ++i)
        if (!isfinite((double)x[i])) return MQO_DATA;         /* quant.hpp:56-64 */
    float amax = 0.0f;
    for (int64_t i = 0; i < len; ++i) {
        const float a = fabsf(x[i]);
        amax = (amax < a) ? a : amax;                          /* std::max */
    }
    const int qmax = (1 << (bits - 1)) - 1;
    const float fallback = (amax < 1e-8f) ? 1e-8f : amax;
    const float scale = store_scale_f32(amax == 0.0f ? 1e-8f : amax / (float)qmax, fallback, f16);
    for (int64_t i = 0; i < len; ++i) {
        const long code = lround((double)roundf(x[i] / scale));
        codes[i] = (int8_t)clampl(code, -qmax, qmax);
    }
    *scale_out = scale;
    return MQO_OK;
}

/* quant.hpp:117-140, Scalar = double (8-bit weights) */
int mqo_quant_group_sym_f64(const double* x, int64_t len, int bits, int f16,
                            int8_t* codes, float* scale_out) {
    if (bits != 4 && bits != 8) return MQO_USAGE;
    if (len <= 0) return MQO_USAGE;
    for (int64_t i = 0; i < len; ++i)
        if (!isfinite(x[i])) return MQO_DATA;
    double amax = 0.0;
    for (int64_t i = 0; i < len; ++i) {
        const double a = fabs(x[i]);
        amax = (amax < a) ? a : amax;
    }
    const int qmax = (1 << (bits - 1)) - 1;
    const double fallback = (amax < 1e-8) ? 1e-8 : amax;
    const double scale = store_scale_f64(amax == 0.0 ? 1e-8 : amax / (double)qmax, fallback, f16);
    for (int64_t i = 0; i < len; ++i) {
        const long code = lround((double)round(x[i] / scale));
        codes[i] = (int8_t)clampl(code, -qmax, qmax);
    }
    *scale_out = (float)scale;
    return MQO_OK;
}

/* quant.hpp:84-112, Scalar = float */
int mqo_quant_group_asym_f32(const float* x, int64_t len, int bits, int f16,
                             uint8_t* codes, float* scale_out, uint8_t* zp_out) {
    if (bits != 4 && bits != 8) return MQO_USAGE;
    if (len <= 0) return MQO_USAGE;
    for (int64_t i = 0; i < len; ++i)
        if (!isfinite((double)x[i])) return MQO_DATA;
    float mn = x[0], mx = x[0];
    for (int64_t i = 1; i < len; ++i) {
        if (x[i] < mn) mn = x[i];
        if (!(x[i] < mx)) mx = x[i];
    }
    const int qmax = (1 << bits) - 1;
    float fallback = fabsf(mn);
    if (fallback < fabsf(mx)) fallback = fabsf(mx);
    if (fallback < 1e-8f) fallback = 1e-8f;
    const float scale = store_scale_f32((mx == mn) ? fallback : (mx - mn) / (float)qmax, fallback, f16);
    const uint8_t zp = (uint8_t)clampl(lround((double)roundf(-mn / scale)), 0, qmax);
    for (int64_t i = 0; i < len; ++i) {
        const long code = lround((double)roundf(x[i] / scale)) + (long)zp;
        codes[i] = (uint8_t)clampl(code, 0, qmax);
    }
    *scale_out = scale;
    *zp_out = zp;
    return MQO_OK;
}

/* quant.hpp:84-112, Scalar = double (4-bit weights) */
int mqo_quant_group_asym_f64(const double* x, int64_t len, int bits, int f16,
                             uint8_t* codes, float* scale_out, uint8_t* zp_out) {
    if (bits != 4 && bits != 8) return MQO_USAGE;
    if (len <= 0) return MQO_USAGE;
    for (int64_t i = 0; i < len; ++i)
        if (!isfinite(x[i])) return MQO_DATA;
    double mn = x[0], mx = x[0];
    for (int64_t i = 1; i < len; ++i) {
        if (x[i] < mn) mn = x[i];
        if (!(x[i] < mx)) mx = x[i];
    }
    const int qmax = (1 << bits) - 1;
    double fallback = fabs(mn);
    if (fallback < fabs(mx)) fallback = fabs(mx);
    if (fallback < 1e-8) fallback = 1e-8;
    const double scale = store_scale_f64((mx == mn) ? fallback : (mx - mn) / (double)qmax, fallback, f16);
    const uint8_t zp = (uint8_t)clampl(lround((double)round(-mn / scale)), 0, qmax);
    for (int64_t i = 0; i < len; ++i) {
        const long code = lround((double)round(x[i] / scale)) + (long)zp;
        codes[i] = (uint8_t)clampl(code, 0, qmax);
    }
    *scale_out = (float)scale;
    *zp_out = zp;
    return MQO_OK;
}

/* ------------------------------------------------------ quantize_tensor */
/* quant.hpp:154-162 */
int64_t mqo_row_stride(int bits, int64_t cols) { return bits == 4 ? (cols + 1) / 2 : cols; }
int64_t mqo_num_groups(int64_t cols, int group) { return cols == 0 ? 0 : (cols + group - 1) / group; }

/* quant.hpp:165-175 */
int mqo_code(const uint8_t* payload, int bits, int sym, int64_t cols, int64_t r, int64_t c) {
    const int64_t base = r * mqo_row_stride(bits, cols);
    if (bits == 4) {
        const uint8_t byte = payload[base + c / 2];
        return (c % 2 == 0) ? (byte & 0x0F) : (byte >> 4);
    }
    const uint8_t byte = payload[base + c];
    return sym ? (int)(int8_t)byte : (int)byte;
}

/* quant.hpp:183-243, shared body for both scalar types */
#define QUANTIZE_TENSOR_BODY(T, SYMFN, ASYMFN)                                               \
    if (bits != 4 && bits != 8) return MQO_USAGE;                                           \
    if (group < 1) return MQO_USAGE;                                                        \
    if (bits == 4 && sym) return MQO_USAGE;                                                 \
    const int64_t G = mqo_num_groups(cols, group);                                          \
    const int64_t stride = mqo_row_stride(bits, cols);                                      \
    memset(payload, 0, (size_t)(rows * stride));                                            \
    uint8_t* row_u4 = (bits == 4) ? (uint8_t*)malloc((size_t)(cols > 0 ? cols : 1)) : NULL; \
    uint8_t* tmp = (uint8_t*)malloc((size_t)(group));                                       \
    int st = MQO_OK;                                                                        \
    for (int64_t r = 0; r < rows && st == MQO_OK; ++r) {                                    \
        for (int64_t g = 0; g < G; ++g) {                                                   \
            const int64_t begin = g * group;                                                \
            const int64_t len = (cols - begin) < group ? (cols - begin) : group;            \
            const T* x = m + r * cols + begin;                                              \
            if (sym) {                                                                      \
                st = SYMFN(x, len, bits, f16, (int8_t*)tmp, &scales[r * G + g]);            \
                if (st != MQO_OK) { if (err_row) *err_row = r; if (err_group) *err_group = g; break; } \
                memcpy(payload + r * stride + begin, tmp, (size_t)len);                     \
            } else {                                                                        \
                st = ASYMFN(x, len, bits, f16, tmp, &scales[r * G + g], &zps[r * G + g]);   \
                if (st != MQO_OK) { if (err_row) *err_row = r; if (err_group) *err_group = g; break; } \
                if (bits == 4) memcpy(row_u4 + begin, tmp, (size_t)len);                    \
                else memcpy(payload + r * stride + begin, tmp, (size_t)len);                \
            }                                                                               \
        }                                                                                   \
        if (st == MQO_OK && bits == 4 && cols > 0)                                          \
            mqo_pack_nibbles(row_u4, cols, payload + r * stride);                           \
    }                                                                                       \
    free(row_u4);                                                                           \
    free(tmp);                                                                              \
    return st;

int mqo_quantize_tensor_f32(const float* m, int64_t rows, int64_t cols, int bits, int sym,
                            int group, int f16, uint8_t* payload, float* scales,
                            uint8_t* zps, int64_t* err_row, int64_t* err_group) {
    QUANTIZE_TENSOR_BODY(float, mqo_quant_group_sym_f32, mqo_quant_group_asym_f32)
}

int mqo_quantize_tensor_f64(const double* m, int64_t rows, int64_t cols, int bits, int sym,
                            int group, int f16, uint8_t* payload, float* scales,
                            uint8_t* zps, int64_t* err_row, int64_t* err_group) {
    QUANTIZE_TENSOR_BODY(double, mqo_quant_group_sym_f64, mqo_quant_group_asym_f64)
}

/* ------------------------------------------------------------ partition */
/* proj/src/mixed.cpp:56-70 */
int mqo_partition_maps(int64_t out_features, const int32_t* promoted, int64_t n_promoted,
                       int32_t* map8, int64_t* n8, int32_t* map4, int64_t* n4) {
    uint8_t* is_p = (uint8_t*)calloc((size_t)(out_features > 0 ? out_features : 1), 1);
    for (int64_t i = 0; i < n_promoted; ++i) {
        const int32_t ch = promoted[i];
        if (ch < 0 || ch >= out_features || is_p[ch]) { free(is_p); return MQO_USAGE; }
        is_p[ch] = 1;
    }
    int64_t a = 0, b = 0;
    for (int64_t ch = 0; ch < out_features; ++ch) {
        if (is_p[ch]) map8[a++] = (int32_t)ch;
        else map4[b++] = (int32_t)ch;
    }
    *n8 = a;
    *n4 = b;
    free(is_p);
    return MQO_OK;
}

/* -------------------------------------------------------------- prepack */
/* proj/src/gemm.cpp:89-108 with the group_offset of gemm.hpp:54-58 */
void mqo_prepack(const uint8_t* payload, int bits, int sym, int64_t rows, int64_t cols,
                 int group, uint8_t* packed) {
    const int64_t G = mqo_num_groups(cols, group);
    for (int64_t g = 0; g < G; ++g) {
        const int64_t begin = g * group;
        const int64_t len = (cols - begin) < group ? (cols - begin) : group;
        for (int64_t r = 0; r < rows; ++r) {
            uint8_t* dst = packed + rows * begin + r * len;
            for (int64_t i = 0; i < len; ++i)
                dst[i] = (uint8_t)mqo_code(payload, bits, sym, cols, r, begin + i);
        }
    }
}

/* ------------------------------------------------------------ gemm_block */
/* proj/src/gemm.cpp:51-85: g ascending, r, m; int32 group accumulator
 * (fast: pre-biased with 0x4B400000), I2F, then out += gs * (s_a * s_w) as
 * an f32 multiply followed by an f32 add (no FMA: -ffp-contract=off). */
void mqo_gemm_sub(const int8_t* a_codes, const float* a_scales, int64_t a_scale_cols,
                  int64_t M, int64_t K, int group, const uint8_t* w_payload, int w_bits,
                  int w_sym, const float* w_scales, const uint8_t* w_zps, int64_t rows,
                  int fast, int w_u8, float* out) {
    const int64_t G = mqo_num_groups(K, group);
    int32_t* wrow = (int32_t*)malloc(sizeof(int32_t) * (size_t)(group > 0 ? group : 1));
    for (int64_t g = 0; g < G; ++g) {
        const int64_t begin = g * group;
        const int64_t len = (K - begin) < group ? (K - begin) : group;
        for (int64_t r = 0; r < rows; ++r) {
            const int zero = w_sym ? 0 : w_zps[r * G + g];
            const float sw = w_scales[r * G + g];
            /* the reference reads prepacked codes back as uint8_t (gemm.cpp:62,73-74
             * after the uint8_t cast of gemm.cpp:103): w_u8 reproduces that */
            for (int64_t i = 0; i < len; ++i) {
                const int c = mqo_code(w_payload, w_bits, w_sym, K, r, begin + i);
                wrow[i] = (w_u8 ? (int)(uint8_t)c : c) - zero;
            }
            for (int64_t m = 0; m < M; ++m) {
                const int8_t* a = a_codes + m * K + begin;
                int32_t acc = fast ? I2F_BIAS_INT : 0;
                for (int64_t i = 0; i < len; ++i) acc += (int32_t)a[i] * wrow[i];
                const float gs = fast ? bits_to_f32((uint32_t)acc) - bits_to_f32((uint32_t)I2F_BIAS_INT)
                                      : (float)acc;
                const float sa = (a_scale_cols == 1) ? a_scales[m] : a_scales[m * G + g];
                const float t = sa * sw;
                const float p = gs * t;
                out[m * rows + r] = out[m * rows + r] + p;
            }
        }
    }
    free(wrow);
}

/* step-1 integer group sums (gemm.cpp:64-75 without the I2F bias) */
void mqo_group_partials(const int8_t* a_codes, int64_t M, int64_t K, int group,
                        const uint8_t* w_payload, int w_bits, int w_sym,
                        const uint8_t* w_zps, int64_t rows, int w_u8, int32_t* partials) {
    const int64_t G = mqo_num_groups(K, group);
    for (int64_t g = 0; g < G; ++g) {
        const int64_t begin = g * group;
        const int64_t len = (K - begin) < group ? (K - begin) : group;
        for (int64_t m = 0; m < M; ++m)
            for (int64_t r = 0; r < rows; ++r) {
                const int zero = w_sym ? 0 : w_zps[r * G + g];
                int32_t acc = 0;
                for (int64_t i = 0; i < len; ++i) {
                    const int c = mqo_code(w_payload, w_bits, w_sym, K, r, begin + i);
                    acc += (int32_t)a_codes[m * K + begin + i] * ((w_u8 ? (int)(uint8_t)c : c) - zero);
                }
                partials[(g * M + m) * rows + r] = acc;
            }
    }
}

/* -------------------------------------------------------------- scatter */
/* proj/src/mixed.cpp:83-120 */
int mqo_reassemble(const float* y8, int64_t n8, const float* y4, int64_t n4,
                   const int32_t* map8, const int32_t* map4, int64_t M, int64_t N, float* out) {
    uint8_t* written = (uint8_t*)calloc((size_t)(N > 0 ? N : 1), 1);
    int st = MQO_OK;
    for (int pass = 0; pass < 2 && st == MQO_OK; ++pass) {
        const float* y = pass == 0 ? y8 : y4;
        const int64_t n = pass == 0 ? n8 : n4;
        const int32_t* map = pass == 0 ? map8 : map4;
        for (int64_t k = 0; k < n; ++k) {
            const int32_t ch = map[k];
            if (ch < 0 || ch >= N || written[ch]++) { st = MQO_DATA; break; }
            for (int64_t m = 0; m < M; ++m) out[m * N + ch] = y[m * n + k];
        }
    }
    for (int64_t ch = 0; ch < N && st == MQO_OK; ++ch)
        if (!written[ch]) st = MQO_DATA;
    free(written);
    return st;
}

/* ------------------------------------------------------ bench generator */
/* proj/src/gemm.cpp:211-227 */
int64_t mqo_bench_inputs(int64_t m, int64_t n, int64_t k, double percent, uint64_t seed,
                         double* W, float* A, int32_t* promoted) {
    mqo_rng rng;
    mqo_rng_seed(&rng, seed);
    for (int64_t r = 0; r < n; ++r)
        for (int64_t c = 0; c < k; ++c) W[r * k + c] = mqo_rng_normal(&rng);
    for (int64_t r = 0; r < m; ++r)
        for (int64_t c = 0; c < k; ++c) A[r * k + c] = (float)mqo_rng_normal(&rng);
    const int64_t n_prom = llround(percent * (double)n);
    int32_t* all = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) all[i] = (int32_t)i;
    for (int64_t i = n - 1; i > 0; --i) {
        const int64_t j = mqo_rng_uniform_int(&rng, 0, i + 1);
        const int32_t t = all[i];
        all[i] = all[j];
        all[j] = t;
    }
    for (int64_t i = 0; i < n_prom; ++i) promoted[i] = all[i];
    free(all);
    return n_prom;
}

/* ------------------------------------------------- whole mixed linear */
/* proj/src/gemm.cpp:183-192 -> 140-181 -> mixed.cpp:83-120 */
int mqo_mixed_linear(const mqo_layer* L, const float* A, int64_t M, int act_group, int fast,
                     int w8_u8, int8_t* a_codes_out, float* a_scales_out, float* out) {
    const int64_t K = L->K;
    const int64_t Ga = mqo_num_groups(K, act_group);
    int st = mqo_quantize_tensor_f32(A, M, K, 8, 1, act_group, 0, (uint8_t*)a_codes_out,
                                     a_scales_out, NULL, NULL, NULL);
    if (st != MQO_OK) return st;
    float* y8 = (float*)calloc((size_t)(M * L->n8 + 1), sizeof(float));
    float* y4 = (float*)calloc((size_t)(M * L->n4 + 1), sizeof(float));
    const int64_t sc = (act_group == L->group) ? Ga : 1;
    if (act_group != L->group && Ga != 1) { free(y8); free(y4); return MQO_USAGE; }
    if (L->n8 > 0)
        mqo_gemm_sub(a_codes_out, a_scales_out, sc, M, K, L->group, L->p8, 8, 1, L->s8, NULL,
                     L->n8, fast, w8_u8, y8);
    if (L->n4 > 0)
        mqo_gemm_sub(a_codes_out, a_scales_out, sc, M, K, L->group, L->p4, 4, 0, L->s4, L->z4,
                     L->n4, fast, 0, y4);
    st = mqo_reassemble(y8, L->n8, y4, L->n4, L->map8, L->map4, M, L->N, out);
    free(y8);
    free(y4);
    return st;
}

/* ----------------------------------------------------------------- FNV */
/* proj/src/gemm.cpp:194-204 */
uint64_t mqo_fnv1a(const void* data, uint64_t n) {
    const uint8_t* b = (const uint8_t*)data;
    uint64_t h = 0xCBF29CE484222325ULL;
    for (uint64_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 0x100000001B3ULL;
    }
    return h;
}

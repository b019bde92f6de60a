// mq_host.cpp — host-side packing for the MixLLM linear engine: the
// quantizers, nibble codec, partition, reference prepack and the bench
// generator, bit-exact with the reference (proj/). Compiled with
// -ffp-contract=off and no -march so every f32/f64 operation rounds exactly as
// the reference build does (proj/src/CMakeLists.txt:14).
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "mq_internal.hpp"

namespace mq {

thread_local std::string g_last_error;

mq_status fail(mq_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

// ------------------------------------------------------------ f16 rounding
// proj/src/quant.cpp:20-51 — f32 -> binary16 bits, round to nearest even.
static uint16_t to_half_bits(float f) {
    const uint32_t x = std::bit_cast<uint32_t>(f);
    const uint16_t sign = static_cast<uint16_t>((x >> 16) & 0x8000u);
    const uint32_t e = (x >> 23) & 0xFFu;
    uint32_t mant = x & 0x7FFFFFu;
    if (e == 0xFFu) return static_cast<uint16_t>(sign | 0x7C00u | (mant ? 0x200u : 0));
    const int he = static_cast<int>(e) - 112;
    if (he >= 31) return static_cast<uint16_t>(sign | 0x7C00u);
    if (he <= 0) {
        if (he < -10) return sign;
        mant |= 0x800000u;
        const int sh = 14 - he;
        uint32_t hm = mant >> sh;
        const uint32_t rem = mant & ((1u << sh) - 1), half = 1u << (sh - 1);
        hm += (rem > half || (rem == half && (hm & 1u))) ? 1u : 0u;
        return static_cast<uint16_t>(sign | hm);
    }
    uint16_t h = static_cast<uint16_t>(sign | (static_cast<uint32_t>(he) << 10) | (mant >> 13));
    const uint32_t rem = mant & 0x1FFFu;
    h += (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ? 1 : 0;
    return h;
}

// proj/src/quant.cpp:53-77
static float from_half_bits(uint16_t h) {
    const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16;
    uint32_t e = (h >> 10) & 0x1Fu, mant = h & 0x3FFu, bits;
    if (e == 0) {
        if (mant == 0) {
            bits = sign;
        } else {
            int ex = -14;
            for (; !(mant & 0x400u); mant <<= 1) --ex;
            bits = sign | (static_cast<uint32_t>(ex + 127) << 23) | ((mant & 0x3FFu) << 13);
        }
    } else if (e == 0x1Fu) {
        bits = sign | 0x7F800000u | (mant << 13);
    } else {
        bits = sign | ((e + 112) << 23) | (mant << 13);
    }
    return std::bit_cast<float>(bits);
}

float round_scale_f16(float s) {
    const float r = from_half_bits(to_half_bits(s));
    return r > 0.0f ? r : 5.9604644775390625e-8f;  // smallest positive f16 subnormal
}

// ---------------------------------------------------------- group quantizers
// quant.hpp:70-76: scales are stored as f32 (optionally on the f16 grid) and
// codes are computed against the stored value.
template <class S>
static S stored_scale(S s, S fallback, bool f16) {
    float v = static_cast<float>(s);
    if (v == 0.0f) v = static_cast<float>(fallback);
    if (f16) v = round_scale_f16(v);
    return static_cast<S>(v);
}

static long clampl(long v, long lo, long hi) { return std::min(std::max(v, lo), hi); }

template <class S>
static bool all_finite(const S* x, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(static_cast<double>(x[i]))) return false;
    return true;
}

// quant.hpp:117-140 (symmetric): s = amax/qmax, code = clamp(round(x/s)).
template <class S>
static mq_status group_sym(const S* x, int64_t n, int bits, bool f16, uint8_t* codes,
                           float* scale) {
    if (!all_finite(x, n)) return MQ_DATA;
    S amax = 0;
    for (int64_t i = 0; i < n; ++i) amax = std::max(amax, std::abs(x[i]));
    const int qmax = (1 << (bits - 1)) - 1;
    const S s = stored_scale<S>(amax == S(0) ? S(1e-8) : amax / S(qmax),
                                std::max(amax, S(1e-8)), f16);
    for (int64_t i = 0; i < n; ++i) {
        const long c = std::lround(static_cast<double>(std::round(x[i] / s)));
        codes[i] = static_cast<uint8_t>(static_cast<int8_t>(clampl(c, -qmax, qmax)));
    }
    *scale = static_cast<float>(s);
    return MQ_OK;
}

// quant.hpp:84-112 (asymmetric): s = (max-min)/qmax, z = clamp(round(-min/s)).
template <class S>
static mq_status group_asym(const S* x, int64_t n, int bits, bool f16, uint8_t* codes,
                            float* scale, uint8_t* zp) {
    if (!all_finite(x, n)) return MQ_DATA;
    const auto [lo, hi] = std::minmax_element(x, x + n);
    const S mn = *lo, mx = *hi;
    const int qmax = (1 << bits) - 1;
    const S fb = std::max({std::abs(mn), std::abs(mx), S(1e-8)});
    const S s = stored_scale<S>(mx == mn ? fb : (mx - mn) / S(qmax), fb, f16);
    const auto z = static_cast<uint8_t>(
        clampl(std::lround(static_cast<double>(std::round(-mn / s))), 0, qmax));
    for (int64_t i = 0; i < n; ++i) {
        const long c = std::lround(static_cast<double>(std::round(x[i] / s))) + long(z);
        codes[i] = static_cast<uint8_t>(clampl(c, 0, qmax));
    }
    *scale = static_cast<float>(s);
    *zp = z;
    return MQ_OK;
}

mq_status check_scheme(const mq_scheme* s) {
    if (!s) return fail(MQ_USAGE, "scheme is null");
    if (s->bit_width != 4 && s->bit_width != 8)
        return fail(MQ_USAGE, "bit_width must be 4 or 8, got " + std::to_string(s->bit_width));
    if (s->group_size < 1)
        return fail(MQ_USAGE, "group_size must be >= 1, got " + std::to_string(s->group_size));
    return MQ_OK;
}

// quant.hpp:183-243: groups along the row; 4-bit payload packed per row.
template <class S>
static mq_status quantize_tensor(const S* m, int64_t rows, int64_t cols, const mq_scheme* sc,
                                 uint8_t* payload, float* scales, uint8_t* zps,
                                 int64_t* err_row, int64_t* err_group) {
    if (mq_status st = check_scheme(sc)) return st;
    const int bits = sc->bit_width, g = sc->group_size;
    const bool sym = sc->symmetric != 0, f16 = sc->scale_f16_storage != 0;
    if (bits == 4 && sym) return fail(MQ_USAGE, "quantize_tensor: 4-bit symmetric tensors are not supported");
    const int64_t G = num_groups(cols, g), stride = row_stride(bits, cols);
    std::memset(payload, 0, static_cast<size_t>(rows * stride));
    std::vector<uint8_t> row(static_cast<size_t>(std::max<int64_t>(cols, 1)));
    for (int64_t r = 0; r < rows; ++r) {
        for (int64_t gi = 0; gi < G; ++gi) {
            const int64_t b = gi * g, n = std::min<int64_t>(g, cols - b);
            const S* x = m + r * cols + b;
            mq_status st = sym ? group_sym(x, n, bits, f16, row.data() + b, &scales[r * G + gi])
                               : group_asym(x, n, bits, f16, row.data() + b, &scales[r * G + gi],
                                            &zps[r * G + gi]);
            if (st != MQ_OK) {
                if (err_row) *err_row = r;
                if (err_group) *err_group = gi;
                return fail(st, "row " + std::to_string(r) + ", group " + std::to_string(gi) +
                                    ": quantize: non-finite input value");
            }
        }
        if (bits == 4) pack_nibbles_raw(row.data(), cols, payload + r * stride);
        else std::memcpy(payload + r * stride, row.data(), static_cast<size_t>(cols));
    }
    return MQ_OK;
}

// ------------------------------------------------------------ nibble codec
// proj/src/tensor.cpp:63-78: byte k = v[2k] | v[2k+1] << 4, pad high nibble 0.
void pack_nibbles_raw(const uint8_t* v, int64_t n, uint8_t* out) {
    for (int64_t k = 0; k < n / 2; ++k) out[k] = static_cast<uint8_t>(v[2 * k] | (v[2 * k + 1] << 4));
    if (n & 1) out[n / 2] = v[n - 1];
}

// ---------------------------------------------------------------- partition
// proj/src/mixed.cpp:56-70: map8 = ascending promoted ids, map4 = the rest.
mq_status partition_maps(int64_t N, const int32_t* promoted, int64_t np,
                         std::vector<int32_t>& map8, std::vector<int32_t>& map4) {
    std::vector<uint8_t> is_p(static_cast<size_t>(N), 0);
    for (int64_t i = 0; i < np; ++i) {
        const int32_t ch = promoted[i];
        if (ch < 0 || ch >= N)
            return fail(MQ_USAGE, "promoted channel " + std::to_string(ch) + " is out of range");
        if (is_p[ch]) return fail(MQ_USAGE, "promoted channel " + std::to_string(ch) + " listed twice");
        is_p[ch] = 1;
    }
    map8.clear();
    map4.clear();
    for (int64_t ch = 0; ch < N; ++ch) (is_p[ch] ? map8 : map4).push_back(static_cast<int32_t>(ch));
    return MQ_OK;
}

// mixed.cpp:14-44 + quant.cpp:81-101 on a descriptor.
mq_status validate_desc(const mq_layer_desc* d) {
    if (mq_status st = validate_maps(d)) return st;
    const int64_t G = num_groups(d->in_features, d->group_size);
    auto positive = [&](const float* s, int64_t n) {
        for (int64_t i = 0; i < n; ++i)
            if (!(s[i] > 0.0f)) return false;
        return true;
    };
    if (d->n8 > 0 && !positive(d->scales8, d->n8 * G))
        return fail(MQ_DATA, "quantized tensor has a non-positive scale");
    if (d->n4 > 0 && !positive(d->scales4, d->n4 * G))
        return fail(MQ_DATA, "quantized tensor has a non-positive scale");
    if (d->n4 > 0)
        for (int64_t i = 0; i < d->n4 * G; ++i)
            if (d->zero_points4[i] > 15) return fail(MQ_DATA, "4-bit zero point out of [0, 15]");
    return MQ_OK;
}

// mixed.cpp:14-44: shapes and index maps (host), payload pointers present.
mq_status validate_maps(const mq_layer_desc* d) {
    if (!d) return fail(MQ_USAGE, "layer descriptor is null");
    if (d->out_features < 0 || d->in_features < 0 || d->n8 < 0 || d->n4 < 0)
        return fail(MQ_DATA, "mixed layer has a negative shape");
    if (d->group_size < 1) return fail(MQ_USAGE, "group_size must be >= 1");
    if (d->n8 + d->n4 != d->out_features)
        return fail(MQ_DATA, "mixed layer: index map sizes disagree with sub-problems");
    std::vector<int> seen(static_cast<size_t>(d->out_features), 0);
    for (int w = 0; w < 2; ++w) {
        const int32_t* map = w ? d->index_map4 : d->index_map8;
        const int64_t n = w ? d->n4 : d->n8;
        if (n > 0 && !map) return fail(MQ_DATA, "mixed layer: missing index map");
        for (int64_t k = 0; k < n; ++k) {
            if (map[k] < 0 || map[k] >= d->out_features)
                return fail(MQ_DATA, "mixed layer: channel index out of range");
            ++seen[map[k]];
        }
    }
    for (size_t ch = 0; ch < seen.size(); ++ch)
        if (seen[ch] != 1)
            return fail(MQ_DATA, "mixed layer: output channel " + std::to_string(ch) +
                                     (seen[ch] == 0 ? " is unassigned" : " is assigned twice"));
    if (d->n8 > 0 && (!d->payload8 || !d->scales8))
        return fail(MQ_DATA, "mixed layer: sub8 payload/scales missing");
    if (d->n4 > 0 && (!d->payload4 || !d->scales4 || !d->zero_points4))
        return fail(MQ_DATA, "asymmetric quantized tensor is missing zero points");
    return MQ_OK;
}

int raw_code(const uint8_t* payload, int bits, int64_t cols, int64_t r, int64_t c) {
    if (bits == 4) {
        const uint8_t b = payload[r * row_stride(4, cols) + c / 2];
        return (c & 1) ? (b >> 4) : (b & 0x0F);
    }
    return static_cast<int8_t>(payload[r * cols + c]);
}

}  // namespace mq

using namespace mq;

// ====================================================================== C ABI
extern "C" {

const char* mq_last_error(void) { return g_last_error.c_str(); }
const char* mq_version(void) { return "mixllm_b200 0.1 (sm_100a tcgen05)"; }

mq_status mq_quantize_tensor_f32(const float* m, int64_t rows, int64_t cols, const mq_scheme* s,
                                 uint8_t* payload, float* scales, uint8_t* zps, int64_t* er,
                                 int64_t* eg) {
    return quantize_tensor<float>(m, rows, cols, s, payload, scales, zps, er, eg);
}

mq_status mq_quantize_tensor_f64(const double* m, int64_t rows, int64_t cols, const mq_scheme* s,
                                 uint8_t* payload, float* scales, uint8_t* zps, int64_t* er,
                                 int64_t* eg) {
    return quantize_tensor<double>(m, rows, cols, s, payload, scales, zps, er, eg);
}

mq_status mq_pack_nibbles(const uint8_t* v, int64_t n, uint8_t* out) {
    for (int64_t i = 0; i < n; ++i)
        if (v[i] > 15)
            return fail(MQ_DATA, "pack_nibbles: value " + std::to_string(v[i]) + " at index " +
                                     std::to_string(i) + " is out of [0, 15]");
    pack_nibbles_raw(v, n, out);
    return MQ_OK;
}

mq_status mq_unpack_nibbles(const uint8_t* b, int64_t nbytes, int64_t count, uint8_t* out) {
    if (count < 0 || count > nbytes * 2)
        return fail(MQ_DATA, "unpack_nibbles: count " + std::to_string(count) +
                                 " exceeds capacity of " + std::to_string(nbytes) + " bytes");
    for (int64_t i = 0; i < count; ++i) out[i] = (i & 1) ? (b[i / 2] >> 4) : (b[i / 2] & 0x0F);
    return MQ_OK;
}

float mq_round_scale_f16(float s) { return round_scale_f16(s); }

float mq_fast_i2f(int32_t x) {
    // gemm.hpp:27-31: exact for x in [-2^22, 2^22).
    return std::bit_cast<float>(static_cast<int32_t>(static_cast<uint32_t>(x) + 0x4B400000u)) -
           12582912.0f;
}

mq_status mq_partition_and_quantize(const double* W, int64_t N, int64_t K, const int32_t* promoted,
                                    int64_t np, const mq_scheme* large, const mq_scheme* small,
                                    mq_host_layer_t* out) {
    if (!W && N * K > 0) return fail(MQ_USAGE, "weight matrix is null");
    if (mq_status st = check_scheme(large)) return st;
    if (mq_status st = check_scheme(small)) return st;
    if (large->group_size != small->group_size)
        return fail(MQ_DATA, "mixed layer: sub-problems must share group boundaries");
    auto* h = new mq_host_layer_s;
    if (mq_status st = partition_maps(N, promoted, np, h->map8, h->map4)) {
        delete h;
        return st;
    }
    h->N = N;
    h->K = K;
    h->group = large->group_size;
    h->large = *large;
    h->small = *small;
    const int64_t G = num_groups(K, h->group);
    auto quantize_sub = [&](const std::vector<int32_t>& map, const mq_scheme* sc,
                            std::vector<uint8_t>& payload, std::vector<float>& scales,
                            std::vector<uint8_t>& zps) -> mq_status {
        const int64_t rows = static_cast<int64_t>(map.size());
        std::vector<double> sub(static_cast<size_t>(rows * K));
        for (int64_t k = 0; k < rows; ++k)  // gather (mixed.cpp:72-76)
            std::copy(W + map[k] * K, W + (map[k] + 1) * K, sub.begin() + k * K);
        payload.assign(static_cast<size_t>(rows * row_stride(sc->bit_width, K)), 0);
        scales.assign(static_cast<size_t>(rows * G), 0.0f);
        zps.assign(sc->symmetric ? 0 : static_cast<size_t>(rows * G), 0);
        return quantize_tensor<double>(sub.data(), rows, K, sc, payload.data(), scales.data(),
                                       sc->symmetric ? nullptr : zps.data(), nullptr, nullptr);
    };
    mq_status st = quantize_sub(h->map8, large, h->p8, h->s8, h->z8);
    if (st == MQ_OK) st = quantize_sub(h->map4, small, h->p4, h->s4, h->z4);
    if (st != MQ_OK) {
        delete h;
        return st;
    }
    *out = h;
    return MQ_OK;
}

mq_status mq_host_layer_desc(mq_host_layer_t h, mq_layer_desc* d) {
    if (!h || !d) return fail(MQ_USAGE, "null host layer");
    if (h->large.bit_width != 8 || !h->large.symmetric || h->small.bit_width != 4 ||
        h->small.symmetric)
        return fail(MQ_USAGE, "engine requires 8-bit symmetric / 4-bit asymmetric sub-problems");
    d->out_features = h->N;
    d->in_features = h->K;
    d->group_size = h->group;
    d->n8 = static_cast<int64_t>(h->map8.size());
    d->n4 = static_cast<int64_t>(h->map4.size());
    d->index_map8 = h->map8.data();
    d->index_map4 = h->map4.data();
    d->payload8 = h->p8.data();
    d->scales8 = h->s8.data();
    d->payload4 = h->p4.data();
    d->scales4 = h->s4.data();
    d->zero_points4 = h->z4.data();
    return MQ_OK;
}

void mq_host_layer_destroy(mq_host_layer_t h) { delete h; }

mq_status mq_validate_layer(const mq_layer_desc* d) { return validate_desc(d); }

mq_status mq_prepack_reference(const mq_layer_desc* d, int32_t which, uint8_t* out) {
    if (mq_status st = validate_desc(d)) return st;
    // gemm.cpp:89-108 with gemm.hpp:54-58: codes[rows*begin + r*len + i].
    const int bits = which == 0 ? 8 : 4;
    const int64_t rows = which == 0 ? d->n8 : d->n4, K = d->in_features;
    const uint8_t* p = which == 0 ? d->payload8 : d->payload4;
    const int g = d->group_size;
    for (int64_t gi = 0; gi < num_groups(K, g); ++gi) {
        const int64_t b = gi * g, n = std::min<int64_t>(g, K - b);
        for (int64_t r = 0; r < rows; ++r)
            for (int64_t i = 0; i < n; ++i)
                out[rows * b + r * n + i] = static_cast<uint8_t>(raw_code(p, bits, K, r, b + i));
    }
    return MQ_OK;
}

mq_status mq_reassemble_output(const float* y8, int64_t n8, const float* y4, int64_t n4,
                               const int32_t* map8, const int32_t* map4, int64_t M, int64_t N,
                               float* out) {
    // mixed.cpp:83-120: every output column written exactly once.
    std::vector<uint8_t> written(static_cast<size_t>(N), 0);
    for (int w = 0; w < 2; ++w) {
        const float* y = w ? y4 : y8;
        const int32_t* map = w ? map4 : map8;
        const int64_t n = w ? n4 : n8;
        for (int64_t k = 0; k < n; ++k) {
            const int32_t ch = map[k];
            if (ch < 0 || ch >= N) return fail(MQ_DATA, "reassemble_output: channel index out of range");
            if (written[ch]++)
                return fail(MQ_DATA, "reassemble_output: output channel " + std::to_string(ch) + " written twice");
            for (int64_t m = 0; m < M; ++m) out[m * N + ch] = y[m * n + k];
        }
    }
    for (int64_t ch = 0; ch < N; ++ch)
        if (!written[ch])
            return fail(MQ_DATA, "reassemble_output: output channel " + std::to_string(ch) + " never written");
    return MQ_OK;
}

int64_t mq_bench_inputs(int64_t m, int64_t n, int64_t k, double percent, uint64_t seed,
                        double* W, float* A, int32_t* promoted) {
    // gemm.cpp:211-227 with rng.hpp:16-82, draw for draw.
    Xoshiro rng(seed);
    for (int64_t i = 0; i < n * k; ++i) W[i] = rng.normal();
    for (int64_t i = 0; i < m * k; ++i) A[i] = static_cast<float>(rng.normal());
    const int64_t np = std::llround(percent * static_cast<double>(n));
    std::vector<int32_t> all(static_cast<size_t>(n));
    std::iota(all.begin(), all.end(), 0);
    for (int64_t i = n - 1; i > 0; --i) std::swap(all[i], all[rng.uniform_int(0, i + 1)]);
    std::copy(all.begin(), all.begin() + np, promoted);
    return np;
}

mq_status mq_shard_plan(const mq_layer_desc* d, int32_t world, int64_t* shard_cols, int32_t* colmap) {
    if (!d || !shard_cols) return fail(MQ_USAGE, "mq_shard_plan: null argument");
    if (world < 1) return fail(MQ_USAGE, "world must be >= 1");
    if (d->n8 < 0 || d->n4 < 0 || d->n8 + d->n4 != d->out_features)
        return fail(MQ_DATA, "index maps do not cover the output features");
    auto lo = [&](int64_t n, int64_t r) { return n * r / world; };
    int64_t sc = 0;
    for (int64_t r = 0; r < world; ++r)
        sc = std::max(sc, (lo(d->n8, r + 1) - lo(d->n8, r)) + (lo(d->n4, r + 1) - lo(d->n4, r)));
    *shard_cols = sc;
    if (!colmap) return MQ_OK;
    for (int64_t r = 0; r < world; ++r) {
        int64_t j = 0;
        int32_t* row = colmap + r * sc;
        for (int64_t i = lo(d->n8, r); i < lo(d->n8, r + 1); ++i) row[j++] = d->index_map8[i];
        for (int64_t i = lo(d->n4, r); i < lo(d->n4, r + 1); ++i) row[j++] = d->index_map4[i];
        for (; j < sc; ++j) row[j] = -1;
    }
    return MQ_OK;
}

uint64_t mq_fnv1a(const void* data, uint64_t n) {
    const auto* b = static_cast<const uint8_t*>(data);
    uint64_t h = 0xCBF29CE484222325ULL;
    for (uint64_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001B3ULL;
    return h;
}

}  // extern "C"

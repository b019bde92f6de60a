// ref_capi.cpp — extern "C" harness around the REFERENCE's own implementation.
//
// TEST INFRASTRUCTURE ONLY (the checker and the CPU baseline, never product).
// Compiled by oracle/Makefile.ref together with the reference sources as they
// lie under /root/reference/proj/src (not copied) into oracle/_ref/libmqref.so.
// Each entry calls the reference's public C++ API unchanged:
//   partition_and_quantize   proj/src/mixed.cpp:46-81
//   execute_mixed_linear     proj/src/gemm.cpp:183-192
//   quantize_tensor          proj/include/mixquant/quant.hpp:183-243
//   prepack_weights          proj/src/gemm.cpp:89-108
//   run_bench                proj/src/gemm.cpp:206-259
//   save/load_quantized_model proj/src/mixed.cpp:308-370 (quantized.json I/O)
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "mixquant/gemm.hpp"
#include "mixquant/mixed.hpp"
#include "mixquant/quant.hpp"
#include "mixquant/tensor.hpp"

using namespace mixquant;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const UsageError& e) {
        g_err = e.what();
        return 1;
    } catch (const DataError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

struct RefLayer {
    MixedLinearLayer layer;
};
} // namespace

extern "C" {

const char* mqref_last_error() { return g_err.c_str(); }

int mqref_run_bench(int64_t m, int64_t n, int64_t k, double percent, int group, int fast,
                    int workers, int repeats, uint64_t seed, double* wall_ms, double* gops,
                    char* checksum17) {
    return guarded([&] {
        const BenchResult r = run_bench(m, n, k, percent, group,
                                        fast ? I2FMode::Fast : I2FMode::Native, workers,
                                        repeats, seed);
        *wall_ms = r.wall_ms;
        *gops = r.gops;
        std::snprintf(checksum17, 17, "%s", r.checksum.c_str());
    });
}

int mqref_layer_create(const double* W, int64_t n, int64_t k, const int32_t* promoted,
                       int64_t n_promoted, int group, void** out) {
    return guarded([&] {
        MatrixRMd w(n, k);
        std::memcpy(w.data(), W, sizeof(double) * static_cast<size_t>(n * k));
        std::vector<int> prom(promoted, promoted + n_promoted);
        QuantScheme largebit{8, true, group, false};
        QuantScheme smallbit{4, false, group, false};
        auto* h = new RefLayer;
        h->layer = partition_and_quantize(w, prom, largebit, smallbit, "ref");
        *out = h;
    });
}

void mqref_layer_destroy(void* h) { delete static_cast<RefLayer*>(h); }

void mqref_layer_dims(void* hv, int64_t* n8, int64_t* n4) {
    auto* h = static_cast<RefLayer*>(hv);
    *n8 = h->layer.sub8.rows;
    *n4 = h->layer.sub4.rows;
}

// Exports the reference layouts: maps, payloads, scales, zero points.
void mqref_layer_export(void* hv, int32_t* map8, int32_t* map4, uint8_t* p8, float* s8,
                        uint8_t* p4, float* s4, uint8_t* z4) {
    auto* h = static_cast<RefLayer*>(hv);
    const auto& L = h->layer;
    std::copy(L.index_map8.begin(), L.index_map8.end(), map8);
    std::copy(L.index_map4.begin(), L.index_map4.end(), map4);
    if (L.sub8.rows > 0) {
        std::memcpy(p8, L.sub8.payload.data(), L.sub8.payload.size());
        std::memcpy(s8, L.sub8.scales.data(), sizeof(float) * L.sub8.scales.size());
    }
    if (L.sub4.rows > 0) {
        std::memcpy(p4, L.sub4.payload.data(), L.sub4.payload.size());
        std::memcpy(s4, L.sub4.scales.data(), sizeof(float) * L.sub4.scales.size());
        std::memcpy(z4, L.sub4.zero_points.data(), L.sub4.zero_points.size());
    }
}

// Reference prepack of one sub-problem (0 = sub8, 1 = sub4).
int mqref_layer_prepack(void* hv, int which, uint8_t* out) {
    auto* h = static_cast<RefLayer*>(hv);
    return guarded([&] {
        const PrepackedWeights p = prepack_weights(which == 0 ? h->layer.sub8 : h->layer.sub4);
        std::memcpy(out, p.codes.data(), p.codes.size());
    });
}

// The reference forward. Times exactly the execute_mixed_linear call
// (activation quantization + per-call prepack + GEMM + scatter).
// execute_mixed_linear with the activation scheme {8, sym, layer group, act_f16}.
int mqref_layer_forward_f16(void* hv, const float* A, int64_t m, int act_f16, int fast, int workers, float* out,
                            double* ms) {
    auto* h = static_cast<RefLayer*>(hv);
    return guarded([&] {
        MatrixRMf a(m, h->layer.in_features);
        std::memcpy(a.data(), A, sizeof(float) * static_cast<size_t>(a.size()));
        QuantScheme act{8, true, h->layer.sub4.rows > 0 ? h->layer.sub4.scheme.group_size
                                                          : h->layer.sub8.scheme.group_size,
                        act_f16 != 0};
        const auto t0 = std::chrono::steady_clock::now();
        MatrixRMf y = execute_mixed_linear(a, h->layer, act, TileConfig{},
                                           fast ? I2FMode::Fast : I2FMode::Native, workers);
        const auto t1 = std::chrono::steady_clock::now();
        if (ms) *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        std::memcpy(out, y.data(), sizeof(float) * static_cast<size_t>(y.size()));
    });
}

int mqref_layer_forward(void* hv, const float* A, int64_t m, int fast, int workers, float* out, double* ms) {
    return mqref_layer_forward_f16(hv, A, m, 0, fast, workers, out, ms);
}

// quantize_tensor on a float (activation) or double (weight) matrix.
int mqref_quantize_tensor(const void* m, int is_double, int64_t rows, int64_t cols, int bits,
                          int sym, int group, int f16, uint8_t* payload, float* scales,
                          uint8_t* zps) {
    return guarded([&] {
        QuantScheme s{bits, sym != 0, group, f16 != 0};
        QuantizedTensor q;
        if (is_double) {
            MatrixRMd x(rows, cols);
            std::memcpy(x.data(), m, sizeof(double) * static_cast<size_t>(rows * cols));
            q = quantize_tensor<double>(x, s);
        } else {
            MatrixRMf x(rows, cols);
            std::memcpy(x.data(), m, sizeof(float) * static_cast<size_t>(rows * cols));
            q = quantize_tensor<float>(x, s);
        }
        std::memcpy(payload, q.payload.data(), q.payload.size());
        std::memcpy(scales, q.scales.data(), sizeof(float) * q.scales.size());
        if (!sym && zps) std::memcpy(zps, q.zero_points.data(), q.zero_points.size());
    });
}

float mqref_fast_i2f(int32_t x) { return fast_i2f(x); }

// Writes a "mixquant-quantized-v1" directory with the reference's own writer:
// the listed layer handles (mqref_layer_create, renamed) as qm.linears.
int mqref_save_quantized(void* const* layers, const char* const* names, int n_layers, const char* source_model,
                         double percent, int group, const char* dir) {
    return guarded([&] {
        QuantizedModel qm;
        qm.source_model = source_model;
        qm.percent = percent;
        qm.act_scheme = QuantScheme{8, true, group, false};
        qm.largebit = QuantScheme{8, true, group, false};
        qm.smallbit = QuantScheme{4, false, group, false};
        for (int i = 0; i < n_layers; ++i) {
            MixedLinearLayer l = static_cast<RefLayer*>(layers[i])->layer;
            l.name = names[i];
            qm.linears.push_back(std::move(l));
        }
        save_quantized_model(qm, dir);
    });
}

// The reference's reader: one layer handle per linear (N, K per layer in dims).
int mqref_load_quantized(const char* dir, void** handles, int max_layers, int* n_layers, int64_t* dims) {
    return guarded([&] {
        QuantizedModel qm = load_quantized_model(dir);
        *n_layers = static_cast<int>(qm.linears.size());
        for (int i = 0; i < *n_layers && i < max_layers; ++i) {
            auto* h = new RefLayer;
            h->layer = std::move(qm.linears[static_cast<size_t>(i)]);
            dims[2 * i] = h->layer.out_features;
            dims[2 * i + 1] = h->layer.in_features;
            handles[i] = h;
        }
    });
}

} // extern "C"

// C++ drop-in test: the reference's own call shapes (proj/src/gemm.cpp:206-259
// run_bench, proj/src/analysis.cpp:64-75 quantized_forward) compiled against
// include/mixllm/mixquant.hpp. Host checks always run; `--gpu` adds the
// device forward checks (bit-exact against the reference's golden checksums,
// tests/golden/golden.json). Exit code 0 = pass.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "mixllm/mixquant.hpp"

using namespace mixquant;

static int g_fail = 0;
#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c); \
            ++g_fail;                                              \
        }                                                          \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static void host_checks() {
    // quant_core KATs (proj/tests/test_quant_core.cpp:33-80)
    MatrixRMd r(1, 4);
    for (int i = 0; i < 4; ++i) r(0, i) = i;
    auto q = quantize_tensor<double>(r, QuantScheme{4, false, 128, false});
    CHECK(q.scales(0, 0) == 0.2f && q.zero_points(0, 0) == 0);
    CHECK(q.code(0, 0) == 0 && q.code(0, 1) == 5 && q.code(0, 2) == 10 && q.code(0, 3) == 15);
    MatrixRMd s(1, 2);
    s(0, 0) = -1.0, s(0, 1) = 0.5;
    auto q8 = quantize_tensor<double>(s, QuantScheme{8, true, 128, false});
    CHECK(q8.code(0, 0) == -127 && q8.code(0, 1) == 64);
    CHECK(throws<UsageError>([] { quantize_tensor<double>(MatrixRMd(1, 8), QuantScheme{4, true, 128, false}); }));
    MatrixRMd bad(2, 4);
    bad(1, 1) = NAN;
    try {
        quantize_tensor<double>(bad, QuantScheme{4, false, 2, false});
        CHECK(false);
    } catch (const DataError& e) {
        CHECK(std::string(e.what()).find("row 1, group 0") != std::string::npos);
    }
    // nibble codec KATs (proj/tests/test_tensor_store.cpp:10-24)
    CHECK(pack_nibbles({3, 5}) == std::vector<std::uint8_t>{0x53});
    CHECK((pack_nibbles({15, 15, 1}) == std::vector<std::uint8_t>{0xFF, 0x01}));
    CHECK(throws<DataError>([] { pack_nibbles({16}); }));
    // partition + scatter
    MatrixRMd W(6, 8);
    for (int i = 0; i < 48; ++i) W.data()[i] = std::sin(0.37 * i);
    auto L = partition_and_quantize(W, {4, 1}, QuantScheme{8, true, 4, false}, QuantScheme{4, false, 4, false});
    CHECK((L.index_map8 == std::vector<int>{1, 4}) && (L.index_map4 == std::vector<int>{0, 2, 3, 5}));
    CHECK(throws<UsageError>([&] {
        partition_and_quantize(W, {6}, QuantScheme{8, true, 4, false}, QuantScheme{4, false, 4, false});
    }));
    MatrixRMf y8(1, 2), y4(1, 4);
    y8(0, 0) = 10, y8(0, 1) = 40, y4(0, 1) = 2, y4(0, 2) = 3, y4(0, 3) = 5;
    auto Y = reassemble_output(y8, y4, L.index_map8, L.index_map4, 6);
    const float expect[6] = {0, 10, 2, 3, 40, 5};
    CHECK(std::memcmp(Y.data(), expect, sizeof expect) == 0);
    auto pp = prepack_weights(L.sub4);
    CHECK(pp.codes.size() == 32 && pp.codes[pp.group_offset(1, 2)] == uint8_t(L.sub4.code(2, 4)));
    CHECK(fast_i2f(5) == 5.0f && fast_i2f(-(1 << 22)) == -4194304.0f);
}

static void gpu_checks() {
    // C1 through run_bench: the reference's golden checksum
    BenchResult r = run_bench(16, 4096, 4096, 0.10, 128, I2FMode::Fast, 1, 3, 1);
    std::printf("run_bench C1: %.4f ms/call, %.1f GOP/s, checksum %s\n", r.wall_ms, r.gops, r.checksum.c_str());
    CHECK(r.checksum == "5bb508ecbf3b895f");
    r = run_bench(1, 4096, 4096, 0.10, 128, I2FMode::Native, 1, 2, 1);
    CHECK(r.checksum == "eff1a4ac37c56ef3");
    // execute_mixed_linear / execute_mixed_on_codes agree with each other and the golden case (64, 256, 512)
    MatrixRMd W(256, 512);
    MatrixRMf A(64, 512);
    std::vector<int32_t> prom(256);
    const int64_t np = mq_bench_inputs(64, 256, 512, 0.10, 1, W.data(), A.data(), prom.data());
    auto L = partition_and_quantize(W, std::vector<int>(prom.begin(), prom.begin() + np),
                                    QuantScheme{8, true, 128, false}, QuantScheme{4, false, 128, false});
    const QuantScheme act{8, true, 128, false};
    auto Y = execute_mixed_linear(A, L, act);
    CHECK(fnv1a_hex(Y.data(), size_t(Y.size()) * 4) == "d086f2794bbbd731");
    auto Aq = quantize_tensor<float>(A, act);
    auto Y2 = execute_mixed_on_codes(Aq, L);
    CHECK(Y2 == Y);
    // quantized_forward-style chain (analysis.cpp:64-75): linear -> ReLU -> linear
    MatrixRMf H = Y;
    for (Index i = 0; i < H.size(); ++i) H.data()[i] = std::max(H.data()[i], 0.0f);
    MatrixRMd W2(128, 256);
    for (Index i = 0; i < W2.size(); ++i) W2.data()[i] = std::cos(0.01 * double(i));
    auto L2 = partition_and_quantize(W2, {3, 77}, QuantScheme{8, true, 128, false}, QuantScheme{4, false, 128, false});
    auto Z = execute_mixed_linear(H, L2, act);
    CHECK(Z.rows() == 64 && Z.cols() == 128 && std::isfinite(Z(5, 7)));
    // errors before compute
    MatrixRMf An = A;
    An(3, 200) = INFINITY;
    try {
        execute_mixed_linear(An, L, act);
        CHECK(false);
    } catch (const DataError& e) {
        CHECK(std::string(e.what()).find("row 3, group 1") != std::string::npos);
    }
    CHECK(throws<UsageError>([&] { execute_mixed_linear(A, L, QuantScheme{4, false, 128, false}); }));
    CHECK(throws<UsageError>([&] { execute_mixed_on_codes(quantize_tensor<float>(A, QuantScheme{8, true, 64, false}), L); }));
}

int main(int argc, char** argv) {
    host_checks();
    if (argc > 1 && std::string(argv[1]) == "--gpu") gpu_checks();
    std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ok", g_fail);
    return g_fail ? 1 : 0;
}

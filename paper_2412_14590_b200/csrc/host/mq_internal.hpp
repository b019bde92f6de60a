// mq_internal.hpp — internal declarations shared by the host code and the
// kernel launchers of libmixllm_b200.so. Not part of the ABI.
#pragma once

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "mixllm/capi.h"

struct mq_host_layer_s {
    int64_t N = 0, K = 0;
    int group = 128;
    mq_scheme large{}, small{};
    std::vector<int32_t> map8, map4;
    std::vector<uint8_t> p8, z8, p4, z4;
    std::vector<float> s8, s4;
};

namespace mq {

extern thread_local std::string g_last_error;
mq_status fail(mq_status st, const std::string& msg);

inline int64_t num_groups(int64_t cols, int g) { return cols == 0 ? 0 : (cols + g - 1) / g; }
inline int64_t row_stride(int bits, int64_t cols) { return bits == 4 ? (cols + 1) / 2 : cols; }

void pack_nibbles_raw(const uint8_t* v, int64_t n, uint8_t* out);
int raw_code(const uint8_t* payload, int bits, int64_t cols, int64_t r, int64_t c);
mq_status validate_desc(const mq_layer_desc* d);
mq_status validate_maps(const mq_layer_desc* d);
mq_status check_scheme(const mq_scheme* s);
mq_status partition_maps(int64_t N, const int32_t* promoted, int64_t np, std::vector<int32_t>& map8,
                         std::vector<int32_t>& map4);
float round_scale_f16(float s);
// NCCL binding resolved at run time (mq_nccl.cpp)
mq_status nccl_check_comm(void* comm, int world, int rank);
mq_status nccl_all_gather(const void* send, void* recv, size_t count, int dtype, void* comm, cudaStream_t stream);

// proj/include/mixquant/rng.hpp:16-82 (SplitMix64 seeding, xoshiro256++,
// 53-bit uniforms, Box-Muller normals with a cached spare).
class Xoshiro {
  public:
    explicit Xoshiro(uint64_t seed) {
        for (auto& w : s_) {
            uint64_t z = (seed += 0x9E3779B97F4A7C15ULL);
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
            w = z ^ (z >> 31);
        }
    }
    uint64_t next() {
        const uint64_t out = rotl(s_[0] + s_[3], 23) + s_[0], t = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= t;
        s_[3] = rotl(s_[3], 45);
        return out;
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    int64_t uniform_int(int64_t lo, int64_t hi) {
        const auto span = static_cast<uint64_t>(hi - lo);
        return lo + static_cast<int64_t>((static_cast<unsigned __int128>(next()) * span) >> 64);
    }
    double normal() {
        if (spare_ok_) {
            spare_ok_ = false;
            return spare_;
        }
        const double u1 = static_cast<double>((next() >> 11) + 1) * 0x1.0p-53;
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1)), a = 2.0 * M_PI * u2;
        spare_ = r * std::sin(a);
        spare_ok_ = true;
        return r * std::cos(a);
    }

  private:
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    uint64_t s_[4];
    bool spare_ok_ = false;
    double spare_ = 0.0;
};

}  // namespace mq

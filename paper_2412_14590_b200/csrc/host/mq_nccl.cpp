// mq_nccl.cpp — the engine's NCCL binding, resolved at run time.
//
// libmixllm_b200.so does not link NCCL: a communicator is only meaningful to
// the NCCL build that created it, so the engine binds to the NCCL already
// loaded in the process (e.g. the one PyTorch's ProcessGroupNCCL uses, so a
// torch communicator from ProcessGroupNCCL._comm_ptr() can be passed in), and
// only otherwise loads libnccl.so.2. Types come from nccl.h (ABI-stable);
// functions from dlsym.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "mq_internal.hpp"

namespace mq {
namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = nullptr;
        if (dlsym(RTLD_DEFAULT, "ncclAllGather")) h = RTLD_DEFAULT;           // already global
        if (!h) h = dlopen("libnccl.so.2", RTLD_LAZY | RTLD_NOLOAD);          // already loaded (local)
        if (!h) h = dlopen("libnccl.so.2", RTLD_LAZY | RTLD_LOCAL);           // system NCCL
        if (!h) {
            a.why = "libnccl.so.2 is not loadable";
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
        a.comm_count = reinterpret_cast<decltype(a.comm_count)>(sym("ncclCommCount"));
        a.comm_user_rank = reinterpret_cast<decltype(a.comm_user_rank)>(sym("ncclCommUserRank"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(sym("ncclAllGather"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
        a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.comm_count && a.comm_user_rank &&
               a.all_gather && a.error_string;
        if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
    });
    return a;
}

mq_status nccl_fail(ncclResult_t r, const char* what) {
    return fail(MQ_CUDA, std::string(what) + ": " + api().error_string(r));
}

}  // namespace

mq_status nccl_check_comm(void* comm, int world, int rank) {
    NcclApi& a = api();
    if (!a.ok) return fail(MQ_CUDA, "NCCL unavailable: " + a.why);
    if (!comm) return fail(MQ_USAGE, "communicator is null");
    int n = 0, r = 0;
    if (ncclResult_t e = a.comm_count(static_cast<ncclComm_t>(comm), &n)) return nccl_fail(e, "ncclCommCount");
    if (ncclResult_t e = a.comm_user_rank(static_cast<ncclComm_t>(comm), &r)) return nccl_fail(e, "ncclCommUserRank");
    if (n != world || r != rank)
        return fail(MQ_USAGE, "communicator is rank " + std::to_string(r) + " of " + std::to_string(n) +
                                  ", the layer shard is rank " + std::to_string(rank) + " of " + std::to_string(world));
    return MQ_OK;
}

mq_status nccl_all_gather(const void* send, void* recv, size_t count, int dtype, void* comm, cudaStream_t stream) {
    const ncclDataType_t t = dtype == MQ_F32 ? ncclFloat32 : dtype == MQ_F16 ? ncclFloat16 : ncclBfloat16;
    if (ncclResult_t e = api().all_gather(send, recv, count, t, static_cast<ncclComm_t>(comm), stream))
        return nccl_fail(e, "ncclAllGather");
    return MQ_OK;
}

}  // namespace mq

using namespace mq;

extern "C" {

mq_status mq_nccl_unique_id(uint8_t* id) {
    NcclApi& a = api();
    if (!a.ok) return fail(MQ_CUDA, "NCCL unavailable: " + a.why);
    if (!id) return fail(MQ_USAGE, "id buffer is null");
    ncclUniqueId u;
    if (ncclResult_t e = a.get_unique_id(&u)) return nccl_fail(e, "ncclGetUniqueId");
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    return MQ_OK;
}

mq_status mq_nccl_comm_init(const uint8_t* id, int32_t world, int32_t rank, int device, void** comm) {
    NcclApi& a = api();
    if (!a.ok) return fail(MQ_CUDA, "NCCL unavailable: " + a.why);
    if (!id || !comm) return fail(MQ_USAGE, "null argument");
    if (world < 1 || rank < 0 || rank >= world) return fail(MQ_USAGE, "bad rank/world");
    if (cudaSetDevice(device) != cudaSuccess) return fail(MQ_CUDA, "bad device ordinal");
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t c = nullptr;
    if (ncclResult_t e = a.comm_init_rank(&c, world, u, rank)) return nccl_fail(e, "ncclCommInitRank");
    *comm = c;
    return MQ_OK;
}

mq_status mq_nccl_comm_destroy(void* comm) {
    NcclApi& a = api();
    if (!a.ok) return fail(MQ_CUDA, "NCCL unavailable: " + a.why);
    if (!comm) return MQ_OK;
    if (ncclResult_t e = a.comm_destroy(static_cast<ncclComm_t>(comm))) return nccl_fail(e, "ncclCommDestroy");
    return MQ_OK;
}

}  // extern "C"

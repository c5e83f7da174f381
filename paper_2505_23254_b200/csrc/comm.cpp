// NCCL inside the library: the cross-rank skip decision of the data-parallel
// step (SURVEY.md §8(b) C-ABI proposal `ma_init(device, ncclUniqueId*, rank,
// world)` / `ma_flag_allreduce_max`; north star: "a single NCCL
// all-reduce(max) over NVLink of the overflow flag so every rank makes the
// same skip-step decision").  The reference is single-process and makes ONE
// global decision over the whole flat buffer (proj/src/simulator.cpp:
// 431-440); across ranks that decision is the OR of the per-rank K1 flags,
// which ncclAllReduce(max) of the uint32 flag computes on the compute stream
// between K1 and K2 — no host round trip, capturable in a CUDA graph.
//
// libnccl.so.2 is resolved at run time (dlopen): when torch has already
// loaded its own NCCL the same library is reused (RTLD_NOLOAD first), a C++
// trainer without torch gets the system one, and a box without NCCL can
// still load this library (every other entry point works).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "memascend_b200.h"

namespace ma {
void set_error(const std::string& msg);
}

struct ma_comm {
    ncclComm_t comm = nullptr;
    int world = 1;
    int rank = 0;
};

namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                               ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    ncclResult_t (*get_version)(int*) = nullptr;
    std::string why;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            n.h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
            if (n.h) break;
        }
        for (const char* nm : names) {
            if (n.h) break;
            n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        }
        if (!n.h) {
            n.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return;
        }
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(n.h, "ncclGetUniqueId"));
        n.init_rank = reinterpret_cast<decltype(n.init_rank)>(dlsym(n.h, "ncclCommInitRank"));
        n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(n.h, "ncclCommDestroy"));
        n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(n.h, "ncclAllReduce"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(n.h, "ncclGetErrorString"));
        n.get_version = reinterpret_cast<decltype(n.get_version)>(dlsym(n.h, "ncclGetVersion"));
        if (!n.get_unique_id || !n.init_rank || !n.destroy || !n.all_reduce || !n.error_string)
            n.why = "libnccl.so.2 lacks a required symbol";
    });
    return n;
}

int nccl_fail(ncclResult_t r, const char* what) {
    ma::set_error(std::string(what) + ": " + nccl().error_string(r));
    return MA_ERR_NCCL;
}

int need_nccl() {
    Nccl& n = nccl();
    if (!n.why.empty()) {
        ma::set_error(n.why);
        return MA_ERR_NCCL;
    }
    return MA_OK;
}

}  // namespace

extern "C" {

int ma_comm_unique_id(void* id_out) {
    if (!id_out) {
        ma::set_error("null output");
        return MA_ERR_INVALID_ARGUMENT;
    }
    if (int e = need_nccl()) return e;
    static_assert(sizeof(ncclUniqueId) == MA_NCCL_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId id;
    if (ncclResult_t r = nccl().get_unique_id(&id)) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof id);
    return MA_OK;
}

int ma_comm_create(const void* nccl_unique_id, int world, int rank, ma_comm** out) {
    if (!nccl_unique_id || !out || world < 1 || rank < 0 || rank >= world) {
        ma::set_error("ma_comm_create: bad id / world / rank");
        return MA_ERR_INVALID_ARGUMENT;
    }
    if (int e = need_nccl()) return e;
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof id);
    auto* c = new ma_comm();
    c->world = world;
    c->rank = rank;
    if (ncclResult_t r = nccl().init_rank(&c->comm, world, id, rank)) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    *out = c;
    return MA_OK;
}

int ma_comm_destroy(ma_comm* c) {
    if (!c) return MA_OK;
    ncclResult_t r = ncclSuccess;
    if (c->comm) r = nccl().destroy(c->comm);
    delete c;
    return r ? nccl_fail(r, "ncclCommDestroy") : MA_OK;
}

int ma_comm_info(ma_comm* c, int* world, int* rank, int* nccl_version) {
    if (!c) {
        ma::set_error("null communicator");
        return MA_ERR_INVALID_ARGUMENT;
    }
    if (world) *world = c->world;
    if (rank) *rank = c->rank;
    if (nccl_version) {
        *nccl_version = 0;
        if (nccl().get_version) nccl().get_version(nccl_version);
    }
    return MA_OK;
}

int ma_comm_allreduce_max_u32(ma_comm* c, uint32_t* d_buf, uint64_t count, void* stream) {
    if (!c || (count && !d_buf)) {
        ma::set_error("null communicator / buffer");
        return MA_ERR_INVALID_ARGUMENT;
    }
    if (ncclResult_t r = nccl().all_reduce(d_buf, d_buf, count, ncclUint32, ncclMax, c->comm,
                                           static_cast<cudaStream_t>(stream)))
        return nccl_fail(r, "ncclAllReduce");
    return MA_OK;
}

int ma_stepper_allreduce_flag_async(ma_stepper* s, ma_comm* c, void* stream) {
    if (!s) {
        ma::set_error("null stepper");
        return MA_ERR_INVALID_ARGUMENT;
    }
    return ma_comm_allreduce_max_u32(c, ma_stepper_flag(s), 1, stream);
}

}  // extern "C"

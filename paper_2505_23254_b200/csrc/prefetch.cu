// Device-side adaptive pool (ma_dpool) and the weight prefetcher
// (ma_prefetcher): SURVEY.md §8(f) row 4.  See include/memascend_b200.h.
//
// Reference behaviour followed (/root/reference/proj):
//   slot planning: per shape class, payload rounded up to 4096 for the
//     stride, classes back to back in one backing region ... src/pool.cpp:22-68
//   class choice for a payload: the tightest class that fits .. src/pool.cpp:111-131
//   checkout blocks while the class is exhausted; stats ........ src/pool.cpp:133-188
//   prefetch/hold pipeline (prefetcher thread reads each tensor
//     into a pool slot, the consumer holds it, then checks in) .. src/simulator.cpp:367-425
// Here the pool lives in HBM and the pipeline ends in it: store -> registered
// host slot (store workers) -> device slot (copy stream) -> consumer stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "memascend_b200.h"
#include "swap.hpp"

namespace ma {
void set_error(const std::string& msg);  // capi.cu
}

namespace {

using ma::swp::fail;

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(e == cudaErrorMemoryAllocation ? MA_ERR_OUT_OF_MEMORY : MA_ERR_CUDA,
             std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define CKP(call) ck((call), #call)

template <typename F>
int guard(F&& fn) {
    try {
        fn();
        return MA_OK;
    } catch (const ma::swp::Failure& f) {
        ma::set_error(f.msg);
        return f.code;
    } catch (const std::bad_alloc&) {
        ma::set_error("host allocation failed");
        return MA_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        ma::set_error(e.what());
        return MA_ERR_DEVICE_ERROR;
    }
}

void need_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        fail(MA_ERR_NO_DEVICE, "no CUDA device visible: the memascend B200 path has no CPU fallback");
    }
}

constexpr uint64_t kAlign = 4096;
uint64_t align_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

}  // namespace

struct ma_dpool {
    struct Cls {
        uint64_t payload = 0, stride = 0, base = 0;
        uint32_t count = 0;
        std::vector<uint32_t> free;
    };
    std::vector<Cls> cls;
    char* d_base = nullptr;
    int device = 0;
    std::mutex mu;
    std::condition_variable cv;
    ma_dpool_stats st{};
    std::vector<uint64_t> live_len;        // per global slot id
    std::vector<cudaEvent_t> release_ev;   // per global slot id (reuse fence)
    std::vector<char> release_valid;
    std::vector<uint32_t> first_gid;       // per class

    ~ma_dpool() {
        for (cudaEvent_t e : release_ev)
            if (e) cudaEventDestroy(e);
        if (d_base) cudaFree(d_base);
    }

    // tightest class whose payload fits (pool.cpp:111-131)
    uint32_t class_for(uint64_t bytes) const {
        uint32_t best = UINT32_MAX;
        for (uint32_t c = 0; c < cls.size(); ++c)
            if (cls[c].payload >= bytes && (best == UINT32_MAX || cls[c].payload < cls[best].payload))
                best = c;
        if (best == UINT32_MAX)
            fail(MA_ERR_SIZE_VIOLATION,
                 "payload of " + std::to_string(bytes) + " bytes fits no device slot class");
        return best;
    }

    // Blocks while the class is exhausted (or until *stop).
    bool checkout(uint64_t bytes, const std::atomic<bool>* stop, uint32_t* gid, char** dptr) {
        const uint32_t c = class_for(bytes);
        std::unique_lock<std::mutex> lock(mu);
        cv.wait(lock, [&] { return !cls[c].free.empty() || (stop && *stop); });
        if (cls[c].free.empty()) return false;
        const uint32_t s = cls[c].free.back();
        cls[c].free.pop_back();
        *gid = first_gid[c] + s;
        *dptr = d_base + cls[c].base + static_cast<uint64_t>(s) * cls[c].stride;
        live_len[*gid] = bytes;
        st.live_bytes += bytes;
        st.peak_live_bytes = std::max(st.peak_live_bytes, st.live_bytes);
        st.checkout_count += 1;
        return true;
    }

    void checkin(uint32_t gid, cudaStream_t after) {
        std::lock_guard<std::mutex> lock(mu);
        if (!release_ev[gid]) CKP(cudaEventCreateWithFlags(&release_ev[gid], cudaEventDisableTiming));
        CKP(cudaEventRecord(release_ev[gid], after));
        release_valid[gid] = 1;
        uint32_t c = 0;
        while (c + 1 < cls.size() && first_gid[c + 1] <= gid) ++c;
        cls[c].free.push_back(gid - first_gid[c]);
        st.live_bytes -= live_len[gid];
        live_len[gid] = 0;
        st.checkin_count += 1;
        cv.notify_all();
    }

    // the copy into slot gid must follow the previous holder's work
    void fence(uint32_t gid, cudaStream_t copy) {
        std::lock_guard<std::mutex> lock(mu);
        if (release_valid[gid]) CKP(cudaStreamWaitEvent(copy, release_ev[gid], 0));
    }
};

struct ma_prefetcher {
    struct Item {
        std::string key;
        uint64_t bytes = 0;
        uint32_t gid = 0;
        char* dptr = nullptr;
        uint32_t hslot = 0;
        bool slotted = false;  // holds device slot gid
        ma::swp::Op* op = nullptr;
        cudaEvent_t ready = nullptr;
        int state = 0;  // 0 queued, 1 reading, 2 uploaded, 3 acquired
        int err = 0;
        std::string msg;
    };
    ma::swp::Engine* eng = nullptr;
    ma_dpool* pool = nullptr;
    char* hbase = nullptr;
    uint64_t hslot_bytes = 0;
    uint32_t hslots = 0;
    cudaStream_t copy = nullptr;
    int device = 0;

    std::mutex mu;
    std::condition_variable cv;
    std::deque<Item*> todo;
    std::deque<Item*> reading;
    std::unordered_map<std::string, std::unique_ptr<Item>> items;
    std::vector<int> hstate;  // 0 free, 1 being read / uploaded, 2 copy enqueued (hev)
    std::vector<cudaEvent_t> hev;
    std::atomic<bool> stop{false};
    std::thread reader, uploader;

    void set_err(Item* it, int code, const std::string& msg) {
        std::lock_guard<std::mutex> lock(mu);
        it->err = code;
        it->msg = msg;
        it->state = 2;
        cv.notify_all();
    }

    void reader_loop() {
        cudaSetDevice(device);
        for (;;) {
            Item* it = nullptr;
            {
                std::unique_lock<std::mutex> lock(mu);
                cv.wait(lock, [&] { return stop || !todo.empty(); });
                if (stop) return;
                it = todo.front();
                todo.pop_front();
            }
            int h = -1;
            try {
                const ma::swp::Location loc = eng->location(it->key);
                if (loc.padded > hslot_bytes)
                    fail(MA_ERR_SIZE_VIOLATION, "tensor '" + it->key + "' (" +
                                                    std::to_string(loc.padded) +
                                                    " padded bytes) exceeds a host slot");
                it->bytes = loc.logical;
                if (!pool->checkout(loc.logical, &stop, &it->gid, &it->dptr)) return;
                it->slotted = true;
                int hs = 0;
                {
                    std::unique_lock<std::mutex> lock(mu);
                    cv.wait(lock, [&] {
                        if (stop) return true;
                        for (uint32_t k = 0; k < hslots; ++k)
                            if (hstate[k] != 1) return true;
                        return false;
                    });
                    if (stop) return;
                    for (h = 0; hstate[h] == 1; ++h) {
                    }
                    hs = hstate[h];
                    hstate[h] = 1;
                }
                if (hs == 2) CKP(cudaEventSynchronize(hev[h]));  // last copy out of the slot done
                it->hslot = static_cast<uint32_t>(h);
                it->op = eng->submit_read(it->key, hbase + it->hslot * hslot_bytes, hslot_bytes);
                std::lock_guard<std::mutex> lock(mu);
                it->state = 1;
                reading.push_back(it);
                cv.notify_all();
            } catch (const ma::swp::Failure& f) {
                if (it->slotted) {
                    it->slotted = false;
                    try {
                        pool->checkin(it->gid, copy);
                    } catch (const ma::swp::Failure&) {
                    }
                }
                if (h >= 0) {
                    std::lock_guard<std::mutex> lock(mu);
                    hstate[h] = 0;
                }
                set_err(it, f.code, f.msg);
            }
        }
    }

    void uploader_loop() {
        cudaSetDevice(device);
        for (;;) {
            Item* it = nullptr;
            {
                std::unique_lock<std::mutex> lock(mu);
                cv.wait(lock, [&] { return !reading.empty() || stop; });
                if (reading.empty()) return;  // stopping and drained
                it = reading.front();
                reading.pop_front();
            }
            int code = 0;
            std::string msg;
            try {
                ma::swp::Op* op = it->op;
                it->op = nullptr;
                eng->wait(op);
                pool->fence(it->gid, copy);
                CKP(cudaMemcpyAsync(it->dptr, hbase + it->hslot * hslot_bytes, it->bytes,
                                    cudaMemcpyHostToDevice, copy));
                CKP(cudaEventCreateWithFlags(&it->ready, cudaEventDisableTiming));
                CKP(cudaEventRecord(it->ready, copy));
                CKP(cudaEventRecord(hev[it->hslot], copy));
            } catch (const ma::swp::Failure& f) {
                code = f.code;
                msg = f.msg;
            }
            if (code && it->slotted) {
                it->slotted = false;
                try {
                    pool->checkin(it->gid, copy);
                } catch (const ma::swp::Failure&) {
                }
            }
            std::lock_guard<std::mutex> lock(mu);
            hstate[it->hslot] = code ? 0 : 2;
            it->state = 2;
            it->err = code;
            it->msg = msg;
            cv.notify_all();
        }
    }
};

extern "C" {

int ma_dpool_create(const uint64_t* slot_payload_bytes, const uint32_t* slot_counts,
                    uint32_t nclasses, ma_dpool** out) {
    return guard([&] {
        if (!out || (nclasses && (!slot_payload_bytes || !slot_counts)) || nclasses == 0)
            fail(MA_ERR_INVALID_ARGUMENT, "device pool needs >= 1 slot class");
        need_device();
        std::unique_ptr<ma_dpool> p(new ma_dpool);
        CKP(cudaGetDevice(&p->device));
        uint64_t off = 0;
        uint32_t gid = 0;
        for (uint32_t c = 0; c < nclasses; ++c) {
            if (slot_payload_bytes[c] == 0 || slot_counts[c] == 0)
                fail(MA_ERR_INVALID_ARGUMENT, "slot classes need a payload and a count");
            ma_dpool::Cls k;
            k.payload = slot_payload_bytes[c];
            k.stride = align_up(k.payload, kAlign);
            k.count = slot_counts[c];
            k.base = off;
            for (uint32_t s = k.count; s > 0; --s) k.free.push_back(s - 1);
            off += k.stride * k.count;
            p->st.capacity_bytes += k.payload * k.count;
            p->first_gid.push_back(gid);
            gid += k.count;
            p->cls.push_back(std::move(k));
        }
        p->st.backing_bytes = off;
        p->live_len.assign(gid, 0);
        p->release_ev.assign(gid, nullptr);
        p->release_valid.assign(gid, 0);
        CKP(cudaMalloc(reinterpret_cast<void**>(&p->d_base), off));
        *out = p.release();
    });
}

int ma_dpool_destroy(ma_dpool* p) {
    return guard([&] { delete p; });
}

int ma_dpool_get_stats(ma_dpool* p, ma_dpool_stats* out) {
    return guard([&] {
        if (!p || !out) fail(MA_ERR_INVALID_ARGUMENT, "null argument");
        std::lock_guard<std::mutex> lock(p->mu);
        *out = p->st;
    });
}

int ma_prefetcher_create(ma_swap* store, ma_dpool* pool, void* h_staging, uint64_t h_slot_bytes,
                         uint32_t host_slots, ma_prefetcher** out) {
    return guard([&] {
        if (!store || !pool || !out) fail(MA_ERR_INVALID_ARGUMENT, "null argument");
        if (!h_staging || host_slots == 0 || h_slot_bytes == 0 || h_slot_bytes % kAlign)
            fail(MA_ERR_INVALID_ARGUMENT, "host staging needs slots of a 4096-multiple size");
        if (reinterpret_cast<uintptr_t>(h_staging) % kAlign)
            fail(MA_ERR_ALIGNMENT, "host staging must be 4096-aligned");
        need_device();
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, h_staging) != cudaSuccess ||
            at.type != cudaMemoryTypeHost) {
            cudaGetLastError();
            fail(MA_ERR_INVALID_ARGUMENT, "host staging must be registered host memory");
        }
        std::unique_ptr<ma_prefetcher> f(new ma_prefetcher);
        f->eng = store->e;
        f->pool = pool;
        f->hbase = static_cast<char*>(h_staging);
        f->hslot_bytes = h_slot_bytes;
        f->hslots = host_slots;
        f->device = pool->device;
        CKP(cudaSetDevice(f->device));
        CKP(cudaStreamCreateWithFlags(&f->copy, cudaStreamNonBlocking));
        f->hstate.assign(host_slots, 0);
        f->hev.assign(host_slots, nullptr);
        for (auto& e : f->hev) CKP(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ma_prefetcher* raw = f.get();
        f->reader = std::thread([raw] { raw->reader_loop(); });
        f->uploader = std::thread([raw] { raw->uploader_loop(); });
        *out = f.release();
    });
}

int ma_prefetch_submit(ma_prefetcher* f, const char* key) {
    return guard([&] {
        if (!f || !key) fail(MA_ERR_INVALID_ARGUMENT, "null argument");
        std::lock_guard<std::mutex> lock(f->mu);
        if (f->items.count(key))
            fail(MA_ERR_ALREADY_CHECKED_OUT, std::string("'") + key + "' is already in flight");
        std::unique_ptr<ma_prefetcher::Item> it(new ma_prefetcher::Item);
        it->key = key;
        f->todo.push_back(it.get());
        f->items.emplace(key, std::move(it));
        f->cv.notify_all();
    });
}

int ma_prefetch_acquire(ma_prefetcher* f, const char* key, void* stream, void** dptr,
                        uint64_t* bytes) {
    return guard([&] {
        if (!f || !key || !dptr) fail(MA_ERR_INVALID_ARGUMENT, "null argument");
        std::unique_lock<std::mutex> lock(f->mu);
        auto found = f->items.find(key);
        if (found == f->items.end())
            fail(MA_ERR_NOT_FOUND, std::string("'") + key + "' was never submitted");
        ma_prefetcher::Item* it = found->second.get();
        if (it->state == 3) fail(MA_ERR_ALREADY_CHECKED_OUT, std::string("'") + key + "' is already acquired");
        f->cv.wait(lock, [&] { return it->state >= 2; });
        if (it->err) {
            const int code = it->err;
            const std::string msg = it->msg;
            f->items.erase(found);
            fail(code, msg);
        }
        CKP(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), it->ready, 0));
        it->state = 3;
        *dptr = it->dptr;
        if (bytes) *bytes = it->bytes;
    });
}

int ma_prefetch_release(ma_prefetcher* f, const char* key, void* stream) {
    return guard([&] {
        if (!f || !key) fail(MA_ERR_INVALID_ARGUMENT, "null argument");
        std::unique_ptr<ma_prefetcher::Item> it;
        {
            std::lock_guard<std::mutex> lock(f->mu);
            auto found = f->items.find(key);
            if (found == f->items.end() || found->second->state != 3)
                fail(MA_ERR_LIFECYCLE, std::string("release of '") + key + "', which is not acquired");
            it = std::move(found->second);
            f->items.erase(found);
        }
        it->slotted = false;
        f->pool->checkin(it->gid, reinterpret_cast<cudaStream_t>(stream));
        if (it->ready) cudaEventDestroy(it->ready);
    });
}

int ma_prefetcher_destroy(ma_prefetcher* f) {
    return guard([&] {
        if (!f) return;
        {
            std::lock_guard<std::mutex> lock(f->mu);
            f->stop = true;
            f->cv.notify_all();
        }
        {
            std::lock_guard<std::mutex> lock(f->pool->mu);
            f->pool->cv.notify_all();  // a reader blocked on a device slot
        }
        f->reader.join();
        f->uploader.join();
        // items the consumer never released still hold device slots
        cudaStreamSynchronize(f->copy);
        for (auto& kv : f->items) {
            if (kv.second->op) {
                try {
                    f->eng->wait(kv.second->op);
                } catch (const ma::swp::Failure&) {
                }
            }
            if (kv.second->slotted) f->pool->checkin(kv.second->gid, f->copy);
            if (kv.second->ready) cudaEventDestroy(kv.second->ready);
        }
        for (cudaEvent_t e : f->hev) cudaEventDestroy(e);
        cudaStreamSynchronize(f->copy);
        cudaStreamDestroy(f->copy);
        delete f;
    });
}

}  // extern "C"

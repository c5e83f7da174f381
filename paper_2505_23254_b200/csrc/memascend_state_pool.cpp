// include/memascend/state_pool.h over the drop-in memascend::Pool: the
// streamed optimizer state of configs[3] lives in pool slots checked out of
// one registered, alignment-free backing region (pool.hpp / pool.cpp:75-222
// semantics: exact-fit classes, key ledger, checkout / span / device_span).
#include "memascend/state_pool.h"

#include <memory>
#include <string>
#include <vector>

#include "memascend/error.hpp"
#include "memascend/pool.hpp"
#include "memascend_b200.h"

struct memascend_state_pool {
    std::unique_ptr<memascend::Pool> pool;
    std::vector<memascend::BufferHandle> handles;  // group-major: p, m, v
    std::vector<std::uint64_t> elems;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return MA_OK;
    } catch (const memascend::Error& e) {
        g_err = e.what();
        return 1 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_err = e.what();
        return MA_ERR_INVALID_ARGUMENT;
    }
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* memascend_last_error(void) {
    return g_err.c_str();
}

__attribute__((visibility("default"))) int memascend_state_pool_create(
    uint64_t n_params, uint64_t subgroup, memascend_state_pool** out) {
    return guarded([&] {
        if (!out || n_params == 0 || subgroup == 0)
            memascend::raise(memascend::ErrorCode::invalid_argument, "state pool: bad arguments");
        auto sp = std::make_unique<memascend_state_pool>();
        std::vector<memascend::TensorDescriptor> inv;
        const char* names[3] = {"master", "m", "v"};
        for (std::uint64_t o = 0, k = 0; o < n_params; o += subgroup, ++k) {
            const std::uint64_t n = std::min(subgroup, n_params - o);
            sp->elems.push_back(n);
            for (const char* nm : names) {
                memascend::TensorDescriptor t;
                t.name = std::string(nm) + ".g" + std::to_string(k);
                t.rows = n;
                t.cols = 1;
                t.precision = memascend::Precision{memascend::PrecisionKind::fp32};
                t.role = memascend::TensorRole::embedding;  // a global (non per-layer) member
                inv.push_back(t);
            }
        }
        memascend::PoolConfig cfg;
        cfg.mode = memascend::PoolMode::adaptive;
        cfg.inflight_blocks = 1;
        sp->pool = std::make_unique<memascend::Pool>(inv, cfg);
        for (const auto& t : inv) sp->handles.push_back(sp->pool->checkout(t.name, 4 * t.rows));
        *out = sp.release();
    });
}

__attribute__((visibility("default"))) int memascend_state_pool_tensor(
    memascend_state_pool* p, uint64_t group, int which, void** host, void** device,
    uint64_t* elems) {
    return guarded([&] {
        if (!p || which < 0 || which > 2 || group >= p->elems.size())
            memascend::raise(memascend::ErrorCode::invalid_argument, "state pool: no such tensor");
        const auto& h = p->handles[3 * group + static_cast<std::uint64_t>(which)];
        if (host) *host = p->pool->span(h).data();
        if (device) *device = p->pool->device_span(h);
        if (elems) *elems = p->elems[group];
    });
}

__attribute__((visibility("default"))) int memascend_state_pool_stats(
    memascend_state_pool* p, uint64_t* capacity_bytes, uint64_t* backing_bytes,
    uint64_t* live_bytes, uint64_t* checkouts, uint64_t* classes) {
    return guarded([&] {
        if (!p) memascend::raise(memascend::ErrorCode::invalid_argument, "null state pool");
        const memascend::PoolStats s = p->pool->stats();
        if (capacity_bytes) *capacity_bytes = s.capacity_bytes;
        if (backing_bytes) *backing_bytes = s.backing_bytes;
        if (live_bytes) *live_bytes = s.live_bytes;
        if (checkouts) *checkouts = s.checkout_count;
        if (classes) *classes = p->pool->class_count();
    });
}

__attribute__((visibility("default"))) int memascend_state_pool_destroy(memascend_state_pool* p) {
    return guarded([&] {
        if (!p) return;
        for (const auto& h : p->handles) p->pool->checkin(h);
        delete p;
    });
}

}  // extern "C"

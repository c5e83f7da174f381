// B200 additions to the reference API (no reference header):
// the adaptive buffer pool placed in HBM and the layer-wise weight prefetcher
// that fills it from the swap store, over the C ABI (ma_dpool_*, ma_prefetch_*
// in include/memascend_b200.h).
//
// DevicePool plans its slot classes exactly as the reference's Pool does
// (proj/src/pool.cpp:22-68: adaptive = one class per tensor shape with
// global_members + members_per_layer x inflight_blocks slots; monolithic =
// one class of the largest tensor), so pool_capacity() of the same inventory
// equals stats().capacity_bytes.  WeightPrefetcher is the prefetch/hold
// pipeline of proj/src/simulator.cpp:367-425 ending in HBM: submit() keys in
// consumption order, acquire() makes a CUDA stream wait for a tensor's copy
// and returns its device address, release() returns the slot once that
// stream's work so far is done.  As with the reference's blocking pool, the
// pipeline is only as deep as the pool: a consumer must release a block's
// tensors before it acquires tensors more than `inflight_blocks` blocks
// ahead, otherwise acquire() waits for a slot that is never returned.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "memascend/direct_io.hpp"
#include "memascend/model.hpp"
#include "memascend/pool.hpp"

struct ma_dpool;
struct ma_prefetcher;

namespace memascend {

class DevicePool {
public:
    DevicePool(const std::vector<TensorDescriptor>& inventory, PoolMode mode,
               std::uint64_t inflight_blocks);
    ~DevicePool();
    DevicePool(const DevicePool&) = delete;
    DevicePool& operator=(const DevicePool&) = delete;

    /// capacity_bytes / backing_bytes / peak_live_bytes / live_bytes /
    /// checkout_count / checkin_count as Pool::stats() defines them.
    PoolStats stats() const;
    const std::vector<Pool::ClassInfo>& classes() const noexcept { return classes_; }
    ma_dpool* handle() const noexcept { return h_; }

private:
    ma_dpool* h_ = nullptr;
    std::vector<Pool::ClassInfo> classes_;
};

class WeightPrefetcher {
public:
    /// host_slots registered host slots of host_slot_bytes (rounded up to
    /// 4096) stage store reads on their way to the device slots.
    WeightPrefetcher(DirectIoEngine& store, DevicePool& pool, std::uint32_t host_slots,
                     std::uint64_t host_slot_bytes);
    ~WeightPrefetcher();
    WeightPrefetcher(const WeightPrefetcher&) = delete;
    WeightPrefetcher& operator=(const WeightPrefetcher&) = delete;

    void submit(const std::string& key);
    /// stream: a cudaStream_t (nullptr = legacy default stream).
    void* acquire(const std::string& key, void* stream, std::uint64_t* bytes = nullptr);
    void release(const std::string& key, void* stream);

private:
    ma_prefetcher* h_ = nullptr;
    PinnedRegion staging_;
};

}  // namespace memascend

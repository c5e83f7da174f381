// B200 addition to the reference API (no reference header): the device-resident
// step driver as a C++ class, for a C++ trainer such as the reference's
// run_training (proj/src/simulator.cpp:427-492) that wants the whole step —
// check, cross-rank decision, update, loss scaler — on the GPU without host
// round trips.  A thin RAII layer over ma_stepper_* (include/memascend_b200.h);
// every failure is a memascend::Error with the reference's ErrorCode.
//
//   memascend::StepDriver drv(hyper, LossScaler{}, ma_dtype::MA_DT_BF16, MA_DT_BF16);
//   memascend::Communicator comm(world, rank, id);       // multi-rank only (NCCL)
//   for (step ...) {
//       drv.check(d_grads, n, stream);                    // K1 -> device flag
//       drv.exchange(comm, stream);                        // ncclAllReduce(max) of the flag
//       drv.apply(groups, stream);                          // K2, skipped on the flag
//       // or drv.apply_swapped(engine, swap_groups, staging, stream)  (state on NVMe)
//       drv.finish(stream);                                 // LossScaler on the device
//   }
//   LossScaler s = drv.scaler();                            // synchronises
//
// A restored run continues bit-exactly: StepDriver(hyper, saved_scaler, ...,
// saved_step_t) — or drv.resume(scaler, step_t) — sets the device state to the
// saved LossScaler and OptimizerState::step_t (optimizer.hpp:19-35,60-66).
// The per-step chain can be captured once into a CUDA graph (capture_begin /
// capture_end, StepGraph::launch) and replayed with one launch per step.
#pragma once

#include <array>
#include <cstdint>
#include <span>

#include "memascend/direct_io.hpp"
#include "memascend/optimizer.hpp"
#include "memascend_b200.h"

namespace memascend {

/// Registered host slots + device slots for StepDriver::apply_swapped.
struct SwapStaging {
    void* host = nullptr;        // registered, 4096-aligned: host_slots x 3 x align4096(4 x slot_elems)
    std::uint32_t host_slots = 0;
    float* device = nullptr;     // dev_slots x 3 x slot_elems floats
    std::uint32_t dev_slots = 0;
    std::uint64_t slot_elems = 0;
    void* h2d_stream = nullptr;  // copy streams (cudaStream_t)
    void* d2h_stream = nullptr;
};

/// NCCL communicator of the data-parallel group (ma_comm_*).  Rank 0 calls
/// unique_id() and distributes the bytes over any host channel.
class Communicator {
public:
    static std::array<unsigned char, MA_NCCL_ID_BYTES> unique_id();
    Communicator(int world, int rank, const std::array<unsigned char, MA_NCCL_ID_BYTES>& id);
    ~Communicator();
    Communicator(const Communicator&) = delete;
    Communicator& operator=(const Communicator&) = delete;
    int world() const noexcept { return world_; }
    int rank() const noexcept { return rank_; }
    ma_comm* handle() const noexcept { return h_; }

private:
    ma_comm* h_ = nullptr;
    int world_ = 1, rank_ = 0;
};

/// A captured step chain (ma_graph): launch() replays it with one launch.
class StepGraph {
public:
    explicit StepGraph(ma_graph* g) noexcept : g_(g) {}
    ~StepGraph();
    StepGraph(StepGraph&& o) noexcept : g_(o.g_) { o.g_ = nullptr; }
    StepGraph(const StepGraph&) = delete;
    StepGraph& operator=(const StepGraph&) = delete;
    void launch(void* stream);

private:
    ma_graph* g_ = nullptr;
};

class StepDriver {
public:
    /// `scaler` may be a restored LossScaler (any clean_steps) and
    /// `step_t` the restored OptimizerState::step_t (applied updates).
    StepDriver(const AdamHyper& hyper, const LossScaler& scaler, int grad_dtype,
               int working_dtype, std::uint64_t step_t = 0);
    ~StepDriver();
    StepDriver(const StepDriver&) = delete;
    StepDriver& operator=(const StepDriver&) = delete;

    /// K1 over a gradient buffer of the driver's gradient kind (device memory).
    void check(const void* grads, std::uint64_t n, void* stream);
    /// Device uint32 holding this step's overflow flag (all-reduce it MAX
    /// across ranks before apply).
    std::uint32_t* flag() const;
    /// K2 over HBM-resident sub-groups; a no-op on the device when flagged.
    void apply(std::span<const ma_subgroup> groups, void* stream);
    /// configs[4]: state in the swap store (keys) or the registered DRAM tier;
    /// returns true when the step was skipped (nothing read or written).
    bool apply_swapped(DirectIoEngine& store, std::span<const ma_swap_group> groups,
                       const SwapStaging& staging, void* stream);
    /// LossScaler::on_overflow / on_clean_step and the update counter, on the device.
    void finish(void* stream);
    /// Multi-rank: the step's single global skip decision (simulator.cpp:
    /// 431-440) as ncclAllReduce(max) of flag() on `stream`, between check and apply.
    void exchange(Communicator& comm, void* stream);
    /// Restore a saved LossScaler and Adam step count (synchronous).
    void resume(const LossScaler& scaler, std::uint64_t step_t);
    /// CUDA-graph capture of the *_async calls issued on `stream` (a
    /// non-default stream) between the two calls; nothing executes until
    /// StepGraph::launch.  `reserve_steps` bounds how many replays the graph's
    /// bias-correction table covers.
    void capture_begin(void* stream, std::uint64_t reserve_steps = 1u << 20);
    StepGraph capture_end(void* stream);

    /// Synchronises with the last stream used and returns the scaler state.
    LossScaler scaler() const;
    /// Applied updates (the Adam t of the last update).
    std::uint64_t updates() const;

    ma_stepper* handle() const noexcept { return h_; }

private:
    ma_stepper* h_ = nullptr;
};

}  // namespace memascend

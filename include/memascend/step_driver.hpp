// B200 addition to the reference API (no reference header): the device-resident
// step driver as a C++ class, for a C++ trainer such as the reference's
// run_training (proj/src/simulator.cpp:427-492) that wants the whole step —
// check, cross-rank decision, update, loss scaler — on the GPU without host
// round trips.  A thin RAII layer over ma_stepper_* (include/memascend_b200.h);
// every failure is a memascend::Error with the reference's ErrorCode.
//
//   memascend::StepDriver drv(hyper, LossScaler{}, ma_dtype::MA_DT_BF16, MA_DT_BF16);
//   for (step ...) {
//       drv.check(d_grads, n, stream);                    // K1 -> device flag
//       // multi-rank: ncclAllReduce(drv.flag(), ..., ncclMax, ...)
//       drv.apply(groups, stream);                          // K2, skipped on the flag
//       // or drv.apply_swapped(engine, swap_groups, staging, stream)  (state on NVMe)
//       drv.finish(stream);                                 // LossScaler on the device
//   }
//   LossScaler s = drv.scaler();                            // synchronises
#pragma once

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

class StepDriver {
public:
    StepDriver(const AdamHyper& hyper, const LossScaler& scaler, int grad_dtype,
               int working_dtype);
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

    /// Synchronises with the last stream used and returns the scaler state.
    LossScaler scaler() const;
    /// Applied updates (the Adam t of the last update).
    std::uint64_t updates() const;

    ma_stepper* handle() const noexcept { return h_; }

private:
    ma_stepper* h_ = nullptr;
};

}  // namespace memascend

// memascend::StepDriver (include/memascend/step_driver.hpp) over ma_stepper_*.
// The composition it drives is simulator.cpp:427-492 (check -> skip or
// update -> LossScaler), with the scaler and t kept on the device.
#include "memascend/step_driver.hpp"

#include "memascend/error.hpp"

namespace memascend {

namespace {

void check_status(int status) {
    if (status == MA_OK) return;
    const std::string msg = ma_last_error();
    if (status >= 1 && status <= 17) raise(static_cast<ErrorCode>(status - 1), msg);
    raise(ErrorCode::device_error, msg);
}

}  // namespace

StepDriver::StepDriver(const AdamHyper& hyper, const LossScaler& scaler, int grad_dtype,
                       int working_dtype) {
    if (scaler.clean_steps != 0)
        raise(ErrorCode::invalid_argument,
              "StepDriver starts a fresh LossScaler (clean_steps must be 0)");
    const ma_adam_hyper h{hyper.lr, hyper.beta1, hyper.beta2, hyper.eps, hyper.weight_decay};
    check_status(ma_stepper_create(&h, scaler.scale, scaler.growth_interval, grad_dtype, working_dtype,
                            nullptr, &h_));
}

StepDriver::~StepDriver() {
    if (h_) ma_stepper_destroy(h_);
}

void StepDriver::check(const void* grads, std::uint64_t n, void* stream) {
    check_status(ma_stepper_check_async(h_, grads, n, stream));
}

std::uint32_t* StepDriver::flag() const { return ma_stepper_flag(h_); }

void StepDriver::apply(std::span<const ma_subgroup> groups, void* stream) {
    check_status(ma_stepper_apply_async(h_, groups.data(),
                                            static_cast<uint32_t>(groups.size()), stream));
}

bool StepDriver::apply_swapped(DirectIoEngine& store, std::span<const ma_swap_group> groups,
                               const SwapStaging& st, void* stream) {
    int skipped = 0;
    check_status(ma_stepper_apply_swapped(
        h_, store.handle(), groups.data(), static_cast<uint32_t>(groups.size()), st.host,
        st.host_slots, st.device, st.dev_slots, st.slot_elems, stream, st.h2d_stream,
        st.d2h_stream, &skipped));
    return skipped != 0;
}

void StepDriver::finish(void* stream) { check_status(ma_stepper_finish_async(h_, stream)); }

LossScaler StepDriver::scaler() const {
    ma_step_state s{};
    check_status(ma_stepper_state(h_, &s));
    LossScaler out;
    out.scale = s.scale;
    out.growth_interval = s.growth_interval;
    out.clean_steps = s.clean_steps;
    return out;
}

std::uint64_t StepDriver::updates() const {
    ma_step_state s{};
    check_status(ma_stepper_state(h_, &s));
    return s.updates;
}

}  // namespace memascend

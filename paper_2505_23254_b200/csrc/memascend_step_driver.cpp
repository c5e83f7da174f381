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
                       int working_dtype, std::uint64_t step_t) {
    const ma_adam_hyper h{hyper.lr, hyper.beta1, hyper.beta2, hyper.eps, hyper.weight_decay};
    check_status(ma_stepper_create(&h, scaler.scale, scaler.growth_interval, grad_dtype,
                                   working_dtype, nullptr, &h_));
    if (scaler.clean_steps != 0 || step_t != 0) {
        const int st = ma_stepper_set_state(h_, scaler.scale, scaler.clean_steps, step_t);
        if (st != MA_OK) {
            ma_stepper_destroy(h_);
            h_ = nullptr;
            check_status(st);
        }
    }
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

void StepDriver::exchange(Communicator& comm, void* stream) {
    check_status(ma_stepper_allreduce_flag_async(h_, comm.handle(), stream));
}

void StepDriver::resume(const LossScaler& scaler, std::uint64_t step_t) {
    check_status(ma_stepper_set_state(h_, scaler.scale, scaler.clean_steps, step_t));
}

void StepDriver::capture_begin(void* stream, std::uint64_t reserve_steps) {
    check_status(ma_stepper_graph_begin(h_, reserve_steps, stream));
}

StepGraph StepDriver::capture_end(void* stream) {
    ma_graph* g = nullptr;
    check_status(ma_stepper_graph_end(h_, stream, &g));
    return StepGraph(g);
}

StepGraph::~StepGraph() {
    if (g_) ma_graph_destroy(g_);
}

void StepGraph::launch(void* stream) { check_status(ma_graph_launch(g_, stream)); }

std::array<unsigned char, MA_NCCL_ID_BYTES> Communicator::unique_id() {
    std::array<unsigned char, MA_NCCL_ID_BYTES> id{};
    check_status(ma_comm_unique_id(id.data()));
    return id;
}

Communicator::Communicator(int world, int rank,
                           const std::array<unsigned char, MA_NCCL_ID_BYTES>& id)
    : world_(world), rank_(rank) {
    check_status(ma_comm_create(id.data(), world, rank, &h_));
}

Communicator::~Communicator() {
    if (h_) ma_comm_destroy(h_);
}

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

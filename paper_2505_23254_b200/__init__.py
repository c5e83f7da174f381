"""B200-native MemAscend optimizer hot path (arXiv 2505.23254).

Fused overflow check (K1) + unscale/AdamW/cast-back (K2) + device-resident
loss scaler, as sm_100a CUDA kernels behind the C ABI in
include/memascend_b200.h (libmemascend_b200.so) and the drop-in C++ API in
include/memascend/*.hpp.  This Python package is a ctypes binding used by the
tests and bench; it never computes anything itself.
"""
from .capi import LIB_PATH, AdamHyper, MemAscendError, lib  # noqa: F401
from .api import (  # noqa: F401
    DevicePool,
    DirectIoEngine,
    NcclComm,
    StatePool,
    StepGraph,
    WeightPrefetcher,
    aligned_host_buffer,
    uring_available,
    OptimizerState,
    OverflowResult,
    Stepper,
    adam_step,
    adam_step_bf16,
    adam_step_fp32,
    adam_step_fp32_async,
    device_info,
    fused_overflow_check,
    gen_pseudo_grads,
    gen_seeded_weights,
    host_register,
    host_unregister,
    overflow_check_async,
    plant_bits,
    pointer_kind,
    torch_broadcast_bytes,
)

"""ctypes binding of the C ABI in include/memascend_b200.h.

This is the same binding a maintainer would add on the reference side
(INTEGRATION.md): plain pointers and sizes.  It loads the in-tree
``paper_2505_23254_b200/lib/libmemascend_b200.so`` and fails loudly when the
library is missing — there is no Python or CPU fallback for any compute entry
point.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libmemascend_b200.so")
if os.environ.get("MA_LIB_PATH"):  # A/B builds of the same C ABI (tools/, never by default)
    LIB_PATH = os.environ["MA_LIB_PATH"]

# status codes: 1 + memascend::ErrorCode (proj/include/memascend/error.hpp:9-27)
ERROR_NAMES = {
    1: "invalid-argument", 2: "out-of-memory", 3: "overflow", 4: "lifecycle",
    5: "unknown-region", 6: "pool-exhausted", 7: "size-violation", 8: "already-checked-out",
    9: "not-found", 10: "storage-full", 11: "device-error", 12: "capability", 13: "io-error",
    14: "alignment", 15: "busy", 16: "uncalibrated", 17: "bad-config",
    100: "cuda-error", 101: "no-device", 102: "nccl-error",
}

DT_F32, DT_BF16, DT_F16, DT_NONE = 0, 1, 2, 3
STEPPER_STATE_BYTES = 64
IPC_HANDLE_BYTES = 64
RS_HANDLE_BYTES = 192
NCCL_ID_BYTES = 128
DTYPES = {"f32": DT_F32, "bf16": DT_BF16, "f16": DT_F16, "none": DT_NONE}


class MemAscendError(RuntimeError):
    """memascend::Error equivalent: carries the reference ErrorCode name."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = ERROR_NAMES.get(status, f"status-{status}")
        super().__init__(f"{self.code}: {message}")


class AdamHyper(C.Structure):
    """AdamHyper, proj/include/memascend/optimizer.hpp:9-15 (same defaults)."""

    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float), ("weight_decay", C.c_float)]

    def __init__(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0):
        super().__init__(lr, beta1, beta2, eps, weight_decay)


class Subgroup(C.Structure):
    _fields_ = [("p", C.c_void_p), ("m", C.c_void_p), ("v", C.c_void_p), ("g", C.c_void_p),
                ("w", C.c_void_p), ("n", C.c_uint64)]


class SubgroupBf16(C.Structure):
    _fields_ = [("p", C.c_void_p), ("m", C.c_void_p), ("v", C.c_void_p), ("g", C.c_void_p),
                ("n", C.c_uint64)]


class StepState(C.Structure):
    _fields_ = [("scale", C.c_float), ("clean_steps", C.c_uint32), ("updates", C.c_uint64),
                ("steps", C.c_uint64), ("last_overflow", C.c_uint32),
                ("growth_interval", C.c_uint32)]


class SwapDevice(C.Structure):
    _fields_ = [("path", C.c_char_p), ("capacity_bytes", C.c_uint64), ("kind", C.c_int)]


class SwapConfig(C.Structure):
    _fields_ = [("workers", C.c_uint32), ("queue_depth", C.c_uint32), ("backend", C.c_int),
                ("cache_bypass", C.c_int), ("manifest_path", C.c_char_p)]


class SwapExtent(C.Structure):
    _fields_ = [("device_index", C.c_uint32), ("device_offset", C.c_uint64),
                ("length", C.c_uint64)]


class SwapStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("bytes_written", "bytes_read", "write_requests",
                                          "read_requests", "submitted_ios", "abandoned_bytes")]


class SwapGroup(C.Structure):
    _fields_ = [("key_p", C.c_char_p), ("key_m", C.c_char_p), ("key_v", C.c_char_p),
                ("p", C.c_void_p), ("m", C.c_void_p), ("v", C.c_void_p), ("g", C.c_void_p),
                ("w", C.c_void_p), ("n", C.c_uint64)]


class DPoolStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("capacity_bytes", "backing_bytes", "peak_live_bytes",
                                          "live_bytes", "checkout_count", "checkin_count")]


class SwapGroupBf16(C.Structure):
    _fields_ = [("key_m", C.c_char_p), ("key_v", C.c_char_p), ("m", C.c_void_p),
                ("v", C.c_void_p), ("p", C.c_void_p), ("g", C.c_void_p), ("n", C.c_uint64)]


IO_AUTO, IO_SYNC, IO_POSIX_AIO, IO_URING = 0, 1, 2, 3
IO_BACKENDS = {"auto": IO_AUTO, "sync": IO_SYNC, "aio": IO_POSIX_AIO, "uring": IO_URING}
IO_TRACE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int)

# (name, restype, argtypes) for every symbol the header declares
_VP, _U64, _I, _U32, _F = C.c_void_p, C.c_uint64, C.c_int, C.c_uint32, C.c_float
SIGNATURES = [
    ("ma_last_error", C.c_char_p, []),
    ("ma_abi_version", _I, []),
    ("ma_device_info", _I, [C.POINTER(_I)] * 4),
    ("ma_overflow_check_async", _I, [_VP, _U64, _I, _VP, _VP, _VP]),
    ("ma_overflow_check", _I, [_VP, _U64, _I, _I, C.POINTER(_I), C.POINTER(_U64)]),
    ("ma_adam_step_async", _I, [_VP, _VP, _VP, _VP, _I, _U64, _U64, C.POINTER(AdamHyper), _F,
                                _VP, _I, _VP, _VP]),
    ("ma_adam_step", _I, [_VP, _VP, _VP, _VP, _I, _U64, _U64, C.POINTER(AdamHyper), _F, _VP,
                          _I]),
    ("ma_adam_step_bf16", _I, [_VP, _VP, _VP, _VP, _U64, _U64, C.POINTER(AdamHyper), _F]),
    ("ma_stepper_create", _I, [C.POINTER(AdamHyper), _F, _U32, _I, _I, _VP, C.POINTER(_VP)]),
    ("ma_stepper_destroy", _I, [_VP]),
    ("ma_stepper_check_async", _I, [_VP, _VP, _U64, _VP]),
    ("ma_stepper_check_host_async", _I, [_VP, _VP, _VP, _U64, _U64, _VP, _VP]),
    ("ma_stepper_check_host_spec_async", _I, [_VP, _VP, _VP, _U64, _U64, _VP, _U32, _VP, _U64,
                                              _VP, _VP]),
    ("ma_stepper_apply_spec_async", _I, [_VP, _VP, _U32, _VP]),
    ("ma_stepper_check_host_spec_bf16_async", _I, [_VP, _VP, _VP, _U64, _U64, _VP, _U32, _VP,
                                                   _U64, _VP, _VP]),
    ("ma_stepper_apply_spec_bf16_async", _I, [_VP, _VP, _U32, _VP]),
    ("ma_xchg_create", _I, [_I, _I, C.POINTER(_VP), _VP]),
    ("ma_xchg_open", _I, [_VP, _VP]),
    ("ma_xchg_error", _I, [_VP, C.POINTER(_I)]),
    ("ma_xchg_destroy", _I, [_VP]),
    ("ma_stepper_check_xchg_async", _I, [_VP, _VP, _U64, _VP, _VP]),
    ("ma_stepper_ingest_async", _I, [_VP, _VP, _I, _VP, _U64, _VP]),
    ("ma_stepper_reduce_check_async", _I, [_VP, _VP, _I, _I, _U64, _F, _VP, _VP]),
    ("ma_rs_create", _I, [_I, _I, _VP, _U64, _I, C.POINTER(_VP), _VP]),
    ("ma_rs_open", _I, [_VP, _VP]),
    ("ma_rs_error", _I, [_VP, C.POINTER(_I)]),
    ("ma_rs_destroy", _I, [_VP]),
    ("ma_stepper_reduce_scatter_async", _I, [_VP, _VP, _U64, _U64, _F, _VP, _VP]),
    ("ma_stepper_apply_allgather_async", _I, [_VP, C.POINTER(Subgroup), _U32, _VP, _VP]),
    ("ma_stepper_flag", _VP, [_VP]),
    ("ma_stepper_scale", _VP, [_VP]),
    ("ma_stepper_apply_async", _I, [_VP, C.POINTER(Subgroup), _U32, _VP]),
    ("ma_stepper_apply_bf16_async", _I, [_VP, C.POINTER(SubgroupBf16), _U32, _VP]),
    ("ma_stepper_apply_streamed", _I, [_VP, C.POINTER(Subgroup), _U32, _VP, _U64, _U32, _VP,
                                       _VP, _VP, C.POINTER(_I)]),
    ("ma_stepper_finish_async", _I, [_VP, _VP]),
    ("ma_stepper_state", _I, [_VP, C.POINTER(StepState)]),
    ("ma_stepper_history", _I, [_VP, _VP, _VP, _U64, C.POINTER(_U64)]),
    ("ma_stepper_set_state", _I, [_VP, _F, _U32, _U64]),
    ("ma_stepper_graph_begin", _I, [_VP, _U64, _VP]),
    ("ma_stepper_graph_end", _I, [_VP, _VP, C.POINTER(_VP)]),
    ("ma_graph_launch", _I, [_VP, _VP]),
    ("ma_graph_destroy", _I, [_VP]),
    ("ma_comm_unique_id", _I, [_VP]),
    ("ma_comm_create", _I, [_VP, _I, _I, C.POINTER(_VP)]),
    ("ma_comm_destroy", _I, [_VP]),
    ("ma_comm_info", _I, [_VP, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
    ("ma_comm_allreduce_max_u32", _I, [_VP, _VP, _U64, _VP]),
    ("ma_stepper_allreduce_flag_async", _I, [_VP, _VP, _VP]),
    ("ma_gen_seeded_weights_async", _I, [_VP, _VP, _I, _U64, _U64, _U64, _VP]),
    ("ma_gen_pseudo_grads_async", _I, [_VP, _I, _VP, _I, _U64, _U64, _U64, _U64, _VP, _F, _VP]),
    ("ma_plant_bits_async", _I, [_VP, _I, _U64, _U32, _VP]),
    ("ma_swap_create", _I, [C.POINTER(SwapDevice), _U32, C.POINTER(SwapConfig), C.POINTER(_VP)]),
    ("ma_swap_destroy", _I, [_VP]),
    ("ma_swap_allocate", _I, [_VP, C.c_char_p, _U64, C.POINTER(SwapExtent), _U32,
                              C.POINTER(_U32)]),
    ("ma_swap_write", _I, [_VP, C.c_char_p, _VP, _U64, _U64]),
    ("ma_swap_read", _I, [_VP, C.c_char_p, _VP, _U64, C.POINTER(_U64)]),
    ("ma_swap_write_async", _I, [_VP, C.c_char_p, _VP, _U64, _U64, C.POINTER(_VP)]),
    ("ma_swap_read_async", _I, [_VP, C.c_char_p, _VP, _U64, C.POINTER(_VP)]),
    ("ma_swap_wait", _I, [_VP, C.POINTER(_U64)]),
    ("ma_swap_contains", _I, [_VP, C.c_char_p, C.POINTER(_I)]),
    ("ma_swap_location", _I, [_VP, C.c_char_p, C.POINTER(_U64), C.POINTER(_U64),
                              C.POINTER(SwapExtent), _U32, C.POINTER(_U32)]),
    ("ma_swap_keys", _I, [_VP, _VP, _U64, C.POINTER(_U64)]),
    ("ma_swap_get_stats", _I, [_VP, C.POINTER(SwapStats)]),
    ("ma_swap_info", _I, [_VP, C.POINTER(_I), C.POINTER(_U64), C.POINTER(_U32)]),
    ("ma_swap_set_trace", _I, [_VP, IO_TRACE_FN, _VP]),
    ("ma_swap_save_manifest", _I, [_VP]),
    ("ma_swap_create_virtual_devices", _I, [C.c_char_p, _U32, _U64]),
    ("ma_swap_uring_available", _I, []),
    ("ma_cursor_open", _I, [_U32, C.c_char_p, C.POINTER(_VP)]),
    ("ma_cursor_close", _I, [_VP]),
    ("ma_cursor_advance", _I, [_VP, _U32, _U64, C.POINTER(_U64)]),
    ("ma_cursor_position", _I, [_VP, _U32, C.POINTER(_U64)]),
    ("ma_cursor_restore", _I, [_VP, _U32, _U64]),
    ("ma_stepper_apply_swapped", _I, [_VP, _VP, C.POINTER(SwapGroup), _U32, _VP, _U32, _VP, _U32,
                                      _U64, _VP, _VP, _VP, C.POINTER(_I)]),
    ("ma_dpool_create", _I, [_VP, _VP, _U32, C.POINTER(_VP)]),
    ("ma_dpool_destroy", _I, [_VP]),
    ("ma_dpool_get_stats", _I, [_VP, C.POINTER(DPoolStats)]),
    ("ma_prefetcher_create", _I, [_VP, _VP, _VP, _U64, _U32, C.POINTER(_VP)]),
    ("ma_prefetch_submit", _I, [_VP, C.c_char_p]),
    ("ma_prefetch_acquire", _I, [_VP, C.c_char_p, _VP, C.POINTER(_VP), C.POINTER(_U64)]),
    ("ma_prefetch_release", _I, [_VP, C.c_char_p, _VP]),
    ("ma_prefetcher_destroy", _I, [_VP]),
    ("ma_stepper_apply_swapped_bf16", _I, [_VP, _VP, C.POINTER(SwapGroupBf16), _U32, _VP, _U32,
                                           _VP, _U32, _U64, _VP, _VP, _VP, C.POINTER(_I)]),
    ("ma_host_register", _I, [_VP, _U64]),
    ("ma_host_unregister", _I, [_VP]),
    ("ma_pointer_kind", _I, [_VP, C.POINTER(_I)]),
    ("ma_device_numa_node", _I, [C.POINTER(_I)]),
    ("ma_host_place", _I, [_VP, _U64]),
    ("ma_host_numa_node", _I, [_VP, C.POINTER(_I)]),
    ("ma_debug_cast_sweep", _I, [_I, _I, _VP]),
    ("ma_debug_mask_sweep", _I, [_I, C.POINTER(_U64)]),
    ("ma_debug_fast_sweep", _I, [_I, _VP, _U32, _U64, _U64, C.POINTER(_U64), C.POINTER(_U64)]),
]

_lib = None


def lib():
    """The loaded C ABI library (raises ImportError if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            if os.environ.get("MA_LIB_PATH") and not hasattr(L, name):
                continue  # an older A/B build may predate a symbol
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        raise MemAscendError(status, lib().ma_last_error().decode(errors="replace"))

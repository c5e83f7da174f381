"""Python mirror of the reference hot-path interface over the C ABI.

Names, argument meaning and error behaviour follow the reference's C++ API
(proj/include/memascend/{overflow,optimizer}.hpp) so tests read like the
reference's own tests; tensors are torch tensors (device or host) or numpy
arrays (host).  Everything computes in libmemascend_b200.so on the GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import capi
from .capi import AdamHyper, MemAscendError, check  # noqa: F401  (re-exported)

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None

_TORCH_DT = {}
if torch is not None:
    _TORCH_DT = {torch.float32: capi.DT_F32, torch.bfloat16: capi.DT_BF16,
                 torch.float16: capi.DT_F16}
_NP_DT = {np.dtype(np.float32): capi.DT_F32, np.dtype(np.float16): capi.DT_F16}


def _info(x, kind=None):
    """(pointer, element count, dtype code) of a tensor / array / None."""
    if x is None:
        return None, 0, capi.DT_NONE
    if torch is not None and isinstance(x, torch.Tensor):
        if not x.is_contiguous():
            raise MemAscendError(1, "tensor must be contiguous")
        dt = capi.DTYPES[kind] if kind else _TORCH_DT.get(x.dtype)
        if dt is None:
            raise MemAscendError(1, f"unsupported dtype {x.dtype} (pass kind=)")
        return x.data_ptr(), x.numel(), dt
    a = x
    if not a.flags["C_CONTIGUOUS"]:
        raise MemAscendError(1, "array must be C-contiguous")
    dt = capi.DTYPES[kind] if kind else _NP_DT.get(a.dtype)
    if dt is None:
        raise MemAscendError(1, f"unsupported dtype {a.dtype} (pass kind=)")
    return a.ctypes.data, a.size, dt


def _kind_ok(x, kind):
    """x holds elements of `kind`: the matching torch dtype, or a raw-bits view
    of the same width (int32 for f32, int16 for the 16-bit kinds)."""
    if torch is None or not isinstance(x, torch.Tensor):
        return True
    code = _TORCH_DT.get(x.dtype)
    if code is not None:
        return code == capi.DTYPES[kind]
    return x.element_size() == (4 if kind == "f32" else 2) and not x.is_floating_point()


def _stream_ptr(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream if torch is not None else None
    return stream if isinstance(stream, int) else stream.cuda_stream


# ----------------------------------------------------------------- K1
@dataclass
class OverflowResult:
    """overflow.hpp:41-44"""

    overflow: bool = False
    first_offending_index: int | None = None


def fused_overflow_check(values, track_first_index: bool = False, kind: str | None = None):
    """overflow.hpp:56-62 / overflow.cpp:73-145 on the GPU (K1)."""
    ptr, n, dt = _info(values, kind)
    of, first = C.c_int(), C.c_uint64()
    check(capi.lib().ma_overflow_check(ptr, n, dt, int(track_first_index), C.byref(of),
                                       C.byref(first)))
    res = OverflowResult(bool(of.value))
    if track_first_index and of.value:
        res.first_offending_index = first.value
    return res


def overflow_check_async(values, d_flag, d_first=None, kind=None, stream=None):
    ptr, n, dt = _info(values, kind)
    check(capi.lib().ma_overflow_check_async(ptr, n, dt, d_flag.data_ptr(),
                                             d_first.data_ptr() if d_first is not None else None,
                                             _stream_ptr(stream)))


# ----------------------------------------------------------------- K2/K3
def adam_step_fp32(params, momentum, variance, grads, t: int, hyper: AdamHyper | None = None,
                   loss_scale: float = 1.0, w_out=None, grad_kind=None, w_kind=None):
    """optimizer.hpp:48-50 / optimizer.cpp:103-109 (+ the cast-back into w_out)."""
    hyper = hyper or AdamHyper()
    pp, n, _ = _info(params)
    mp, nm, _ = _info(momentum)
    vp, nv, _ = _info(variance)
    gp, ng, gdt = _info(grads, grad_kind)
    wp, nw, wdt = _info(w_out, w_kind)
    if not (n == nm == nv == ng) or (w_out is not None and nw != n):
        raise MemAscendError(1, "adam_step: parameter/state/grad lengths differ")
    check(capi.lib().ma_adam_step(pp, mp, vp, gp, gdt, n, t, C.byref(hyper), loss_scale, wp,
                                  wdt))


def adam_step_fp32_async(params, momentum, variance, grads, t, hyper=None, loss_scale=1.0,
                         w_out=None, skip_flag=None, stream=None, grad_kind=None, w_kind=None):
    hyper = hyper or AdamHyper()
    pp, n, _ = _info(params, "f32")
    mp, nm, _ = _info(momentum, "f32")
    vp, nv, _ = _info(variance, "f32")
    gp, ng, gdt = _info(grads, grad_kind)
    wp, nw, wdt = _info(w_out, w_kind)
    for x in (params, momentum, variance):
        if torch is not None and isinstance(x, torch.Tensor) and x.dtype != torch.float32:
            raise MemAscendError(1, "adam_step: p/m/v must be float32")
    if not (n == nm == nv == ng) or (w_out is not None and nw != n):
        raise MemAscendError(1, "adam_step: parameter/state/grad lengths differ")
    check(capi.lib().ma_adam_step_async(pp, mp, vp, gp, gdt, n, t, C.byref(hyper),
                                        loss_scale, wp, wdt,
                                        skip_flag.data_ptr() if skip_flag is not None else None,
                                        _stream_ptr(stream)))


def adam_step_bf16(params, momentum, variance, grads, t: int, hyper: AdamHyper | None = None,
                   loss_scale: float = 1.0):
    """optimizer.hpp:54-57 / optimizer.cpp:111-118 (bf16 state as raw uint16 bits)."""
    hyper = hyper or AdamHyper()
    pp, n, _ = _info(params, "bf16")
    mp, nm, _ = _info(momentum, "bf16")
    vp, nv, _ = _info(variance, "bf16")
    gp, ng, _ = _info(grads, "f32")
    if not (n == nm == nv == ng):
        raise MemAscendError(1, "adam_step: parameter/state/grad lengths differ")
    check(capi.lib().ma_adam_step_bf16(pp, mp, vp, gp, n, t, C.byref(hyper), loss_scale))


@dataclass
class OptimizerState:
    """optimizer.hpp:60-66"""

    master_params: object
    momentum_m: object
    variance_v: object
    step_t: int = 0
    hyper: AdamHyper | None = None


def adam_step(state: OptimizerState, grads, scale: float) -> None:
    """optimizer.cpp:120-124: increments step_t, then the fp32 step."""
    state.step_t += 1
    adam_step_fp32(state.master_params, state.momentum_m, state.variance_v, grads, state.step_t,
                   state.hyper or AdamHyper(), scale)


# ----------------------------------------------------------------- step driver
class Stepper:
    """Device-resident composition of simulator.cpp:427-492 (see the header).

    The scaler state lives in a 64-byte torch uint8 tensor so the overflow
    flag can be all-reduced in place (``flag`` is an int32 view of byte 0).
    """

    def __init__(self, hyper: AdamHyper | None = None, init_scale: float = 65536.0,
                 growth_interval: int = 2000, g_dtype: str = "bf16", w_dtype: str = "bf16",
                 device=None):
        self.hyper = hyper or AdamHyper()
        self.g_dtype, self.w_dtype = g_dtype, w_dtype
        self.state_t = torch.zeros(capi.STEPPER_STATE_BYTES, dtype=torch.uint8,
                                   device=device or "cuda")
        self.flag = self.state_t[0:4].view(torch.int32)
        self.scale_t = self.state_t[8:12].view(torch.float32)
        h = C.c_void_p()
        check(capi.lib().ma_stepper_create(C.byref(self.hyper), init_scale, growth_interval,
                                           capi.DTYPES[g_dtype], capi.DTYPES[w_dtype],
                                           self.state_t.data_ptr(), C.byref(h)))
        self._h = h

    def close(self):
        if self._h:
            capi.lib().ma_stepper_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, grads, stream=None, xchg: "FlagExchange | None" = None):
        """K1 into this step's flag; with `xchg`, K1's last CTA also ORs the
        flag across all ranks over peer memory (use it for the step's last
        gradient buffer only)."""
        if xchg is not None:
            check(capi.lib().ma_stepper_check_xchg_async(
                self._h, grads.data_ptr() if grads is not None else None,
                grads.numel() if grads is not None else 0, xchg._h, _stream_ptr(stream)))
            return
        check(capi.lib().ma_stepper_check_async(self._h, grads.data_ptr(), grads.numel(),
                                                _stream_ptr(stream)))

    def ingest(self, src, dst, src_kind=None, stream=None):
        """dst = src * scale in the stepper's gradient kind, checked in the same pass."""
        sp, n, sdt = _info(src, src_kind)
        check(capi.lib().ma_stepper_ingest_async(self._h, sp, sdt, dst.data_ptr(), n,
                                                 _stream_ptr(stream)))

    def reduce_check(self, srcs, dst, post_scale=1.0, src_kind=None, stream=None):
        """K4: dst = post_scale * (srcs[0] + srcs[1] + ...) (fp32, list order) in
        the stepper's gradient kind, overflow-checked in the same pass."""
        infos = [_info(x, src_kind) for x in srcs]
        n, sdt = infos[0][1], infos[0][2]
        if any(i[1] != n or i[2] != sdt for i in infos) or dst.numel() != n:
            raise MemAscendError(1, "sources and destination must agree in length and kind")
        ptrs = (C.c_void_p * len(infos))(*[i[0] for i in infos])
        check(capi.lib().ma_stepper_reduce_check_async(self._h, ptrs, len(infos), sdt, n,
                                                       post_scale, dst.data_ptr(),
                                                       _stream_ptr(stream)))

    def reduce_scatter(self, rs: "GradReduceScatter", base, n, dst, post_scale=1.0, stream=None):
        """K4 over NVLink peer memory: elements [base, base+n) of every rank's
        shared gradient buffer, summed in rank order into dst; on completion
        the stepper's flag is the OR over all ranks (no all-reduce needed)."""
        if n and dst.numel() < n:
            raise MemAscendError(1, "destination shorter than the partition")
        check(capi.lib().ma_stepper_reduce_scatter_async(
            self._h, rs._h, base, n, post_scale, dst.data_ptr() if n else None,
            _stream_ptr(stream)))

    def check_from_host(self, host_g, dev_g, chunk_elems=64 << 20, stream=None,
                        copy_stream=None):
        """H2D of pinned host gradients into dev_g, K1 overlapped per chunk."""
        if copy_stream is None:
            copy_stream = self._copy_stream = getattr(self, "_copy_stream", None) or \
                torch.cuda.Stream(device=dev_g.device)
        check(capi.lib().ma_stepper_check_host_async(
            self._h, host_g.data_ptr(), dev_g.data_ptr(), dev_g.numel(), chunk_elems,
            _stream_ptr(stream), _stream_ptr(copy_stream)))

    def check_from_host_spec(self, host_g, dev_g, groups, backup, chunk_elems=64 << 20,
                             stream=None, copy_stream=None):
        """check_from_host with the update of each sub-group started as soon
        as its gradients have landed (p/m/v/w backed up into `backup`, a
        device tensor); finish the step with apply_spec(groups) (after any
        flag exchange), then finish().  groups: a subgroups() array whose g
        views tile dev_g in order."""
        arr = self._groups(groups)
        if copy_stream is None:
            copy_stream = self._copy_stream = getattr(self, "_copy_stream", None) or \
                torch.cuda.Stream(device=dev_g.device)
        bp, nb = (backup.data_ptr(), backup.numel() * backup.element_size()) \
            if backup is not None else (None, 0)
        check(capi.lib().ma_stepper_check_host_spec_async(
            self._h, host_g.data_ptr(), dev_g.data_ptr(), dev_g.numel(), chunk_elems, arr,
            len(arr), bp, nb, _stream_ptr(stream), _stream_ptr(copy_stream)))

    def apply_spec(self, groups, stream=None):
        """The step's decision after check_from_host_spec (same groups)."""
        arr = self._groups(groups)
        check(capi.lib().ma_stepper_apply_spec_async(self._h, arr, len(arr), _stream_ptr(stream)))

    @staticmethod
    def subgroups(groups, g_dtype=None, w_dtype=None):
        """ma_subgroup array of (p, m, v, g, w) tensors.  Every tensor must be
        contiguous; p/m/v float32 of one length; g (and w, unless None) of that
        length and — when given — of the stepper's gradient / working kinds."""
        arr = (capi.Subgroup * len(groups))()
        for k, (p, m, v, g, w) in enumerate(groups):
            n = p.numel()
            for name, x in (("p", p), ("m", m), ("v", v)):
                _info(x, "f32")
                if isinstance(x, torch.Tensor) and x.dtype != torch.float32:
                    raise MemAscendError(1, f"sub-group {k}: {name} must be float32")
                if x.numel() != n:
                    raise MemAscendError(1, f"sub-group {k}: p/m/v lengths differ")
            _, ng, _ = _info(g, g_dtype)
            if ng != n:
                raise MemAscendError(1, f"sub-group {k}: gradient length differs")
            if g_dtype is not None and not _kind_ok(g, g_dtype):
                raise MemAscendError(1, f"sub-group {k}: gradients are {g.dtype}, the stepper's "
                                        f"gradient kind is {g_dtype}")
            if w is not None:
                _, nw, _ = _info(w, w_dtype if w_dtype not in (None, "none") else "bf16")
                if nw != n:
                    raise MemAscendError(1, f"sub-group {k}: working-weight length differs")
                if w.element_size() != 2:
                    raise MemAscendError(1, f"sub-group {k}: working weights must be 16-bit")
            elif w_dtype not in (None, "none"):
                raise MemAscendError(1, f"sub-group {k}: the stepper writes {w_dtype} working "
                                        "weights but w is None")
            arr[k] = capi.Subgroup(p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(),
                                   w.data_ptr() if w is not None else None, n)
        return arr

    def _groups(self, groups):
        if isinstance(groups, C.Array):
            return groups
        return self.subgroups(groups, self.g_dtype, self.w_dtype)

    def apply(self, groups, stream=None):
        """groups: list of (p, m, v, g, w) tensors, or a prebuilt subgroups() array."""
        arr = self._groups(groups)
        check(capi.lib().ma_stepper_apply_async(self._h, arr, len(arr), _stream_ptr(stream)))

    def apply_allgather(self, groups, ag: "GradReduceScatter", stream=None):
        """K2 fused with the weight all-gather: `ag` shares every rank's
        full-length working-weight buffer (a GradReduceScatter over it);
        groups' w are views of this rank's buffer."""
        arr = self._groups(groups)
        check(capi.lib().ma_stepper_apply_allgather_async(self._h, arr, len(arr), ag._h,
                                                          _stream_ptr(stream)))

    def apply_bf16(self, groups, stream=None):
        """Pure-bf16 mode: groups of (p_bf16, m_bf16, v_bf16, g) tensors (K3)."""
        arr = self.subgroups_bf16(groups)
        check(capi.lib().ma_stepper_apply_bf16_async(self._h, arr, len(arr), _stream_ptr(stream)))

    def subgroups_bf16(self, groups):
        """ma_subgroup_bf16 array of (p_bf16, m_bf16, v_bf16, g) tensors, checked
        (kinds, lengths, contiguity); a prebuilt array passes through."""
        if isinstance(groups, C.Array):
            return groups
        arr = (capi.SubgroupBf16 * len(groups))()
        for k, (p, m, v, g) in enumerate(groups):
            n = p.numel()
            for name, x in (("p", p), ("m", m), ("v", v)):
                _, nx, _ = _info(x, "bf16")
                if nx != n:
                    raise MemAscendError(1, f"sub-group {k}: p/m/v lengths differ")
                if not _kind_ok(x, "bf16"):
                    raise MemAscendError(1, f"sub-group {k}: {name} must hold bf16 bits")
            _, ng, _ = _info(g, self.g_dtype)
            if ng != n:
                raise MemAscendError(1, f"sub-group {k}: gradient length differs")
            if not _kind_ok(g, self.g_dtype):
                raise MemAscendError(1, f"sub-group {k}: gradients are {g.dtype}, the stepper's "
                                        f"gradient kind is {self.g_dtype}")
            arr[k] = capi.SubgroupBf16(p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(), n)
        return arr

    def check_from_host_spec_bf16(self, host_g, dev_g, groups, backup, chunk_elems=64 << 20,
                                  stream=None, copy_stream=None):
        """check_from_host_spec in the pure-bf16 mode (K3; groups of
        (p_bf16, m_bf16, v_bf16, g) whose g views tile dev_g in order)."""
        arr = self.subgroups_bf16(groups)
        if copy_stream is None:
            copy_stream = self._copy_stream = getattr(self, "_copy_stream", None) or \
                torch.cuda.Stream(device=dev_g.device)
        bp, nb = (backup.data_ptr(), backup.numel() * backup.element_size()) \
            if backup is not None else (None, 0)
        check(capi.lib().ma_stepper_check_host_spec_bf16_async(
            self._h, host_g.data_ptr(), dev_g.data_ptr(), dev_g.numel(), chunk_elems, arr,
            len(arr), bp, nb, _stream_ptr(stream), _stream_ptr(copy_stream)))

    def apply_spec_bf16(self, groups, stream=None):
        """The step's decision after check_from_host_spec_bf16 (same groups)."""
        arr = self.subgroups_bf16(groups)
        check(capi.lib().ma_stepper_apply_spec_bf16_async(self._h, arr, len(arr),
                                                          _stream_ptr(stream)))

    def apply_streamed(self, groups, staging, slot_elems, slots=2, stream=None,
                       h2d_stream=None, d2h_stream=None) -> bool:
        """groups' p/m/v in registered host memory, g/w on the device; staging
        is a device fp32 tensor of 3 * slots * slot_elems.  Returns True when
        the step was skipped (no state moved)."""
        arr = self._groups(groups)
        if staging.dtype != torch.float32 or not staging.is_contiguous() or \
                staging.numel() < 3 * slots * slot_elems:
            raise MemAscendError(1, "staging must be a contiguous float32 tensor of at least "
                                    "3 * slots * slot_elems elements")
        if h2d_stream is None:
            self._h2d = getattr(self, "_h2d", None) or torch.cuda.Stream(device=staging.device)
            h2d_stream = self._h2d
        if d2h_stream is None:
            self._d2h = getattr(self, "_d2h", None) or torch.cuda.Stream(device=staging.device)
            d2h_stream = self._d2h
        skipped = C.c_int()
        check(capi.lib().ma_stepper_apply_streamed(
            self._h, arr, len(arr), staging.data_ptr(), slot_elems, slots, _stream_ptr(stream),
            _stream_ptr(h2d_stream), _stream_ptr(d2h_stream), C.byref(skipped)))
        return bool(skipped.value)

    def apply_swapped(self, store: "DirectIoEngine", groups, host_staging, host_slots,
                      dev_staging, dev_slots, slot_elems, stream=None, h2d_stream=None,
                      d2h_stream=None) -> bool:
        """Config 5: groups are (keys, g, w) with keys = (key_p, key_m, key_v)
        of the fp32 master/m/v in `store`, or ((p, m, v), g, w) with p/m/v in
        registered host memory.  host_staging: registered, 4096-aligned host
        buffer of host_slots x 3 x align4096(4 * slot_elems) bytes;
        dev_staging: device fp32 tensor of 3 * dev_slots * slot_elems.
        Returns True when the step was skipped (nothing read or written)."""
        _check_staging(host_staging, host_slots, dev_staging, dev_slots, slot_elems, 3, 4)
        arr = (capi.SwapGroup * len(groups))()
        keep = []
        for k, (state, g, w) in enumerate(groups):
            n = g.numel()
            if n > slot_elems:  # the C ABI's code for this case (size_violation)
                raise MemAscendError(7, f"group {k}: {n} elements exceed slot_elems {slot_elems}")
            if w is not None and w.numel() != n:
                raise MemAscendError(1, f"group {k}: working-weight length differs")
            if isinstance(state[0], str):
                keys = [x.encode() for x in state]
                keep.append(keys)
                arr[k] = capi.SwapGroup(keys[0], keys[1], keys[2], None, None, None,
                                        g.data_ptr(), w.data_ptr() if w is not None else None, n)
            else:
                if any(_raw(x)[1] < 4 * n for x in state):
                    raise MemAscendError(1, f"group {k}: host p/m/v shorter than the group")
                p, m, v = (_raw(x)[0] for x in state)
                arr[k] = capi.SwapGroup(None, None, None, p, m, v, g.data_ptr(),
                                        w.data_ptr() if w is not None else None, n)
        if h2d_stream is None:
            self._h2d = getattr(self, "_h2d", None) or torch.cuda.Stream(device=dev_staging.device)
            h2d_stream = self._h2d
        if d2h_stream is None:
            self._d2h = getattr(self, "_d2h", None) or torch.cuda.Stream(device=dev_staging.device)
            d2h_stream = self._d2h
        skipped = C.c_int()
        check(capi.lib().ma_stepper_apply_swapped(
            self._h, store.handle if store is not None else None, arr, len(arr),
            _raw(host_staging)[0], host_slots,
            dev_staging.data_ptr(), dev_slots, slot_elems, _stream_ptr(stream),
            _stream_ptr(h2d_stream), _stream_ptr(d2h_stream), C.byref(skipped)))
        return bool(skipped.value)

    def apply_swapped_bf16(self, store: "DirectIoEngine", groups, host_staging, host_slots,
                           dev_staging, dev_slots, slot_elems, stream=None, h2d_stream=None,
                           d2h_stream=None) -> bool:
        """Pure-bf16 swapped update (K3): groups are (state, p, g) with state
        = (key_m, key_v) in `store` or (m, v) bf16 arrays in registered host
        memory, p the device bf16 weights.  host_staging: host_slots x 2 x
        align4096(2 * slot_elems) bytes; dev_staging: 2 * dev_slots *
        slot_elems bf16 (any 2-byte dtype)."""
        _check_staging(host_staging, host_slots, dev_staging, dev_slots, slot_elems, 2, 2)
        arr = (capi.SwapGroupBf16 * len(groups))()
        keep = []
        for k, (state, p, g) in enumerate(groups):
            if p.numel() > slot_elems:
                raise MemAscendError(7, f"group {k}: {p.numel()} elements exceed slot_elems "
                                        f"{slot_elems}")
            if g.numel() != p.numel():
                raise MemAscendError(1, f"group {k}: gradient and weight lengths differ")
            if isinstance(state[0], str):
                keys = [x.encode() for x in state]
                keep.append(keys)
                arr[k] = capi.SwapGroupBf16(keys[0], keys[1], None, None, p.data_ptr(),
                                            g.data_ptr(), p.numel())
            else:
                arr[k] = capi.SwapGroupBf16(None, None, _raw(state[0])[0], _raw(state[1])[0],
                                            p.data_ptr(), g.data_ptr(), p.numel())
        if h2d_stream is None:
            self._h2d = getattr(self, "_h2d", None) or torch.cuda.Stream(device=dev_staging.device)
            h2d_stream = self._h2d
        if d2h_stream is None:
            self._d2h = getattr(self, "_d2h", None) or torch.cuda.Stream(device=dev_staging.device)
            d2h_stream = self._d2h
        skipped = C.c_int()
        check(capi.lib().ma_stepper_apply_swapped_bf16(
            self._h, store.handle if store is not None else None, arr, len(arr),
            _raw(host_staging)[0], host_slots,
            dev_staging.data_ptr(), dev_slots, slot_elems, _stream_ptr(stream),
            _stream_ptr(h2d_stream), _stream_ptr(d2h_stream), C.byref(skipped)))
        return bool(skipped.value)

    def finish(self, stream=None):
        check(capi.lib().ma_stepper_finish_async(self._h, _stream_ptr(stream)))

    def allreduce_flag(self, comm: "NcclComm", stream=None):
        """The step's cross-rank skip decision inside the library: one
        ncclAllReduce(max) of the flag on the compute stream."""
        check(capi.lib().ma_stepper_allreduce_flag_async(self._h, comm._h, _stream_ptr(stream)))

    def set_state(self, scale: float, clean_steps: int, updates: int):
        """Resume a saved run: LossScaler {scale, clean_steps} and the Adam
        step count (OptimizerState::step_t); the next update uses t = updates + 1."""
        check(capi.lib().ma_stepper_set_state(self._h, scale, clean_steps, updates))

    def capture(self, fn, stream, reserve_steps: int = 1 << 20) -> "StepGraph":
        """Record the *_async calls fn() makes on `stream` (a non-default
        torch.cuda.Stream, which fn must use) into a CUDA graph; replay it
        with StepGraph.launch().  Nothing executes during the capture."""
        sp = _stream_ptr(stream)
        check(capi.lib().ma_stepper_graph_begin(self._h, reserve_steps, sp))
        g = C.c_void_p()
        try:
            with torch.cuda.stream(stream):
                fn()
        except BaseException:
            # end the capture (the stream must not stay in capture mode) and
            # drop the partial graph
            if capi.lib().ma_stepper_graph_end(self._h, sp, C.byref(g)) == 0 and g:
                capi.lib().ma_graph_destroy(g)
            raise
        check(capi.lib().ma_stepper_graph_end(self._h, sp, C.byref(g)))
        return StepGraph(g, self)

    def step(self, grads_list, groups, allreduce=None, stream=None):
        """One full step: check every grad buffer, optional cross-rank OR, update, scaler."""
        for g in grads_list:
            self.check(g, stream)
        if allreduce is not None:
            allreduce(self.flag)
        self.apply(groups, stream)
        self.finish(stream)

    def state(self) -> dict:
        s = capi.StepState()
        check(capi.lib().ma_stepper_state(self._h, C.byref(s)))
        return {"scale": s.scale, "clean_steps": s.clean_steps, "updates": s.updates,
                "steps": s.steps, "last_overflow": s.last_overflow,
                "growth_interval": s.growth_interval}

    def history(self, cap: int = 65536):
        of = np.zeros(cap, np.uint8)
        sc = np.zeros(cap, np.float32)
        cnt = C.c_uint64()
        check(capi.lib().ma_stepper_history(self._h, of.ctypes.data, sc.ctypes.data, cap,
                                            C.byref(cnt)))
        return of[:cnt.value].astype(bool), sc[:cnt.value]


class StepGraph:
    """A captured step chain (ma_graph): launch() replays it on a stream."""

    def __init__(self, handle, stepper):
        self._h, self._stepper = handle, stepper

    def launch(self, stream=None):
        check(capi.lib().ma_graph_launch(self._h, _stream_ptr(stream)))

    def close(self):
        if self._h:
            capi.lib().ma_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NcclComm:
    """NCCL communicator owned by the library (ma_comm_*).  Rank 0's unique id
    is distributed by `broadcast(id_bytes_or_None) -> bytes` (any host
    channel; `torch_broadcast_bytes()` uses torch.distributed)."""

    def __init__(self, world: int, rank: int, broadcast):
        uid = None
        if rank == 0:
            buf = (C.c_ubyte * capi.NCCL_ID_BYTES)()
            check(capi.lib().ma_comm_unique_id(buf))
            uid = bytes(buf)
        uid = broadcast(uid)
        assert len(uid) == capi.NCCL_ID_BYTES
        h = C.c_void_p()
        check(capi.lib().ma_comm_create((C.c_ubyte * capi.NCCL_ID_BYTES).from_buffer_copy(uid),
                                        world, rank, C.byref(h)))
        self._h = h
        self.world, self.rank = world, rank

    def info(self) -> dict:
        w, r, v = C.c_int(), C.c_int(), C.c_int()
        check(capi.lib().ma_comm_info(self._h, C.byref(w), C.byref(r), C.byref(v)))
        return {"world": w.value, "rank": r.value, "nccl_version": v.value}

    def allreduce_max_u32(self, t, stream=None):
        """In-place all-reduce(max) of a device int32/uint32 tensor."""
        if t.element_size() != 4 or not t.is_cuda or not t.is_contiguous():
            raise MemAscendError(1, "allreduce_max_u32 needs a contiguous 4-byte device tensor")
        check(capi.lib().ma_comm_allreduce_max_u32(self._h, t.data_ptr(), t.numel(),
                                                   _stream_ptr(stream)))

    def close(self):
        if self._h:
            capi.lib().ma_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def torch_broadcast_bytes(group=None, src=0):
    """broadcast callable for NcclComm over torch.distributed (gloo or nccl)."""
    import torch.distributed as dist

    def bcast(b):
        obj = [b]
        dist.broadcast_object_list(obj, src=src, group=group)
        return obj[0]

    return bcast


class FlagExchange:
    """Cross-rank skip decision over peer memory, fused into K1 (ma_xchg_*).

    `all_gather(handle: bytes) -> list[bytes]` must return every rank's
    64-byte CUDA IPC handle in rank order (e.g. torch.distributed
    all_gather_object); it is the only host-side exchange, done once."""

    def __init__(self, world: int, rank: int, all_gather):
        h = C.c_void_p()
        buf = (C.c_ubyte * capi.IPC_HANDLE_BYTES)()
        check(capi.lib().ma_xchg_create(world, rank, C.byref(h), buf))
        self._h = h
        handles = all_gather(bytes(buf))
        assert len(handles) == world and all(len(x) == capi.IPC_HANDLE_BYTES for x in handles)
        joined = (C.c_ubyte * (capi.IPC_HANDLE_BYTES * world)).from_buffer_copy(b"".join(handles))
        check(capi.lib().ma_xchg_open(self._h, joined))

    def timed_out(self) -> bool:
        e = C.c_int()
        check(capi.lib().ma_xchg_error(self._h, C.byref(e)))
        return bool(e.value)

    def close(self):
        if self._h:
            capi.lib().ma_xchg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GradReduceScatter:
    """Shares this rank's full-length gradient buffer with every peer (ma_rs_*)
    for Stepper.reduce_scatter.  `all_gather(record: bytes) -> list[bytes]`
    returns every rank's record in rank order; it runs once."""

    def __init__(self, world: int, rank: int, grads, all_gather, kind=None):
        gp, n, dt = _info(grads, kind)
        h = C.c_void_p()
        buf = (C.c_ubyte * capi.RS_HANDLE_BYTES)()
        check(capi.lib().ma_rs_create(world, rank, gp, n, dt, C.byref(h), buf))
        self._h = h
        self.grads = grads
        recs = all_gather(bytes(buf))
        assert len(recs) == world and all(len(x) == capi.RS_HANDLE_BYTES for x in recs)
        joined = (C.c_ubyte * (capi.RS_HANDLE_BYTES * world)).from_buffer_copy(b"".join(recs))
        check(capi.lib().ma_rs_open(self._h, joined))

    def timed_out(self) -> bool:
        e = C.c_int()
        check(capi.lib().ma_rs_error(self._h, C.byref(e)))
        return bool(e.value)

    def close(self):
        if self._h:
            capi.lib().ma_rs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def torch_all_gather_bytes(group=None):
    """all_gather callable for FlagExchange over torch.distributed."""
    import torch.distributed as dist

    def gather(b: bytes):
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, b, group=group)
        return out

    return gather


# ----------------------------------------------------------------- workload
def gen_seeded_weights(p, w, n=None, base=0, seed=1, w_kind=None, stream=None):
    wp, _, wdt = _info(w, w_kind)
    n = n if n is not None else (p.numel() if p is not None else w.numel())
    check(capi.lib().ma_gen_seeded_weights_async(p.data_ptr() if p is not None else None, wp,
                                                 wdt, n, base, seed, _stream_ptr(stream)))


def gen_pseudo_grads(g, w, step, base=0, seed=1, scale=65536.0, d_scale=None, g_kind=None,
                     w_kind=None, stream=None):
    gp, n, gdt = _info(g, g_kind)
    wp, _, wdt = _info(w, w_kind)
    check(capi.lib().ma_gen_pseudo_grads_async(gp, gdt, wp, wdt, n, base, seed, step,
                                               d_scale.data_ptr() if d_scale is not None else None,
                                               scale, _stream_ptr(stream)))


def plant_bits(buf, index, bits, kind=None, stream=None):
    bp, _, dt = _info(buf, kind)
    check(capi.lib().ma_plant_bits_async(bp, dt, index, bits, _stream_ptr(stream)))


# ----------------------------------------------------------------- swap store
class DirectIoEngine:
    """DirectIoEngine (proj/include/memascend/direct_io.hpp:94-178) over
    ma_swap_*: key-addressed O_DIRECT tensor store striped over devices.
    devices: list of (path, capacity_bytes[, kind]) or create_virtual_devices'
    result; backend "auto" | "sync" | "aio" | "uring"."""

    def __init__(self, devices, workers=2, queue_depth=8, backend="auto", cache_bypass=True,
                 manifest_path=None):
        devs = (capi.SwapDevice * max(1, len(devices)))()
        self._paths = [d[0].encode() for d in devices]
        for i, d in enumerate(devices):
            devs[i] = capi.SwapDevice(self._paths[i], d[1], d[2] if len(d) > 2 else 1)
        cfg = capi.SwapConfig(workers, queue_depth, capi.IO_BACKENDS[backend],
                              1 if cache_bypass else 0,
                              manifest_path.encode() if manifest_path else None)
        h = C.c_void_p()
        check(capi.lib().ma_swap_create(devs, len(devices), C.byref(cfg), C.byref(h)))
        self.handle = h.value
        self._trace = None

    def close(self):
        if getattr(self, "handle", None):
            check(capi.lib().ma_swap_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @staticmethod
    def create_virtual_devices(directory: str, count: int, nbytes: int):
        check(capi.lib().ma_swap_create_virtual_devices(directory.encode(), count, nbytes))
        return [(f"{directory}/vdev{d}.img", nbytes, 1) for d in range(count)]

    @property
    def backend(self) -> str:
        b = C.c_int()
        check(capi.lib().ma_swap_info(self.handle, C.byref(b), None, None))
        return {v: k for k, v in capi.IO_BACKENDS.items()}[b.value]

    @property
    def total_capacity(self) -> int:
        t = C.c_uint64()
        check(capi.lib().ma_swap_info(self.handle, None, C.byref(t), None))
        return t.value

    def allocate_extents(self, key: str, logical: int):
        ext = (capi.SwapExtent * 64)()
        n = C.c_uint32()
        check(capi.lib().ma_swap_allocate(self.handle, key.encode(), logical, ext, 64,
                                          C.byref(n)))
        return [(e.device_index, e.device_offset, e.length) for e in ext[:n.value]]

    def write_tensor(self, key: str, src, logical: int) -> None:
        ptr, nbytes = _raw(src)
        check(capi.lib().ma_swap_write(self.handle, key.encode(), ptr, nbytes, logical))

    def read_tensor(self, key: str, dst) -> int:
        ptr, nbytes = _raw(dst)
        out = C.c_uint64()
        check(capi.lib().ma_swap_read(self.handle, key.encode(), ptr, nbytes, C.byref(out)))
        return out.value

    def write_tensor_async(self, key: str, src, logical: int) -> "SwapOp":
        ptr, nbytes = _raw(src)
        op = C.c_void_p()
        check(capi.lib().ma_swap_write_async(self.handle, key.encode(), ptr, nbytes, logical,
                                             C.byref(op)))
        return SwapOp(op.value, src)

    def read_tensor_async(self, key: str, dst) -> "SwapOp":
        ptr, nbytes = _raw(dst)
        op = C.c_void_p()
        check(capi.lib().ma_swap_read_async(self.handle, key.encode(), ptr, nbytes, C.byref(op)))
        return SwapOp(op.value, dst)

    def contains(self, key: str) -> bool:
        r = C.c_int()
        check(capi.lib().ma_swap_contains(self.handle, key.encode(), C.byref(r)))
        return bool(r.value)

    def location(self, key: str) -> dict:
        lg, pd, n = C.c_uint64(), C.c_uint64(), C.c_uint32()
        ext = (capi.SwapExtent * 64)()
        check(capi.lib().ma_swap_location(self.handle, key.encode(), C.byref(lg), C.byref(pd),
                                          ext, 64, C.byref(n)))
        return {"logical": lg.value, "padded": pd.value,
                "extents": [(e.device_index, e.device_offset, e.length) for e in ext[:n.value]]}

    def stats(self) -> dict:
        st = capi.SwapStats()
        check(capi.lib().ma_swap_get_stats(self.handle, C.byref(st)))
        return {f: getattr(st, f) for f, _ in capi.SwapStats._fields_}

    def set_io_trace(self, fn) -> None:
        """fn(device, offset, length, write) per device-level submission."""
        self._trace = capi.IO_TRACE_FN(lambda _u, d, o, n, w: fn(d, o, n, bool(w))) if fn else None
        check(capi.lib().ma_swap_set_trace(self.handle, self._trace or capi.IO_TRACE_FN(), None))

    def save_manifest(self) -> None:
        check(capi.lib().ma_swap_save_manifest(self.handle))


class SwapOp:
    """An in-flight store operation; wait() returns the logical length and
    raises the op's error.  The key stays busy until then."""

    def __init__(self, handle, buf):
        self._h, self._buf = handle, buf

    def wait(self) -> int:
        if self._h is None:
            raise MemAscendError(4, "operation already waited on")
        out = C.c_uint64()
        h, self._h = self._h, None
        try:
            check(capi.lib().ma_swap_wait(h, C.byref(out)))
        finally:
            self._buf = None
        return out.value

    def __del__(self):
        # dropped without wait(): the store's workers may still read or write
        # the buffer — finish the operation (and release the key) before the
        # buffer reference goes away; its error, if any, is swallowed here
        if getattr(self, "_h", None) is not None:
            try:
                capi.lib().ma_swap_wait(self._h, C.byref(C.c_uint64()))
            except Exception:
                pass
            self._h = None


class StatePool:
    """configs[3]'s host-resident optimizer state in the drop-in memascend::Pool
    (include/memascend/state_pool.h over pool.hpp, libmemascend.so): an
    adaptive, alignment-free, cudaHostRegister'd pool; every sub-group's
    master / m / v is a checked-out slot, exposed as torch tensors over the
    slot's host span (registered memory: ma_stepper_apply_streamed DMAs from
    and to it directly)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            import os

            path = os.path.join(os.path.dirname(capi.LIB_PATH), "libmemascend.so")
            L = C.CDLL(path)
            L.memascend_last_error.restype = C.c_char_p
            L.memascend_state_pool_create.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(C.c_void_p)]
            L.memascend_state_pool_tensor.argtypes = [C.c_void_p, C.c_uint64, C.c_int,
                                                      C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                                      C.POINTER(C.c_uint64)]
            L.memascend_state_pool_stats.argtypes = [C.c_void_p] + [C.POINTER(C.c_uint64)] * 5
            L.memascend_state_pool_destroy.argtypes = [C.c_void_p]
            cls._lib = L
        return cls._lib

    def _check(self, st):
        if st != 0:
            raise MemAscendError(st, self.lib().memascend_last_error().decode(errors="replace"))

    def __init__(self, n_params: int, subgroup: int):
        h = C.c_void_p()
        self._check(self.lib().memascend_state_pool_create(n_params, subgroup, C.byref(h)))
        self._h = h
        self.groups = (n_params + subgroup - 1) // subgroup

    def tensor(self, group: int, which: int):
        """(host float32 tensor over the slot, device pointer) of master (0), m (1) or v (2)."""
        host, dev, n = C.c_void_p(), C.c_void_p(), C.c_uint64()
        self._check(self.lib().memascend_state_pool_tensor(self._h, group, which, C.byref(host),
                                                           C.byref(dev), C.byref(n)))
        arr = np.ctypeslib.as_array((C.c_float * n.value).from_address(host.value))
        return torch.from_numpy(arr), dev.value

    def stats(self) -> dict:
        v = [C.c_uint64() for _ in range(5)]
        self._check(self.lib().memascend_state_pool_stats(self._h, *[C.byref(x) for x in v]))
        return dict(zip(("capacity_bytes", "backing_bytes", "live_bytes", "checkouts",
                         "classes"), (x.value for x in v)))

    def close(self):
        if self._h:
            self.lib().memascend_state_pool_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DevicePool:
    """Exact-fit slot pool in HBM (ma_dpool): classes = [(payload_bytes,
    slot_count), ...], planned like pool.cpp:22-68 (4096-rounded strides)."""

    def __init__(self, classes):
        nb = (C.c_uint64 * len(classes))(*[c[0] for c in classes])
        nc = (C.c_uint32 * len(classes))(*[c[1] for c in classes])
        h = C.c_void_p()
        check(capi.lib().ma_dpool_create(nb, nc, len(classes), C.byref(h)))
        self.handle = h.value

    def stats(self) -> dict:
        st = capi.DPoolStats()
        check(capi.lib().ma_dpool_get_stats(self.handle, C.byref(st)))
        return {f: getattr(st, f) for f, _ in capi.DPoolStats._fields_}

    def close(self):
        if getattr(self, "handle", None):
            check(capi.lib().ma_dpool_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class _DeviceBytes:
    """__cuda_array_interface__ view of a device allocation (no copy)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


class WeightPrefetcher:
    """Store -> registered host slot -> HBM slot pipeline (ma_prefetcher):
    submit(key) in consumption order; acquire(key, stream) returns a uint8
    device tensor view of the slot (stream waits for its copy);
    release(key, stream) returns the slot after stream's work so far."""

    def __init__(self, store: "DirectIoEngine", pool: DevicePool, host_slots: int,
                 host_slot_bytes: int):
        self.staging = aligned_host_buffer(host_slots * host_slot_bytes, register=True)
        h = C.c_void_p()
        check(capi.lib().ma_prefetcher_create(store.handle, pool.handle, self.staging.ctypes.data,
                                              host_slot_bytes, host_slots, C.byref(h)))
        self.handle = h.value
        self._keep = (store, pool)

    def submit(self, key: str) -> None:
        check(capi.lib().ma_prefetch_submit(self.handle, key.encode()))

    def acquire(self, key: str, stream=None):
        ptr, n = C.c_void_p(), C.c_uint64()
        check(capi.lib().ma_prefetch_acquire(self.handle, key.encode(), _stream_ptr(stream),
                                             C.byref(ptr), C.byref(n)))
        return torch.as_tensor(_DeviceBytes(ptr.value, n.value), device="cuda")

    def release(self, key: str, stream=None) -> None:
        check(capi.lib().ma_prefetch_release(self.handle, key.encode(), _stream_ptr(stream)))

    def close(self):
        if getattr(self, "handle", None):
            check(capi.lib().ma_prefetcher_destroy(self.handle))
            self.handle = None
            host_unregister(self.staging)

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def uring_available() -> bool:
    return bool(capi.lib().ma_swap_uring_available())


_REGISTERED: set = set()  # base addresses registered through host_register


def _unregister_at(ptr: int) -> None:
    if ptr in _REGISTERED:
        _REGISTERED.discard(ptr)
        capi.lib().ma_host_unregister(C.c_void_p(ptr))


def aligned_host_buffer(nbytes: int, register: bool = False) -> np.ndarray:
    """A 4096-aligned uint8 host array (the swap store's O_DIRECT buffers),
    optionally registered for DMA (PinnedAllocator's registered state).  A
    registered buffer is unregistered automatically when its memory is
    released (a finalizer on the owning allocation, run before numpy frees
    it), so freed pages never stay registered behind the allocator's back."""
    import weakref

    raw = np.empty(nbytes + 4096, np.uint8)
    off = (-raw.ctypes.data) % 4096
    buf = raw[off:off + nbytes]
    if register:
        host_register(buf)
        weakref.finalize(raw, _unregister_at, buf.ctypes.data)
    return buf


# ----------------------------------------------------------------- host memory
def _check_staging(host_staging, host_slots, dev_staging, dev_slots, slot_elems, ntens, esize):
    """Sizes of the swapped pipeline's staging buffers (ma_stepper_apply_swapped*)."""
    stride = (esize * slot_elems + 4095) // 4096 * 4096
    if host_slots < 1 or dev_slots < 1 or slot_elems < 1:
        raise MemAscendError(1, "host_slots, dev_slots and slot_elems must be >= 1")
    if _raw(host_staging)[1] < host_slots * ntens * stride:
        raise MemAscendError(1, f"host staging needs {host_slots * ntens * stride} bytes "
                                f"({host_slots} slots x {ntens} x {stride})")
    if not dev_staging.is_contiguous() or \
            dev_staging.numel() * dev_staging.element_size() < dev_slots * ntens * slot_elems * esize:
        raise MemAscendError(1, "device staging smaller than dev_slots x tensors x slot_elems")


def _raw(x):
    """(pointer, bytes) of any tensor / array, whatever its dtype."""
    if torch is not None and isinstance(x, torch.Tensor):
        return x.data_ptr(), x.numel() * x.element_size()
    return x.ctypes.data, x.nbytes


def host_register(array) -> None:
    """PinnedAllocator's "registered" state, made real (pinned.cpp:122-124)."""
    ptr, nbytes = _raw(array)
    check(capi.lib().ma_host_register(ptr, nbytes))
    _REGISTERED.add(ptr)


def host_unregister(array) -> None:
    ptr, _ = _raw(array)
    _REGISTERED.discard(ptr)
    check(capi.lib().ma_host_unregister(ptr))


def pointer_kind(x) -> int:
    ptr, _ = _raw(x)
    k = C.c_int()
    check(capi.lib().ma_pointer_kind(ptr, C.byref(k)))
    return k.value


def device_info() -> dict:
    d, s, a, b = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    check(capi.lib().ma_device_info(C.byref(d), C.byref(s), C.byref(a), C.byref(b)))
    return {"device": d.value, "sm_count": s.value, "cc": (a.value, b.value)}


def debug_cast_sweep(kind: str, block_log2: int = 20) -> np.ndarray:
    out = np.zeros(1 << (32 - block_log2), np.uint64)
    check(capi.lib().ma_debug_cast_sweep(capi.DTYPES[kind], block_log2, out.ctypes.data))
    return out


def debug_fast_sweep(mode: int, divisors=None, samples: int = 0, seed: int = 1):
    """(mismatches, checked) of the Adam fast path vs the IEEE intrinsics."""
    mm, n = C.c_uint64(), C.c_uint64()
    arr = np.ascontiguousarray(divisors if divisors is not None else [], dtype=np.float32)
    check(capi.lib().ma_debug_fast_sweep(mode, arr.ctypes.data if arr.size else None, arr.size,
                                         samples, seed, C.byref(mm), C.byref(n)))
    return mm.value, n.value


def debug_mask_sweep(kind: str) -> int:
    mm = C.c_uint64()
    check(capi.lib().ma_debug_mask_sweep(capi.DTYPES[kind], C.byref(mm)))
    return mm.value

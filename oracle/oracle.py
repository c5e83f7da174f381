"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes + numpy front end for the plain-C restatement of the MemAscend hot path
(oracle/memascend_oracle.c) and, when it has been built, for the unmodified
reference library (oracle/_ref/libmemascend_ref.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker or the
CPU baseline.  The product package (paper_2505_23254_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libmemascend_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmemascend_ref.so")

F32, BF16, F16, NONE = 0, 1, 2, 3
KIND = {"f32": F32, "bf16": BF16, "f16": F16, "none": NONE}


class Hyper(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float), ("weight_decay", C.c_float)]


class Scaler(C.Structure):
    _fields_ = [("scale", C.c_float), ("growth_interval", C.c_uint32),
                ("clean_steps", C.c_uint32)]


class Fault(C.Structure):
    _fields_ = [("step", C.c_uint64), ("index", C.c_uint64), ("bits", C.c_uint32)]


class TrainCfg(C.Structure):
    _fields_ = [("n", C.c_uint64), ("base", C.c_uint64), ("steps", C.c_uint64),
                ("seed", C.c_uint64), ("mixed", C.c_int), ("g_kind", C.c_int),
                ("w_kind", C.c_int), ("hyper", Hyper), ("scaler", Scaler),
                ("faults", C.POINTER(Fault)), ("n_faults", C.c_uint64),
                ("forced_overflow", C.POINTER(C.c_uint8))]


class TrainOut(C.Structure):
    _fields_ = [("p", C.c_void_p), ("m", C.c_void_p), ("v", C.c_void_p),
                ("w", C.c_void_p), ("m16", C.c_void_p), ("v16", C.c_void_p),
                ("overflow", C.c_void_p), ("scale_after", C.c_void_p),
                ("final_scale", C.c_float), ("updates", C.c_uint64)]


class MT64(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        L = C.CDLL(ORACLE_SO)
        L.ora_bf16_from_float.restype = C.c_uint16
        L.ora_bf16_from_float.argtypes = [C.c_float]
        L.ora_fp16_from_float.restype = C.c_uint16
        L.ora_fp16_from_float.argtypes = [C.c_float]
        L.ora_bf16_to_float.restype = C.c_float
        L.ora_bf16_to_float.argtypes = [C.c_uint16]
        L.ora_fp16_to_float.restype = C.c_float
        L.ora_fp16_to_float.argtypes = [C.c_uint16]
        L.ora_cast_from_f32.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int]
        L.ora_widen_to_f32.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int]
        L.ora_cast_sweep_checksums.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int]
        L.ora_overflow_check.restype = C.c_int
        L.ora_overflow_check.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_uint64)]
        L.ora_step_scalars.argtypes = [C.c_uint64, C.c_float, C.c_float,
                                       C.POINTER(C.c_float), C.POINTER(C.c_float)]
        L.ora_adam_step.restype = C.c_int
        L.ora_adam_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                    C.c_uint64, C.c_uint64, C.POINTER(Hyper), C.c_float,
                                    C.c_void_p, C.c_int]
        L.ora_adam_step_bf16.restype = C.c_int
        L.ora_adam_step_bf16.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_uint64, C.c_uint64, C.POINTER(Hyper), C.c_float]
        L.ora_splitmix64.restype = C.c_uint64
        L.ora_splitmix64.argtypes = [C.c_uint64]
        L.ora_pseudo_gradient.restype = C.c_float
        L.ora_pseudo_gradient.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_float]
        L.ora_seeded_weight.restype = C.c_float
        L.ora_seeded_weight.argtypes = [C.c_uint64, C.c_uint64]
        L.ora_train.restype = C.c_int
        L.ora_train.argtypes = [C.POINTER(TrainCfg), C.POINTER(TrainOut)]
        L.ora_train_sample.restype = C.c_int
        L.ora_train_sample.argtypes = [C.POINTER(TrainCfg), C.c_void_p, C.c_uint64, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ora_fnv1a64.restype = C.c_uint64
        L.ora_fnv1a64.argtypes = [C.c_void_p, C.c_uint64]
        L.ora_fill_weights.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                       C.c_int, C.c_int]
        L.ora_fill_grads.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                     C.c_uint64, C.c_uint64, C.c_float, C.c_int, C.c_int, C.c_int]
        L.ora_mt64_seed.argtypes = [C.POINTER(MT64), C.c_uint64]
        L.ora_mt64_next.restype = C.c_uint64
        L.ora_mt64_next.argtypes = [C.POINTER(MT64)]
        L.ora_adversarial_buffer.argtypes = [C.POINTER(MT64), C.c_void_p, C.c_uint64, C.c_int]
        L.ora_reduce_check.restype = C.c_int
        L.ora_reduce_check.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_float,
                                       C.c_int, C.c_void_p]
        _lib = L
    return _lib


# ---------------------------------------------------------------- helpers
def fnv_hex(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return "%016x" % lib().ora_fnv1a64(_ptr(a), a.nbytes)


def cast_from_f32(x: np.ndarray, kind: str) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape, np.uint16)
    lib().ora_cast_from_f32(_ptr(x), _ptr(out), x.size, KIND[kind])
    return out


def widen(h: np.ndarray, kind: str) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.uint16)
    out = np.empty(h.shape, np.float32)
    lib().ora_widen_to_f32(_ptr(h), _ptr(out), h.size, KIND[kind])
    return out


def cast_sweep_checksums(kind: str, block_log2: int = 20, threads: int | None = None):
    nb = 1 << (32 - block_log2)
    out = np.zeros(nb, np.uint64)
    lib().ora_cast_sweep_checksums(KIND[kind], block_log2, _ptr(out), threads or os.cpu_count())
    return out


def overflow_check(data: np.ndarray, kind: str):
    """Returns (overflow: bool, first_index or None) — overflow.cpp:73-145."""
    data = np.ascontiguousarray(data)
    first = C.c_uint64(0)
    r = lib().ora_overflow_check(_ptr(data), data.size, KIND[kind], C.byref(first))
    return bool(r), (first.value if r else None)


def step_scalars(t: int, beta1: float = 0.9, beta2: float = 0.999):
    b1, b2 = C.c_float(), C.c_float()
    lib().ora_step_scalars(t, beta1, beta2, C.byref(b1), C.byref(b2))
    return np.float32(b1.value), np.float32(b2.value)


def hyper(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0) -> Hyper:
    return Hyper(lr, beta1, beta2, eps, weight_decay)


def adam_step(p, m, v, g, t, h: Hyper, loss_scale, g_kind="f32", w_kind="none"):
    """In place on p/m/v (float32); returns the working weights (uint16) or None."""
    n = p.size
    w = np.empty(n, np.uint16) if w_kind != "none" else None
    r = lib().ora_adam_step(_ptr(p), _ptr(m), _ptr(v), _ptr(g), KIND[g_kind], n, t,
                            C.byref(h), loss_scale, _ptr(w), KIND[w_kind])
    if r:
        raise ValueError("invalid_argument: adam step count t must be >= 1")
    return w


def adam_step_bf16(p16, m16, v16, g, t, h: Hyper, loss_scale):
    r = lib().ora_adam_step_bf16(_ptr(p16), _ptr(m16), _ptr(v16), _ptr(g), p16.size, t,
                                 C.byref(h), loss_scale)
    if r:
        raise ValueError("invalid_argument: adam step count t must be >= 1")


def reduce_check(srcs, src_kind: str, post_scale: float = 1.0, dst_kind: str = "bf16"):
    """ora_reduce_check: rank-ordered fp32 sum of `srcs` (bit arrays: uint16
    for bf16/f16, float32 for f32) times post_scale, stored as dst_kind.
    Returns (dst, overflow)."""
    srcs = [np.ascontiguousarray(s) for s in srcs]
    n = srcs[0].size
    assert all(s.size == n for s in srcs)
    ptrs = (C.c_void_p * len(srcs))(*[s.ctypes.data for s in srcs])
    dst = np.empty(n, dtype=np.float32 if dst_kind == "f32" else np.uint16)
    flag = lib().ora_reduce_check(ptrs, len(srcs), KIND[src_kind], n, post_scale,
                                  KIND[dst_kind], dst.ctypes.data)
    return dst, bool(flag)


def pseudo_gradient(seed, step, index, weight):
    return lib().ora_pseudo_gradient(seed, step, index, weight)


def seeded_weight(seed, index):
    return lib().ora_seeded_weight(seed, index)


def _cfg(n, steps, seed, mixed=True, g_kind="bf16", w_kind="bf16", base=0, hyp=None,
         scale=65536.0, growth=2000, faults=(), forced=None):
    fa = (Fault * max(1, len(faults)))(*[Fault(int(s), int(i), int(b)) for s, i, b in faults])
    cfg = TrainCfg(n, base, steps, seed, 1 if mixed else 0, KIND[g_kind], KIND[w_kind],
                   hyp or hyper(), Scaler(scale, growth, 0), fa, len(faults), None)
    keep = [fa]
    if forced is not None:
        fo = np.ascontiguousarray(forced, dtype=np.uint8)
        cfg.forced_overflow = fo.ctypes.data_as(C.POINTER(C.c_uint8))
        keep.append(fo)
    return cfg, keep


def train(n, steps, seed, mixed=True, g_kind="bf16", w_kind="bf16", base=0, hyp=None,
          scale=65536.0, growth=2000, faults=(), forced=None):
    """simulator.cpp:427-492 composition over a partition; returns a dict."""
    cfg, keep = _cfg(n, steps, seed, mixed, g_kind, w_kind, base, hyp, scale, growth, faults,
                     forced)
    res = {"w": np.empty(n, np.uint16), "overflow": np.zeros(steps, np.uint8),
           "scale_after": np.zeros(steps, np.float32)}
    if mixed:
        res.update(p=np.empty(n, np.float32), m=np.empty(n, np.float32), v=np.empty(n, np.float32))
    else:
        res.update(m16=np.empty(n, np.uint16), v16=np.empty(n, np.uint16))
    out = TrainOut(*[_ptr(res.get(k)) for k in ("p", "m", "v", "w", "m16", "v16", "overflow",
                                                  "scale_after")], 0.0, 0)
    r = lib().ora_train(C.byref(cfg), C.byref(out))
    if r:
        raise ValueError(f"ora_train failed: {r}")
    res["final_scale"] = out.final_scale
    res["updates"] = out.updates
    del keep
    return res


def train_sample(indices, decisions, steps, seed, g_kind="bf16", w_kind="bf16", hyp=None,
                 scale=65536.0, growth=2000, mixed=True):
    """Elementwise replay of train() at the given global indices under the
    given step decisions (simulator.cpp:427-492 per element).  mixed=False:
    the pure-bf16 mode; p/m/v are then the exact widenings of the bf16 state."""
    idx = np.ascontiguousarray(indices, dtype=np.uint64)
    dec = np.ascontiguousarray(decisions, dtype=np.uint8)
    cfg, keep = _cfg(1, steps, seed, mixed, g_kind, w_kind, 0, hyp, scale, growth)
    k = idx.size
    p, m, v = (np.empty(k, np.float32) for _ in range(3))
    w = np.empty(k, np.uint16)
    r = lib().ora_train_sample(C.byref(cfg), _ptr(idx), k, _ptr(dec), _ptr(p), _ptr(m), _ptr(v),
                               _ptr(w))
    if r:
        raise ValueError(f"ora_train_sample failed: {r}")
    del keep
    return {"p": p, "m": m, "v": v, "w": w}


def fill_weights(n, base=0, seed=1, w_kind="bf16", threads=None):
    p = np.empty(n, np.float32)
    w = np.empty(n, np.uint16)
    lib().ora_fill_weights(_ptr(p), _ptr(w), n, base, seed, KIND[w_kind], threads or os.cpu_count())
    return p, w


def fill_grads(w, step, base=0, seed=1, scale=65536.0, g_kind="bf16", w_kind="bf16",
               widened=True, threads=None):
    """Returns (stored grads, fp32 widening or None)."""
    n = w.size
    g = np.empty(n, np.float32 if g_kind == "f32" else np.uint16)
    g32 = np.empty(n, np.float32) if widened else None
    lib().ora_fill_grads(_ptr(g), _ptr(g32), _ptr(w), n, base, seed, step, scale, KIND[g_kind],
                         KIND[w_kind], threads or os.cpu_count())
    return g, g32


class MT19937_64:
    """std::mt19937_64 restated (the reference tests' input source)."""

    def __init__(self, seed):
        self.s = MT64()
        lib().ora_mt64_seed(C.byref(self.s), seed)

    def __call__(self):
        return lib().ora_mt64_next(C.byref(self.s))


def adversarial_buffer(rng: MT19937_64, n: int, inject: bool) -> np.ndarray:
    """test_overflow.cpp:30-58 on the restated engine; returns uint32 bit patterns."""
    out = np.empty(n, np.uint32)
    lib().ora_adversarial_buffer(C.byref(rng.s), _ptr(out), n, 1 if inject else 0)
    return out


# ------------------------------------------------------- reference (_ref)
_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The unmodified reference compiled from /root/reference (oracle/Makefile)."""
    global _ref
    if _ref is None:
        R = C.CDLL(REF_SO)
        R.ref_last_error.restype = C.c_char_p
        R.ref_fused_overflow_check.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64,
                                               C.c_int, C.c_int, C.POINTER(C.c_int),
                                               C.POINTER(C.c_uint64)]
        R.ref_adam_step_fp32.argtypes = [C.c_void_p] * 4 + [C.c_uint64, C.c_uint64, C.c_void_p,
                                                            C.c_float, C.c_uint32]
        R.ref_adam_step_bf16.argtypes = [C.c_void_p] * 4 + [C.c_uint64, C.c_uint64, C.c_void_p,
                                                            C.c_float, C.c_uint32]
        R.ref_bench_step.argtypes = [C.c_void_p] * 5 + [C.c_int, C.c_uint64, C.c_uint64,
                                                        C.c_uint64, C.c_void_p, C.c_float,
                                                        C.c_uint32, C.POINTER(C.c_int),
                                                        C.POINTER(C.c_double)]
        R.ref_swap_bench.argtypes = [C.c_char_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                                     C.c_uint32, C.c_void_p, C.c_void_p, C.c_float, C.c_uint32,
                                     C.c_uint32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        R.ref_fp16_from_float.restype = C.c_uint16
        R.ref_fp16_from_float.argtypes = [C.c_float]
        R.ref_bf16_from_float.restype = C.c_uint16
        R.ref_bf16_from_float.argtypes = [C.c_float]
        R.ref_cast_sweep_checksums.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int]
        R.ref_pseudo_gradient.restype = C.c_float
        R.ref_pseudo_gradient.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_float]
        R.ref_seeded_weight.restype = C.c_float
        R.ref_seeded_weight.argtypes = [C.c_uint64, C.c_uint64]
        _ref = R
    return _ref


def ref_hyper_array(h: Hyper) -> np.ndarray:
    return np.array([h.lr, h.beta1, h.beta2, h.eps, h.weight_decay], np.float32)


def ref_adam_step_fp32(p, m, v, g, t, h: Hyper, scale, workers=1):
    hv = ref_hyper_array(h)
    r = ref().ref_adam_step_fp32(_ptr(p), _ptr(m), _ptr(v), _ptr(g), p.size, t, _ptr(hv),
                                 scale, workers)
    if r:
        raise ValueError(ref().ref_last_error().decode())


def ref_adam_step_bf16(p16, m16, v16, g, t, h: Hyper, scale, workers=1):
    """The reference's adam_step_bf16 (optimizer.cpp:111-118) on raw bf16
    (uint16) state and fp32 gradients, in place."""
    hv = ref_hyper_array(h)
    r = ref().ref_adam_step_bf16(_ptr(p16), _ptr(m16), _ptr(v16), _ptr(g), p16.size, t,
                                 _ptr(hv), scale, workers)
    if r:
        raise ValueError(ref().ref_last_error().decode())


def ref_fused_overflow_check(g, workers=1, chunk_bytes=1 << 20, early_exit=True, track=False):
    of, first = C.c_int(), C.c_uint64()
    r = ref().ref_fused_overflow_check(_ptr(g), g.size, workers, chunk_bytes, int(early_exit),
                                       int(track), C.byref(of), C.byref(first))
    if r:
        raise ValueError(ref().ref_last_error().decode())
    return bool(of.value), (first.value if of.value and track else None)


def ref_swap_bench(directory, devices, group_elems, groups, steps, warmup, g, h: Hyper, scale,
                   workers, io_workers=2):
    """The reference's swapped step (DirectIoEngine read -> adam_step_fp32 ->
    write, simulator.cpp:453-469) on `groups` groups stored in `directory`;
    returns (median seconds per step, storage bytes moved per step)."""
    hv = ref_hyper_array(h)
    secs, io = C.c_double(), C.c_double()
    r = ref().ref_swap_bench(directory.encode(), devices, group_elems, groups, steps, warmup,
                             _ptr(g), _ptr(hv), scale, workers, io_workers, C.byref(secs),
                             C.byref(io))
    if r:
        raise ValueError(ref().ref_last_error().decode())
    return secs.value, io.value


def ref_bench_step(g, p, m, v, w, w_kind, subgroup, t, h: Hyper, scale, workers):
    hv = ref_hyper_array(h)
    of, secs = C.c_int(), C.c_double()
    r = ref().ref_bench_step(_ptr(g), _ptr(p), _ptr(m), _ptr(v), _ptr(w), KIND[w_kind], p.size,
                             subgroup, t, _ptr(hv), scale, workers, C.byref(of), C.byref(secs))
    if r:
        raise ValueError(ref().ref_last_error().decode())
    return bool(of.value), secs.value

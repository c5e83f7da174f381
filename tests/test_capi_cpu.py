"""CPU-side checks of the drop-in boundary (no GPU needed).

* libmemascend_b200.so loads and exports every symbol include/memascend_b200.h
  declares, with nothing missing from the ctypes binding;
* without a device the compute entry points fail loudly (no CPU fallback).
"""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "memascend_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^MA_API [^(]*?\b(ma_\w+)\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def so_path():
    from paper_2505_23254_b200 import capi

    if not os.path.exists(capi.LIB_PATH):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2505_23254_b200", "csrc")],
                       check=True)
    return capi.LIB_PATH


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert len(syms) >= 25
    for core in ("ma_overflow_check", "ma_adam_step", "ma_stepper_apply_async",
                 "ma_host_register"):
        assert core in syms


def test_library_exports_every_declared_symbol(so_path):
    out = subprocess.run(["nm", "-D", "--defined-only", so_path], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    extra = sorted(s for s in exported if s.startswith("ma_") and s not in declared_symbols())
    assert not extra, f"exported but undeclared: {extra}"


def test_binding_covers_the_header(so_path):
    from paper_2505_23254_b200 import capi

    bound = {name for name, _, _ in capi.SIGNATURES}
    assert bound == set(declared_symbols())
    lib = capi.lib()
    assert lib.ma_abi_version() == 1


def test_sm100a_only(so_path):
    out = subprocess.run(["cuobjdump", "--list-elf", so_path], capture_output=True, text=True,
                         check=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_no_device_fails_loudly(so_path):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2505_23254_b200 import capi

    lib = capi.lib()
    d = C.c_int()
    assert lib.ma_device_info(C.byref(d), None, None, None) == 101  # MA_ERR_NO_DEVICE
    assert b"no CPU fallback" in lib.ma_last_error()
    of = C.c_int()
    buf = (C.c_float * 4)()
    assert lib.ma_overflow_check(buf, 4, 0, 0, C.byref(of), None) == 101
    h = capi.AdamHyper()
    assert lib.ma_adam_step(buf, buf, buf, buf, 0, 4, 1, C.byref(h), 1.0, None, 3) == 101
    # argument validation still reports the reference's invalid_argument first
    assert lib.ma_adam_step(buf, buf, buf, buf, 0, 4, 0, C.byref(h), 1.0, None, 3) == 1
    # the reduce-scatter entry points need a device too
    rs = C.c_void_p()
    rec = (C.c_ubyte * capi.RS_HANDLE_BYTES)()
    assert lib.ma_rs_create(2, 0, buf, 4, 1, C.byref(rs), rec) == 101
    # the device pool and the prefetcher are GPU objects: no host stand-in
    nb = (C.c_uint64 * 1)(1 << 20)
    nc = (C.c_uint32 * 1)(2)
    dp = C.c_void_p()
    assert lib.ma_dpool_create(nb, nc, 1, C.byref(dp)) == 101
    assert b"no CPU fallback" in lib.ma_last_error()


def test_every_public_header_compiles_on_its_own(tmp_path):
    """Each drop-in / B200 header is self-contained (include order free),
    as the reference's headers are."""
    inc = os.path.join(ROOT, "include")
    hdrs = sorted(f for f in os.listdir(os.path.join(inc, "memascend")) if f.endswith(".hpp"))
    assert {"overflow.hpp", "optimizer.hpp", "pinned.hpp", "pool.hpp", "direct_io.hpp",
            "device_pool.hpp", "step_driver.hpp"} <= set(hdrs)
    for h in hdrs + ["../memascend_b200.h"]:
        src = tmp_path / "one.cpp"
        src.write_text(f'#include "memascend/{h}"\nint main() {{ return 0; }}\n')
        p = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", inc, str(src)],
                           capture_output=True, text=True)
        assert p.returncode == 0, (h, p.stderr[-2000:])
    # the C header is C, too
    src = tmp_path / "one.c"
    src.write_text('#include "memascend_b200.h"\nint main(void) { return 0; }\n')
    p = subprocess.run(["gcc", "-std=c11", "-fsyntax-only", "-I", inc, str(src)],
                       capture_output=True, text=True)
    assert p.returncode == 0, p.stderr[-2000:]


def test_nccl_entry_points_without_a_gpu(so_path):
    """The library resolves libnccl.so.2 at run time: the unique id works on
    any host, a communicator needs a device (MA_ERR_NCCL here, no crash),
    bad arguments are rejected before NCCL is touched."""
    import ctypes as C

    import torch

    from paper_2505_23254_b200 import capi

    L = capi.lib()
    uid = (C.c_ubyte * capi.NCCL_ID_BYTES)()
    assert L.ma_comm_unique_id(uid) == 0 and any(bytes(uid))
    h = C.c_void_p()
    assert L.ma_comm_create(uid, 2, 5, C.byref(h)) == 1  # rank >= world
    if not torch.cuda.is_available():
        assert L.ma_comm_create(uid, 1, 0, C.byref(h)) == 102
        assert b"nccl" in L.ma_last_error().lower()


def test_state_pool_shim_plans_the_drop_in_pool():
    """include/memascend/state_pool.h over memascend::Pool (CPU part): the
    adaptive plan of a 1000-param / 300-param-sub-group state has one exact
    class per distinct size, 4096-byte slot strides and every tensor checked
    out; the device view needs a registered backing (a GPU)."""
    import torch

    import paper_2505_23254_b200 as mab

    sp = mab.StatePool(1000, 300)
    st = sp.stats()
    assert st == {"capacity_bytes": 12000, "backing_bytes": 12 * 4096, "live_bytes": 12000,
                  "checkouts": 12, "classes": 2}
    if not torch.cuda.is_available():
        with pytest.raises(mab.MemAscendError) as e:
            sp.tensor(0, 0)
        assert e.value.code == "capability"
    sp.close()


def test_numa_placement_entry_points(so_path):
    """ma_host_numa_node reports the node backing a page; ma_host_place is a
    best-effort no-op where it cannot act (one node / no device); the
    device's node needs a device."""
    import ctypes as C

    import numpy as np
    import torch

    from paper_2505_23254_b200 import capi

    L = capi.lib()
    a = np.ones(1 << 20, np.uint8)
    node = C.c_int()
    assert L.ma_host_numa_node(a.ctypes.data, C.byref(node)) == 0 and node.value >= -1
    assert L.ma_host_place(a.ctypes.data, a.nbytes) == 0
    if not torch.cuda.is_available():
        assert L.ma_device_numa_node(C.byref(node)) == 101

"""Swap store (DirectIoEngine drop-in over ma_swap_*) — host I/O, runs on CPU.

* the reference's own suite proj/tests/test_direct_io.cpp (14 cases),
  compiled unmodified against include/memascend/direct_io.hpp, under every
  backend (pread/pwrite, POSIX AIO, io_uring);
* on-disk compatibility both ways: a store written by the reference engine
  is read by ours and vice versa (oracle/swap_xcompat.cpp built twice);
* the Python binding: round trips at depth, async ops, the busy guard,
  errors, I/O trace alignment, stats.
"""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2505_23254_b200 as mab
from paper_2505_23254_b200.capi import MemAscendError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_OUT = os.path.join(ROOT, "oracle", "_ref")
BACKENDS = ["sync", "aio"] + (["uring"] if mab.uring_available() else [])


@pytest.mark.parametrize("backend", BACKENDS)
def test_reference_direct_io_suite(backend, tmp_path):
    exe = os.path.join(REF_OUT, "dropin_direct_io")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin_direct_io not built (needs /root/reference at build time)")
    env = dict(os.environ, MEMASCEND_IO_BACKEND=backend, TMPDIR=str(tmp_path))
    p = subprocess.run([exe], capture_output=True, text=True, cwd=str(tmp_path), env=env,
                       timeout=600)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", p.stdout)
    assert m and (int(m.group(1)), int(m.group(3))) == (14, 0), p.stdout + p.stderr


@pytest.mark.parametrize("writer,reader", [("ref", "ours"), ("ours", "ref")])
def test_on_disk_compatibility(writer, reader, tmp_path):
    w = os.path.join(REF_OUT, f"xcompat_{writer}")
    r = os.path.join(REF_OUT, f"xcompat_{reader}")
    if not (os.path.exists(w) and os.path.exists(r)):
        pytest.skip("oracle/_ref/xcompat_* not built (needs /root/reference at build time)")
    d = str(tmp_path / "store")
    for exe, mode in ((w, "write"), (r, "read")):
        p = subprocess.run([exe, mode, d], capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stdout + p.stderr


def payload(nbytes, seed):
    buf = mab.aligned_host_buffer(nbytes)
    buf[:] = np.random.default_rng(seed).integers(0, 256, nbytes, dtype=np.uint8)
    return buf


@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("workers,depth", [(1, 1), (2, 8), (4, 32)])
def test_round_trip_depth(backend, workers, depth, tmp_path):
    devs = mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 3, 64 << 20)
    with mab.DirectIoEngine(devs, workers=workers, queue_depth=depth, backend=backend) as e:
        assert e.backend == backend
        sizes = [1, 4095, 4096, 4097, 5000, (1 << 20) + 7, 24 << 20]
        bufs = {}
        for i, n in enumerate(sizes):
            bufs[i] = payload((n + 4095) // 4096 * 4096, i)
            e.write_tensor(f"t{i}", bufs[i], n)
        for i, n in enumerate(sizes):
            out = mab.aligned_host_buffer((n + 4095) // 4096 * 4096)
            assert e.read_tensor(f"t{i}", out) == n
            assert (out[:n] == bufs[i][:n]).all()
        st = e.stats()
        assert st["write_requests"] == st["read_requests"] == len(sizes)
        assert st["bytes_written"] == st["bytes_read"] == sum((n + 4095) // 4096 * 4096
                                                              for n in sizes)


def test_async_ops_overlap_and_busy_guard(tmp_path):
    devs = mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 2, 128 << 20)
    with mab.DirectIoEngine(devs, workers=2, queue_depth=16) as e:
        srcs = [payload(8 << 20, 100 + k) for k in range(6)]
        ops = [e.write_tensor_async(f"k{k}", srcs[k], 8 << 20) for k in range(6)]
        # a second operation on a key whose op is still pending is refused
        with pytest.raises(MemAscendError) as ei:
            e.read_tensor("k0", mab.aligned_host_buffer(8 << 20))
        assert ei.value.code in ("busy", "not-found")
        for op in ops:
            op.wait()
        dsts = [mab.aligned_host_buffer(8 << 20) for _ in range(6)]
        ops = [e.read_tensor_async(f"k{k}", dsts[k]) for k in range(6)]
        with pytest.raises(MemAscendError) as ei:
            e.write_tensor("k3", srcs[3], 8 << 20)
        assert ei.value.code == "busy"
        assert [op.wait() for op in ops] == [8 << 20] * 6
        for k in range(6):
            assert (dsts[k] == srcs[k]).all()


def test_errors_match_reference_codes(tmp_path):
    devs = mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 1, 1 << 20)
    with mab.DirectIoEngine(devs) as e:
        dst = mab.aligned_host_buffer(8192)
        with pytest.raises(MemAscendError) as ei:
            e.read_tensor("never", dst)
        assert ei.value.code == "not-found"
        src = payload(64 << 10, 3)
        e.write_tensor("t", src, 64 << 10)
        with pytest.raises(MemAscendError) as ei:
            e.read_tensor("t", dst)
        assert ei.value.code == "size-violation"
        with pytest.raises(MemAscendError) as ei:
            e.write_tensor("u", src[1:4097], 4096)
        assert ei.value.code == "alignment"
        with pytest.raises(MemAscendError) as ei:
            e.write_tensor("z", src, 0)
        assert ei.value.code == "invalid-argument"
        with pytest.raises(MemAscendError) as ei:
            e.allocate_extents("huge", 2 << 20)
        assert ei.value.code == "storage-full"
    with pytest.raises(MemAscendError) as ei:
        mab.DirectIoEngine([])
    assert ei.value.code == "invalid-argument"
    with pytest.raises(MemAscendError) as ei:
        mab.DirectIoEngine([(str(tmp_path / "missing.img"), 1 << 20)])
    assert ei.value.code == "device-error"


def test_trace_sees_only_granule_aligned_submissions(tmp_path):
    devs = mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 3, 64 << 20)
    seen = []
    with mab.DirectIoEngine(devs, workers=4) as e:
        e.set_io_trace(lambda d, off, n, w: seen.append((d, off, n, w)))
        rng = np.random.default_rng(17)
        for i in range(16):
            n = int(rng.integers(1, 1 << 19))
            e.write_tensor(f"a{i}", payload((n + 4095) // 4096 * 4096, i), n)
        e.set_io_trace(None)
        e.write_tensor("untraced", payload(4096, 0), 4096)
    assert seen and all(off % 4096 == 0 and n % 4096 == 0 and n > 0 for _, off, n, _ in seen)
    assert all(w for *_, w in seen) and {d for d, *_ in seen} == {0, 1, 2}


def test_manifest_restart(tmp_path):
    devs = mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 2, 64 << 20)
    man = str(tmp_path / "m.json")
    src = payload(12288, 21)
    with mab.DirectIoEngine(devs, manifest_path=man) as e:
        e.write_tensor("persisted", src, 10000)
    assert os.path.exists(man)
    with mab.DirectIoEngine(devs, manifest_path=man) as e:
        out = mab.aligned_host_buffer(12288)
        assert e.read_tensor("persisted", out) == 10000
        assert (out[:10000] == src[:10000]).all()
        assert all(off >= 4096 for _, off, _ in e.allocate_extents("after", 4096))
    with open(man, "w") as f:
        f.write('{"version": 2}')
    with pytest.raises(MemAscendError) as ei:
        mab.DirectIoEngine(devs, manifest_path=man)
    assert ei.value.code == "bad-config"


@pytest.mark.parametrize("backend", BACKENDS)
def test_async_shadow_map_stress(backend, tmp_path):
    """Many async operations in flight from several threads (the swapped
    pipeline's pattern) against a shadow map, every backend."""
    import threading

    devs = mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 3, 96 << 20)
    keys = 24
    shadow = [None] * keys
    locks = [threading.Lock() for _ in range(keys)]
    errors = []
    with mab.DirectIoEngine(devs, workers=3, queue_depth=16, backend=backend) as e:
        def worker(seed):
            rng = np.random.default_rng(seed)
            try:
                for _ in range(40):
                    batch = sorted(set(int(k) for k in rng.integers(0, keys, 4)))
                    held = [locks[k] for k in batch]
                    for lk in held:
                        lk.acquire()
                    try:
                        ops = []
                        for k in batch:
                            if shadow[k] is None or rng.random() < 0.5:
                                n = int(rng.integers(1, 1 << 18))
                                buf = mab.aligned_host_buffer((n + 4095) // 4096 * 4096)
                                buf[:n] = rng.integers(0, 256, n, dtype=np.uint8)
                                ops.append((k, "w", e.write_tensor_async(f"s{k}", buf, n), buf, n))
                            else:
                                n = len(shadow[k])
                                # a shrunk key keeps its old extents: size by the location
                                buf = mab.aligned_host_buffer(e.location(f"s{k}")["padded"])
                                ops.append((k, "r", e.read_tensor_async(f"s{k}", buf), buf, n))
                        for k, kind, op, buf, n in ops:
                            got = op.wait()
                            if kind == "w":
                                shadow[k] = buf[:n].copy()
                            elif got != n or not np.array_equal(buf[:n], shadow[k]):
                                errors.append((k, got, n))
                    finally:
                        for lk in held:
                            lk.release()
            except Exception as ex:  # noqa: BLE001
                errors.append(repr(ex))

        threads = [threading.Thread(target=worker, args=(900 + t,)) for t in range(6)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        st = e.stats()
    assert not errors, errors[:3]
    assert st["write_requests"] >= keys and st["read_requests"] > 0


@pytest.mark.parametrize("backend", BACKENDS)
def test_buffered_mode_round_trip(backend, tmp_path):
    """cache_bypass=False opens the devices without O_DIRECT (the reference's
    EngineConfig::cache_bypass); same contract otherwise."""
    devs = mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 2, 16 << 20)
    with mab.DirectIoEngine(devs, backend=backend, cache_bypass=False) as e:
        src = payload(3 << 20, 5)
        e.write_tensor("b", src, (3 << 20) - 17)
        out = mab.aligned_host_buffer(3 << 20)
        assert e.read_tensor("b", out) == (3 << 20) - 17
        assert (out[:(3 << 20) - 17] == src[:(3 << 20) - 17]).all()

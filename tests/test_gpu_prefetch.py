"""Device-side adaptive pool + weight prefetch on the
B200: tensors stream swap store -> registered host slot -> exact-fit HBM slot
in submission order; contents bit-exact, slot reuse fenced after the
consumer's work (a consumer that releases without synchronising still sees
its own tensor), pool accounting as pool.cpp keeps it, errors by code."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2505_23254_b200 as mab  # noqa: E402

pytestmark = pytest.mark.gpu

# a toy GQA decoder: (name, bytes) per layer + the two global tensors
PER_LAYER = [("q", 1 << 20), ("k", (256 << 10) + 100), ("v", (256 << 10) + 100), ("o", 1 << 20),
             ("gate", 3 << 20), ("up", 3 << 20), ("down", 3 << 20)]
GLOBAL = ("emb", (4 << 20) + 2)


def inventory(layers):
    inv = [GLOBAL]
    for li in range(layers):
        inv += [(f"layer{li}.{n}", b) for n, b in PER_LAYER]
    inv.append(("head", GLOBAL[1]))
    return inv


def adaptive_classes(inflight):
    # pool.cpp:36-42: global members + members_per_layer x inflight blocks
    return [(GLOBAL[1], 2), (3 << 20, 3 * inflight), (1 << 20, 2 * inflight),
            ((256 << 10) + 100, 2 * inflight)]


def fill_store(tmp_path, inv):
    devs = mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 2, 64 << 20)
    store = mab.DirectIoEngine(devs, workers=2, queue_depth=16)
    data = {}
    for k, (name, nb) in enumerate(inv):
        buf = mab.aligned_host_buffer((nb + 4095) // 4096 * 4096)
        buf[:] = np.random.default_rng(k).integers(0, 256, buf.size, dtype=np.uint8)
        store.write_tensor(name, buf, nb)
        data[name] = buf[:nb].copy()
    return store, data


@pytest.mark.parametrize("inflight,host_slots", [(1, 1), (2, 3), (3, 8)])
def test_prefetch_stream_bitexact(tmp_path, inflight, host_slots):
    layers = 5
    inv = inventory(layers)
    store, data = fill_store(tmp_path, inv)
    pool = mab.DevicePool(adaptive_classes(inflight))
    pf = mab.WeightPrefetcher(store, pool, host_slots, 5 << 20)
    for name, _ in inv:
        pf.submit(name)
    stream = torch.cuda.current_stream()
    sums = {}
    held = []
    emb = pf.acquire("emb")
    sums["emb"] = emb.to(torch.int64).sum()
    for li in range(layers):
        for n, _ in PER_LAYER:
            key = f"layer{li}.{n}"
            t = pf.acquire(key)
            assert t.numel() == len(data[key])
            sums[key] = t.to(torch.int64).sum()          # consumer work on `stream`
            if li == 2 and n == "up":                     # one full byte compare too
                assert (t.cpu().numpy() == data[key]).all()
            held.append(key)
        for key in held:                                  # block done: release, no sync
            pf.release(key, stream)
        held = []
    head = pf.acquire("head")
    sums["head"] = head.to(torch.int64).sum()
    assert (head.cpu().numpy() == data["head"]).all()
    pf.release("emb", stream)
    pf.release("head", stream)
    torch.cuda.synchronize()
    for name, _ in inv:
        assert int(sums[name]) == int(data[name].astype(np.int64).sum()), name
    st = pool.stats()
    assert st["checkout_count"] == st["checkin_count"] == len(inv)
    assert st["live_bytes"] == 0
    assert st["capacity_bytes"] == sum(b * c for b, c in adaptive_classes(inflight))
    assert st["peak_live_bytes"] <= st["capacity_bytes"]
    assert st["backing_bytes"] == sum((b + 4095) // 4096 * 4096 * c
                                      for b, c in adaptive_classes(inflight))
    pf.close()
    pool.close()
    store.close()


def test_adaptive_vs_monolithic_backing(tmp_path):
    """PAPER.md §4.2 on the GPU: exact-fit classes vs largest-tensor slots."""
    mono = mab.DevicePool([(GLOBAL[1], 2 + 7 * 2)])
    adap = mab.DevicePool(adaptive_classes(2))
    assert adap.stats()["backing_bytes"] < 0.5 * mono.stats()["backing_bytes"]
    mono.close()
    adap.close()


def test_prefetch_errors(tmp_path):
    inv = inventory(1)
    store, _ = fill_store(tmp_path, inv)
    pool = mab.DevicePool([(1 << 20, 1)])  # nothing bigger than 1 MiB fits
    pf = mab.WeightPrefetcher(store, pool, 2, 5 << 20)
    with pytest.raises(mab.MemAscendError) as ei:
        pf.acquire("layer0.q")
    assert ei.value.code == "not-found"                   # never submitted
    pf.submit("layer0.gate")
    pf.submit("layer0.q")
    with pytest.raises(mab.MemAscendError) as ei:
        pf.acquire("layer0.gate")
    assert ei.value.code == "size-violation"              # fits no device class
    with pytest.raises(mab.MemAscendError) as ei:
        pf.submit("layer0.q")
    assert ei.value.code == "already-checked-out"
    t = pf.acquire("layer0.q")
    assert t.numel() == 1 << 20
    with pytest.raises(mab.MemAscendError) as ei:
        pf.release("layer0.o")
    assert ei.value.code == "lifecycle"
    pf.release("layer0.q")
    pf.submit("missing-key")
    with pytest.raises(mab.MemAscendError) as ei:
        pf.acquire("missing-key")
    assert ei.value.code == "not-found"
    pf.submit("layer0.o")                                 # left in flight: close drains it
    pf.close()
    assert pool.stats()["live_bytes"] == 0
    pool.close()
    store.close()


def test_cpp_device_pool_and_prefetcher(tmp_path):
    """include/memascend/device_pool.hpp from C++: class plan equals the
    reference Pool's pool_capacity() on the llama3.1-8b inventory; a toy
    model's tensors stream through WeightPrefetcher bit-exactly."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2505_23254_b200", "lib")
    exe = str(tmp_path / "device_pool_check")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(root, "include"),
                    "-I", "/usr/local/cuda/include", os.path.join(root, "tests", "cpp",
                                                               "device_pool_check.cpp"),
                    "-o", exe, "-L", lib, "-lmemascend", "-lmemascend_b200",
                    "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib}",
                    "-Wl,-rpath,/usr/local/cuda/lib64", "-pthread"], check=True)
    p = subprocess.run([exe, str(tmp_path / "store")], capture_output=True, text=True,
                       timeout=120)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stdout + p.stderr


@pytest.mark.parametrize("mode", ["hbm", "swapped", "nccl", "graph", "resume"])
def test_cpp_step_driver_workload_golden(golden, tmp_path, mode):
    """include/memascend/step_driver.hpp from C++: the reference's workload
    case through StepDriver (HBM-resident and swapped) ends on the golden
    per-step digests of the unmodified reference."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2505_23254_b200", "lib")
    exe = str(tmp_path / "step_driver_check")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(root, "include"),
                    "-I", "/usr/local/cuda/include",
                    os.path.join(root, "tests", "cpp", "step_driver_check.cpp"), "-o", exe,
                    "-L", lib, "-lmemascend", "-lmemascend_b200", "-L", "/usr/local/cuda/lib64",
                    "-lcudart", f"-Wl,-rpath,{lib}", "-Wl,-rpath,/usr/local/cuda/lib64",
                    "-pthread"], check=True)
    p = subprocess.run([exe, mode, str(tmp_path / "store")], capture_output=True, text=True,
                       timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    keys = {"p", "m", "v", "w", "scale", "updates"}
    got = dict(line.split() for line in p.stdout.split("\n")
               if len(line.split()) == 2 and line.split()[0] in keys)
    assert keys <= set(got), p.stdout + p.stderr
    c = next(x for x in golden("workload.json")["cases"] if x["name"] == "cfg_bf16_n100003")
    last = c["per_step"][-1]
    for k in "pmvw":
        assert got[k] == last[f"{k}_fnv"], (k, got[k])
    assert float(got["scale"]) == c["final_scale"] and int(got["updates"]) == c["updates"]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_prefetch_random_stream(tmp_path, seed):
    """200 tensors of random sizes in three classes; the consumer keeps a
    sliding window of held tensors (smaller than every class's slot count),
    reducing each on its stream before releasing it without a sync."""
    rng = np.random.default_rng(seed)
    classes = [(1 << 20, 4), (256 << 10, 6), (37 << 10, 8)]
    window = 3
    names, data = [], {}
    devs = mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 2, 128 << 20)
    store = mab.DirectIoEngine(devs, workers=3, queue_depth=16)
    for k in range(200):
        cap = classes[int(rng.integers(0, 3))][0]
        nb = int(rng.integers(cap // 2 + 1, cap + 1))  # tightest class = the drawn one
        buf = mab.aligned_host_buffer((nb + 4095) // 4096 * 4096)
        buf[:] = rng.integers(0, 256, buf.size, dtype=np.uint8)
        store.write_tensor(f"t{k}", buf, nb)
        names.append(f"t{k}")
        data[f"t{k}"] = int(buf[:nb].astype(np.int64).sum())
    pool = mab.DevicePool(classes)
    pf = mab.WeightPrefetcher(store, pool, int(rng.integers(1, 5)), 1 << 20)
    for nm in names:
        pf.submit(nm)
    stream = torch.cuda.current_stream()
    held, sums = [], {}
    for nm in names:
        t = pf.acquire(nm)
        sums[nm] = t.to(torch.int64).sum()
        held.append(nm)
        if len(held) > window:
            pf.release(held.pop(0), stream)
    for nm in held:
        pf.release(nm, stream)
    torch.cuda.synchronize()
    assert all(int(sums[nm]) == data[nm] for nm in names)
    st = pool.stats()
    assert st["checkout_count"] == st["checkin_count"] == len(names) and st["live_bytes"] == 0
    pf.close()
    pool.close()
    store.close()

"""Config 5 path on the B200: optimizer state in the swap store (NVMe tier)
and in registered host memory (DRAM tier), streamed store -> registered host
slot -> HBM -> K2 -> back by ma_stepper_apply_swapped, against the
reference's per-step digests (tests/golden/workload.json, produced by the
unmodified reference) — bit-exact — plus the I/O accounting of
simulator.cpp:436-469 (a skipped step reads and writes no state)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2505_23254_b200 as mab  # noqa: E402
from oracle import oracle as ora  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"


def u2f(x):
    return float(np.uint32(x).view(np.float32))


def fnv_f32(a) -> str:
    return ora.fnv_hex(np.ascontiguousarray(a, np.float32))


def fnv16(t) -> str:
    return ora.fnv_hex(t.view(torch.int16).cpu().numpy().view(np.uint16))


def align4k(n):
    return (n + 4095) // 4096 * 4096


@pytest.mark.parametrize("backend", ["auto", "sync", "aio"])
@pytest.mark.parametrize("host_slots,dev_slots,tier", [(2, 2, "all-swapped"), (3, 2, "mixed"),
                                                       (4, 3, "mixed")])
def test_swapped_apply_workload_golden(golden, tmp_path, backend, host_slots, dev_slots, tier):
    c = next(x for x in golden("workload.json")["cases"] if x["name"] == "cfg_bf16_n100003")
    n, sub, seed = c["n"], c["subgroup"], c["seed"]
    hyper = mab.AdamHyper(lr=u2f(c["lr"]), beta1=u2f(c["beta1"]), beta2=u2f(c["beta2"]),
                          eps=u2f(c["eps"]), weight_decay=u2f(c["wd"]))
    pd = torch.empty(n, dtype=torch.float32, device=DEV)
    w = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    g = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    mab.gen_seeded_weights(pd, w, seed=seed)
    p0 = pd.cpu().numpy()
    offs = list(range(0, n, sub))
    slot = align4k(sub) // 4 * 4  # elements per slot (multiple of 4, >= sub)
    devs = mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 2, 64 << 20)
    store = mab.DirectIoEngine(devs, workers=2, queue_depth=8, backend=backend)
    # tiering: "mixed" keeps every other group in registered host DRAM
    swapped = [tier == "all-swapped" or k % 2 == 0 for k in range(len(offs))]
    host = {}
    groups = []
    buf = mab.aligned_host_buffer(align4k(sub * 4))
    for k, o in enumerate(offs):
        ln = min(sub, n - o)
        if swapped[k]:
            for name, arr in (("master", p0[o:o + ln]), ("m", np.zeros(ln, np.float32)),
                              ("v", np.zeros(ln, np.float32))):
                buf.view(np.float32)[:ln] = arr
                store.write_tensor(f"{name}.g{k}", buf, ln * 4)
            groups.append(((f"master.g{k}", f"m.g{k}", f"v.g{k}"), g[o:o + ln], w[o:o + ln]))
        else:
            t = [torch.tensor(p0[o:o + ln]).pin_memory(), torch.zeros(ln).pin_memory(),
                 torch.zeros(ln).pin_memory()]
            host[k] = t
            groups.append((tuple(t), g[o:o + ln], w[o:o + ln]))
    hstage = mab.aligned_host_buffer(host_slots * 3 * align4k(slot * 4), register=True)
    dstage = torch.empty(3 * dev_slots * slot, dtype=torch.float32, device=DEV)
    st = mab.Stepper(hyper, c["init_scale"], c["growth_interval"], "bf16", "bf16")

    def gather(name, idx):
        out = np.empty(n, np.float32)
        rb = mab.aligned_host_buffer(align4k(sub * 4))
        for k, o in enumerate(offs):
            ln = min(sub, n - o)
            if swapped[k]:
                assert store.read_tensor(f"{name}.g{k}", rb) == ln * 4
                out[o:o + ln] = rb.view(np.float32)[:ln]
            else:
                out[o:o + ln] = host[k][idx].numpy()
        return out

    n_sw = sum(swapped)
    for s, want in enumerate(c["per_step"]):
        mab.gen_pseudo_grads(g, w, step=s, seed=seed, d_scale=st.scale_t)
        for f in c["faults"]:
            if f["step"] == s:
                mab.plant_bits(g, f["index"] % n, f["bits"])
        st.check(g)
        before = store.stats()
        skipped = st.apply_swapped(store, groups, hstage, host_slots, dstage, dev_slots, slot)
        st.finish()
        torch.cuda.synchronize()
        after = store.stats()
        assert skipped == want["overflow"]
        moved = (after["read_requests"] - before["read_requests"],
                 after["write_requests"] - before["write_requests"])
        assert moved == ((0, 0) if skipped else (3 * n_sw, 3 * n_sw)), (s, moved)
        for key, idx, name in (("p", 0, "master"), ("m", 1, "m"), ("v", 2, "v")):
            assert fnv_f32(gather(name, idx)) == want[f"{key}_fnv"], (s, key)
        assert fnv16(w) == want["w_fnv"], s
    store.close()
    mab.host_unregister(hstage)


def test_swapped_rejects_bad_staging(tmp_path):
    devs = mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 1, 16 << 20)
    store = mab.DirectIoEngine(devs)
    n = 4096
    g = torch.zeros(n, dtype=torch.bfloat16, device=DEV)
    w = torch.zeros(n, dtype=torch.bfloat16, device=DEV)
    st = mab.Stepper(mab.AdamHyper(), 65536.0, 2000, "bf16", "bf16")
    dstage = torch.empty(3 * 2 * n, dtype=torch.float32, device=DEV)
    unregistered = mab.aligned_host_buffer(2 * 3 * n * 4)
    with pytest.raises(mab.MemAscendError) as ei:
        st.apply_swapped(store, [(("a", "b", "c"), g, w)], unregistered, 2, dstage, 2, n)
    assert ei.value.code == "invalid-argument"
    hstage = mab.aligned_host_buffer(2 * 3 * n * 4, register=True)
    with pytest.raises(mab.MemAscendError) as ei:  # group larger than a slot
        st.apply_swapped(store, [(("a", "b", "c"), g, w)], hstage, 2, dstage, 2, n // 2)
    assert ei.value.code == "size-violation"
    st.check(g)
    with pytest.raises(mab.MemAscendError) as ei:  # keys never written
        st.apply_swapped(store, [(("a", "b", "c"), g, w)], hstage, 2, dstage, 2, n)
    assert ei.value.code == "not-found"
    mab.host_unregister(hstage)
    store.close()


def _bf16_run(t, c, sub, mode, tmp_path, fault=None, host_slots=3, dev_slots=2):
    """Pure-bf16 run of the reference trainer's workload (test_simulator.cpp:44-51):
    mode "hbm" = K3 over HBM state (ma_stepper_apply_bf16_async), "swapped" =
    m/v in the store, "mixed" = every other group's m/v in registered DRAM."""
    n, seed = t["n"], c["seed"]
    w = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    g = torch.empty(n, dtype=torch.float32, device=DEV)
    mab.gen_seeded_weights(None, w, n=n, seed=seed)
    st = mab.Stepper(mab.AdamHyper(), 65536.0, 2000, "f32", "none")
    offs = list(range(0, n, sub))
    store = None
    moved = []
    if mode == "hbm":
        m = torch.zeros(n, dtype=torch.int16, device=DEV)
        v = torch.zeros(n, dtype=torch.int16, device=DEV)
        groups = [(w[o:o + sub], m[o:o + sub], v[o:o + sub], g[o:o + sub]) for o in offs]
    else:
        devs = mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 2, 16 << 20)
        store = mab.DirectIoEngine(devs, backend="auto")
        zeros = mab.aligned_host_buffer(align4k(sub * 2))
        zeros[:] = 0
        groups = []
        for k, o in enumerate(offs):
            ln = min(sub, n - o)
            if mode == "swapped" or k % 2 == 0:
                for name in ("m", "v"):
                    store.write_tensor(f"{name}.g{k}", zeros, ln * 2)
                groups.append(((f"m.g{k}", f"v.g{k}"), w[o:o + ln], g[o:o + ln]))
            else:
                mv = (torch.zeros(ln, dtype=torch.int16).pin_memory(),
                      torch.zeros(ln, dtype=torch.int16).pin_memory())
                groups.append((mv, w[o:o + ln], g[o:o + ln]))
        slot = align4k(sub * 2) // 2
        hstage = mab.aligned_host_buffer(host_slots * 2 * align4k(slot * 2), register=True)
        dstage = torch.empty(2 * dev_slots * slot, dtype=torch.int16, device=DEV)
    for s in range(c["steps"]):
        mab.gen_pseudo_grads(g, w, step=s, seed=seed, d_scale=st.scale_t)
        if fault and fault[0] == s:
            mab.plant_bits(g, fault[1], fault[2])
        st.check(g)
        if mode == "hbm":
            st.apply_bf16(groups)
        else:
            before = store.stats()["read_requests"]
            st.apply_swapped_bf16(store, groups, hstage, host_slots, dstage, dev_slots, slot)
            moved.append(store.stats()["read_requests"] - before)
        st.finish()
    torch.cuda.synchronize()
    out = dict(w=fnv16(w), scale=st.state()["scale"], moved=moved)
    if store:
        store.close()
        mab.host_unregister(hstage)
    return out


@pytest.mark.parametrize("mode", ["swapped", "mixed"])
@pytest.mark.parametrize("sub", [10007 * 2, 53248])
def test_swapped_pure_bf16_reference_digest(golden, tmp_path, mode, sub):
    """Pure-bf16 swapped step (bf16 m/v in the store, weights in HBM, K3)
    reproduces the reference simulator's pure-bf16 digest bit for bit."""
    t = golden("trainer.json")
    c = next(x for x in t["cases"] if x["pure_bf16"])
    r = _bf16_run(t, c, sub, mode, tmp_path)
    assert r["w"] == c["sim_digest"]
    assert r["scale"] == c["final_scale"]


def test_swapped_pure_bf16_skip_moves_nothing(golden, tmp_path):
    """A planted NaN: the swapped run skips the step without touching the
    store and stays bitwise equal to the in-HBM K3 run."""
    t = golden("trainer.json")
    c = next(x for x in t["cases"] if x["pure_bf16"])
    fault = (3, 4242, 0x7FC00000)
    a = _bf16_run(t, c, 20014, "hbm", tmp_path, fault)
    b = _bf16_run(t, c, 20014, "swapped", tmp_path, fault)
    assert a["w"] == b["w"] and a["scale"] == b["scale"] == 65536.0 / 2
    groups = (t["n"] + 20013) // 20014
    assert b["moved"] == [0 if s == 3 else 2 * groups for s in range(c["steps"])]


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_swapped_random_groups_equal_hbm_path(tmp_path, seed):
    """Random group boundaries (including 1..9-element groups), random tiers
    and slot counts: the swapped pipeline equals the HBM-resident K2 path
    bit for bit over 3 steps with a planted NaN at step 1."""
    rng = np.random.default_rng(seed)
    cuts = sorted(set(int(x) for x in rng.integers(1, 60_000, 12)) | {3, 7, 16})
    bounds = [0] + cuts + [60_011]
    spans = [(a, b - a) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
    n = bounds[-1]
    g = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    w_ref = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    w_sw = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    p_ref = torch.empty(n, dtype=torch.float32, device=DEV)
    mab.gen_seeded_weights(p_ref, w_ref, seed=seed)
    w_sw.copy_(w_ref)
    m_ref = torch.zeros(n, device=DEV)
    v_ref = torch.zeros(n, device=DEV)
    p0 = p_ref.cpu().numpy()
    hyper = mab.AdamHyper(weight_decay=0.01)
    st_ref = mab.Stepper(hyper, 65536.0, 2000, "bf16", "bf16")
    st_sw = mab.Stepper(hyper, 65536.0, 2000, "bf16", "bf16")
    slot = max(((max(ln for _, ln in spans) + 7) // 8) * 8, 8)
    hslots, dslots = int(rng.integers(2, 5)), int(rng.integers(2, 4))
    devs = mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 2, 32 << 20)
    store = mab.DirectIoEngine(devs, backend="auto")
    buf = mab.aligned_host_buffer(align4k(slot * 4))
    ref_groups, sw_groups, host = [], [], {}
    for k, (o, ln) in enumerate(spans):
        ref_groups.append((p_ref[o:o + ln], m_ref[o:o + ln], v_ref[o:o + ln], g[o:o + ln],
                           w_ref[o:o + ln]))
        if rng.random() < 0.6:
            for name, arr in (("master", p0[o:o + ln]), ("m", np.zeros(ln, np.float32)),
                              ("v", np.zeros(ln, np.float32))):
                buf.view(np.float32)[:ln] = arr
                store.write_tensor(f"{name}.g{k}", buf, ln * 4)
            sw_groups.append(((f"master.g{k}", f"m.g{k}", f"v.g{k}"), g[o:o + ln],
                              w_sw[o:o + ln]))
        else:
            t = [torch.tensor(p0[o:o + ln]).pin_memory(), torch.zeros(ln).pin_memory(),
                 torch.zeros(ln).pin_memory()]
            host[k] = t
            sw_groups.append((tuple(t), g[o:o + ln], w_sw[o:o + ln]))
    hstage = mab.aligned_host_buffer(hslots * 3 * align4k(slot * 4), register=True)
    dstage = torch.empty(3 * dslots * slot, dtype=torch.float32, device=DEV)
    for s in range(3):
        mab.gen_pseudo_grads(g, w_ref, step=s, seed=seed, d_scale=st_ref.scale_t)
        if s == 1:
            mab.plant_bits(g, int(rng.integers(0, n)), 0x7FC0)
        st_ref.check(g)
        st_ref.apply(ref_groups)
        st_ref.finish()
        st_sw.check(g)
        st_sw.apply_swapped(store, sw_groups, hstage, hslots, dstage, dslots, slot)
        st_sw.finish()
        torch.cuda.synchronize()
    rb = mab.aligned_host_buffer(align4k(slot * 4))
    for k, (o, ln) in enumerate(spans):
        for idx, name, ref in ((0, "master", p_ref), (1, "m", m_ref), (2, "v", v_ref)):
            if k in host:
                got = host[k][idx].numpy()
            else:
                store.read_tensor(f"{name}.g{k}", rb)
                got = rb.view(np.float32)[:ln]
            assert np.array_equal(got.view(np.uint32),
                                  ref[o:o + ln].cpu().numpy().view(np.uint32)), (k, name)
    assert torch.equal(w_sw.view(torch.int16), w_ref.view(torch.int16))
    assert st_sw.state()["scale"] == st_ref.state()["scale"] == 32768.0
    store.close()
    mab.host_unregister(hstage)

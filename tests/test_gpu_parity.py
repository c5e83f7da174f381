"""GPU parity: the sm_100a path through the C ABI against the oracle and the
reference's golden vectors (tests/golden, produced by the unmodified
reference).  Integer/bit work is compared bit-exactly; the fp32 Adam state is
compared bit-exactly too (the numeric contract makes 0 ulp achievable; the
north star's tolerance is <= 2 ulp per step, asserted as 0 here).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2505_23254_b200 as mab  # noqa: E402
from oracle import oracle as ora  # noqa: E402

pytestmark = pytest.mark.gpu
f32 = np.float32
DEV = "cuda"


# ------------------------------------------------------------------ helpers
def dev_bits16(a: np.ndarray) -> "torch.Tensor":
    return torch.from_numpy(np.ascontiguousarray(a, np.uint16).view(np.int16)).to(DEV)


def host_bits16(t) -> np.ndarray:
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def host_f32(t) -> np.ndarray:
    return t.cpu().numpy()


def fnv(t) -> str:
    if t.dtype in (torch.bfloat16, torch.float16, torch.int16):
        return ora.fnv_hex(host_bits16(t))
    return ora.fnv_hex(t.cpu().numpy())


def ulp_diff(a: np.ndarray, b: np.ndarray) -> int:
    ia = a.view(np.int32).astype(np.int64)
    ib = b.view(np.int32).astype(np.int64)
    ia = np.where(ia < 0, -(ia & 0x7FFFFFFF), ia)
    ib = np.where(ib < 0, -(ib & 0x7FFFFFFF), ib)
    return int(np.abs(ia - ib).max(initial=0))


def u2f(x):
    return float(np.uint32(x).view(f32))


# ------------------------------------------------------------------ K1
def test_device_info():
    info = mab.device_info()
    assert info["cc"][0] == 10 and info["sm_count"] >= 100


def test_k1_forced_bit_patterns():
    # test_overflow.cpp:62-75
    t = torch.ones(4, dtype=torch.float32, device=DEV)
    for bits, expect in ((0xFF800000, True), (0x7F7FFFFF, False), (0x7F800001, True)):
        t.view(torch.int32)[2] = np.int32(np.uint32(bits).view(np.int32))
        assert mab.fused_overflow_check(t).overflow == expect


def test_k1_all_zero_megabuffer():
    assert not mab.fused_overflow_check(torch.zeros(1 << 20, device=DEV)).overflow


def _nan_index_buffer(g):
    rng = ora.MT19937_64(g["seed"])
    vals = np.array([rng() % 1000 for _ in range(g["n"])], np.uint64).astype(f32) * f32(0.5) - f32(250.0)
    where = rng() % g["n"]
    vals.view(np.uint32)[where] = 0x7F800001
    return vals, where


def test_k1_nan_index_device_host_registered(golden):
    # test_overflow.cpp:85-104 on device, pageable host and registered host memory
    g = golden("nan_index.json")
    vals, where = _nan_index_buffer(g)
    assert where == g["where"]
    r = mab.fused_overflow_check(torch.from_numpy(vals).to(DEV), track_first_index=True)
    assert (r.overflow, r.first_offending_index) == (True, g["first_index"])
    r = mab.fused_overflow_check(vals, track_first_index=True)  # pageable
    assert (r.overflow, r.first_offending_index) == (True, g["first_index"])
    reg = vals.copy()
    mab.host_register(reg)
    try:
        assert mab.pointer_kind(reg) == 2
        r = mab.fused_overflow_check(reg, track_first_index=True)
        assert (r.overflow, r.first_offending_index) == (True, g["first_index"])
    finally:
        mab.host_unregister(reg)


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
def test_k1_adversarial_golden(golden, offset):
    """test_overflow.cpp:106-125: 300 adversarial buffers, reference decisions;
    offset > 0 runs the same buffers through a misaligned view."""
    gj = golden("adversarial.json")
    rng = ora.MT19937_64(gj["seed"])
    for rd in gj["rounds"]:
        n = 1 + rng() % 4096
        inject = rng() % 2 == 0
        buf = ora.adversarial_buffer(rng, n, inject)
        for _ in range(3):
            rng()
        padded = np.concatenate([np.zeros(offset, np.uint32), buf])
        t = torch.from_numpy(padded.view(np.int32)).to(DEV).view(torch.float32)[offset:]
        r = mab.fused_overflow_check(t, track_first_index=True)
        assert r.overflow == rd["overflow"]
        assert r.first_offending_index == rd["first_index"]
        assert mab.fused_overflow_check(t).overflow == rd["overflow"]
        # 16-bit kinds: the top halves as bf16 and fp16 patterns vs the oracle
        hi = (padded >> 16).astype(np.uint16)
        for kind in ("bf16", "f16"):
            th = dev_bits16(hi)[offset:]
            want = ora.overflow_check(hi[offset:], kind)
            r = mab.fused_overflow_check(th, track_first_index=True, kind=kind)
            assert (r.overflow, r.first_offending_index) == want


@pytest.mark.parametrize("kind", ["f32", "bf16", "f16"])
def test_k1_mask_exhaustive(kind):
    # test_overflow.cpp:167-197 (MEMASCEND_EXHAUSTIVE): every pattern
    assert mab.api.debug_mask_sweep(kind) == 0


@pytest.mark.parametrize("kind", ["f32", "bf16"])
def test_k1_large_positions(kind):
    n = (50 << 20) + 7
    dt = torch.float32 if kind == "f32" else torch.bfloat16
    t = torch.full((n + 8,), 0.5, dtype=dt, device=DEV)
    bad = 0x7FC00000 if kind == "f32" else 0x7FC0
    for off in (0, 3):
        view = t[off:off + n]
        assert not mab.fused_overflow_check(view).overflow
        for pos in (0, 1, 5, 1000, n // 2, n - 9, n - 1):
            mab.plant_bits(view, pos, bad)
            r = mab.fused_overflow_check(view, track_first_index=True)
            assert (r.overflow, r.first_offending_index) == (True, pos), (off, pos)
            view[pos] = 0.5


# ------------------------------------------------------------------ casts
@pytest.mark.parametrize("kind,key", [("bf16", "bf16_from_float"), ("f16", "fp16_from_float")])
def test_cast_exhaustive_vs_reference(golden, kind, key):
    """All 2^32 fp32 inputs through the device cast K2 uses, vs the reference."""
    g = golden("halfprec.json")
    got = mab.api.debug_cast_sweep(kind, g["block_log2"])
    want = np.array([int(x, 16) for x in g[key]], np.uint64)
    assert (got == want).all(), np.nonzero(got != want)[0][:5]


# ------------------------------------------------------- Adam fast path
def test_fast_path_sqrt_exhaustive():
    """sqrt_fast == __fsqrt_rn for every input the guarded fast path admits."""
    bad, n = mab.api.debug_fast_sweep(0)
    assert n == 0x60000001 and bad == 0


def test_fast_path_division_by_bias_corrections():
    """m/bc1 and v/bc2 through the per-CTA reciprocal == __fdiv_rn, for the
    bias corrections (glibc powf, as the table holds them) of t = 1..2000 at
    the default betas, t = 1..200 at two other beta pairs and large t, over
    all 2^24 signed significands at eight exponents of the admitted range."""
    ds = set()
    for (b1, b2), ts in (((0.9, 0.999), list(range(1, 2001)) + [10**4, 10**5, 10**6, 10**7]),
                         ((0.95, 0.999), range(1, 201)), ((0.99, 0.9999), range(1, 201))):
        for t in ts:
            ds.update(ora.step_scalars(t, b1, b2))
    divs = np.array(sorted(d for d in ds if 2.0 ** -16 <= d <= 1.0), np.float32)
    assert divs.size > 2500
    bad, n = mab.api.debug_fast_sweep(1, divs)
    assert n == divs.size << 27 and bad == 0


def test_fast_path_general_division_random():
    """mh / den through the refined reciprocal == __fdiv_rn on 2^36 random
    pairs over the admitted ranges."""
    bad, n = mab.api.debug_fast_sweep(2, samples=1 << 36, seed=12345)
    assert n == 1 << 36 and bad == 0


def test_k2_fast_path_fallback_slots_bit_exact():
    """Slots whose new m/v leave the guarded ranges (zeros, tiny and huge
    moments, subnormal gradients) recompute exactly: K2 equals the oracle
    element for element.  (NaN-producing inputs, payloads included:
    tests/test_gpu_nan.py.)"""
    n = 1 << 16
    rs = np.random.default_rng(5)
    g = (rs.standard_normal(n) * 1024).astype(f32)
    m = (rs.standard_normal(n) * 1e-3).astype(f32)
    v = np.abs(rs.standard_normal(n) * 1e-6).astype(f32)
    p = rs.standard_normal(n).astype(f32)
    sel = rs.integers(0, n, 4000)
    g[sel[:500]] = 0.0
    m[sel[:500]] = 0.0
    v[sel[:500]] = 0.0                                        # m = v = 0 exactly
    m[sel[500:1000]] = 1e-30                                  # |m| below 2^-50
    v[sel[1000:1500]] = 1e-35                                 # v below 2^-96
    m[sel[1500:2000]] = 3e17                                  # |m| above 2^50
    v[sel[2000:2500]] = 3e30                                  # v above 2^80
    g[sel[2500:2600]] = 1e-45                                 # subnormal gradients
    p[sel[2600:2700]] = 0.0
    h = ora.hyper(lr=1e-3, weight_decay=0.01)
    for t in (1, 7, 1000):
        want = [x.copy() for x in (p, m, v)]
        ora.adam_step(*want, g, t, h, 1024.0, g_kind="f32", w_kind="none")
        dp, dm, dv, dg = _dev(p, m, v, g)
        mab.adam_step_fp32(dp, dm, dv, dg, t, mab.AdamHyper(lr=1e-3, weight_decay=0.01), 1024.0)
        for a, b in zip((dp, dm, dv), want):
            assert (a.cpu().numpy().view(np.uint32) == b.view(np.uint32)).all(), t


# ------------------------------------------------------------------ K2
def _dev(*arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).to(DEV) for a in arrs]


def test_k2_known_answers(golden):
    g = golden("adam_kat.json")
    p, m, v, gr = _dev(*(np.array([x], f32) for x in (1.0, 0.0, 0.0, 1.0)))
    mab.adam_step_fp32(p, m, v, gr, 1, mab.AdamHyper(lr=0.1), 1.0)
    assert [int(host_f32(x).view(np.uint32)[0]) for x in (p, m, v)] == [g["closed_form"][k] for k in "pmv"]
    p, m, v, gr = _dev(*(np.array([x], f32) for x in (4.0, 0.0, 0.0, 0.0)))
    mab.adam_step_fp32(p, m, v, gr, 1, mab.AdamHyper(lr=0.01, weight_decay=0.1), 1.0)
    assert int(host_f32(p).view(np.uint32)[0]) == g["decay"]["p"]
    p, m, v, gr = _dev(np.array([2.5, -3.75], f32), np.zeros(2, f32), np.zeros(2, f32), np.zeros(2, f32))
    mab.adam_step_fp32(p, m, v, gr, 1, mab.AdamHyper(), 1.0)
    assert host_f32(p).tolist() == [2.5, -3.75]


def test_k2_errors():
    p, m, v, gr = _dev(*(np.zeros(4, f32) for _ in range(4)))
    with pytest.raises(mab.MemAscendError) as e:
        mab.adam_step_fp32(p, m, v, gr, 0, mab.AdamHyper(), 1.0)
    assert e.value.code == "invalid-argument"
    with pytest.raises(mab.MemAscendError):
        mab.adam_step_fp32(p, m, v, gr[:3], 1, mab.AdamHyper(), 1.0)


def test_k2_random100_golden(golden):
    """test_optimizer.cpp:61-98, bitwise per step, against the reference."""
    from kat_inputs import kat_random100_inputs

    r = golden("adam_kat.json")["random100"]
    p0, grads = kat_random100_inputs(r)
    h = mab.AdamHyper(lr=u2f(r["lr"]), weight_decay=u2f(r["wd"]))
    p, m, v = _dev(p0, np.zeros_like(p0), np.zeros_like(p0))
    for t, g in enumerate(grads, start=1):
        (gd,) = _dev(g)
        mab.adam_step_fp32(p, m, v, gd, t, h, f32(r["scale"]))
        got = np.concatenate([host_f32(p), host_f32(m), host_f32(v)])
        assert ora.fnv_hex(got) == r["per_step_pmv_fnv"][t - 1], t
    assert host_f32(p).view(np.uint32).tolist() == r["final_p"]


def _random_state(n, seed, tiny=False):
    rs = np.random.default_rng(seed)
    p = (rs.standard_normal(n) * 0.05).astype(f32)
    m = (rs.standard_normal(n) * 1e-3).astype(f32)
    v = (rs.random(n) * 1e-6).astype(f32)
    if tiny:  # exercise subnormal v / m and underflowing updates
        k = n // 7
        v[:k] = (rs.random(k) * 1e-40).astype(f32)
        m[:k] = (rs.standard_normal(k) * 1e-39).astype(f32)
    return p, m, v


@pytest.mark.parametrize("g_kind", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("w_kind", ["none", "bf16", "f16"])
@pytest.mark.parametrize("offset", [0, 1, 5])
def test_k2_vs_oracle(g_kind, w_kind, offset):
    n = 100003
    p, m, v = _random_state(n + offset, 7 + offset, tiny=True)
    rs = np.random.default_rng(11)
    gs = (rs.standard_normal(n + offset) * 300.0).astype(f32)
    gs[rs.integers(0, n + offset, 50)] = f32(1e-42)  # subnormal grads
    if g_kind == "f32":
        g_host = gs
    else:
        g_host = ora.cast_from_f32(gs, g_kind)
    h = mab.AdamHyper(lr=1e-3, weight_decay=0.01)
    for t, scale in ((1, 65536.0), (37, 1000.0), (4096, 0.5)):
        pd, md, vd = _dev(p, m, v)
        gd = _dev(g_host)[0] if g_kind == "f32" else dev_bits16(g_host)
        wd = None if w_kind == "none" else torch.zeros(n + offset, dtype=torch.int16, device=DEV)
        mab.adam_step_fp32(pd[offset:], md[offset:], vd[offset:], gd[offset:], t, h, scale,
                           w_out=None if wd is None else wd[offset:],
                           grad_kind=g_kind, w_kind=None if w_kind == "none" else w_kind)
        po, mo, vo = p[offset:].copy(), m[offset:].copy(), v[offset:].copy()
        w_or = ora.adam_step(po, mo, vo, g_host[offset:].copy(), t, ora.hyper(lr=1e-3, weight_decay=0.01),
                             scale, g_kind=g_kind, w_kind=w_kind)
        assert ulp_diff(host_f32(pd)[offset:], po) == 0
        assert ulp_diff(host_f32(md)[offset:], mo) == 0
        assert ulp_diff(host_f32(vd)[offset:], vo) == 0
        if wd is not None:
            assert (host_bits16(wd)[offset:] == w_or).all()


def test_k2_skip_flag_touches_nothing():
    n = 4097
    p, m, v = _random_state(n, 3)
    pd, md, vd, gd = _dev(p, m, v, np.ones(n, f32))
    flag = torch.ones(1, dtype=torch.int32, device=DEV)
    mab.adam_step_fp32_async(pd, md, vd, gd, 1, mab.AdamHyper(), 1.0, skip_flag=flag)
    torch.cuda.synchronize()
    assert (host_f32(pd) == p).all() and (host_f32(md) == m).all() and (host_f32(vd) == v).all()


@pytest.mark.parametrize("mode", ["pageable", "registered"])
def test_k2_host_spans(mode):
    n = (16 << 20) + 333  # crosses the 16 Mi-element staging chunk
    p, m, v = _random_state(n, 5)
    g = ora.cast_from_f32((np.random.default_rng(2).standard_normal(n) * 100).astype(f32), "bf16")
    w = np.zeros(n, np.uint16)
    hp, hm, hv, hg = p.copy(), m.copy(), v.copy(), g.copy()
    regs = [hp, hm, hv, hg, w] if mode == "registered" else []
    for a in regs:
        mab.host_register(a)
    try:
        mab.adam_step_fp32(hp, hm, hv, hg, 3, mab.AdamHyper(weight_decay=0.01), 256.0, w_out=w,
                           grad_kind="bf16", w_kind="bf16")
    finally:
        for a in regs:
            mab.host_unregister(a)
    w_or = ora.adam_step(p, m, v, g, 3, ora.hyper(weight_decay=0.01), 256.0, g_kind="bf16",
                         w_kind="bf16")
    assert (hp.view(np.uint32) == p.view(np.uint32)).all()
    assert (hm.view(np.uint32) == m.view(np.uint32)).all()
    assert (hv.view(np.uint32) == v.view(np.uint32)).all()
    assert (w == w_or).all()


def test_k3_bf16_state_vs_oracle():
    n = 65537
    rs = np.random.default_rng(9)
    p = ora.cast_from_f32((rs.standard_normal(n) * 0.5).astype(f32), "bf16")
    m = np.zeros(n, np.uint16)
    v = np.zeros(n, np.uint16)
    h = mab.AdamHyper(lr=0.05)
    pd, md, vd = dev_bits16(p), dev_bits16(m), dev_bits16(v)
    for t in range(1, 21):
        g = (rs.random(n).astype(f32) * 2 - 1).astype(f32)
        (gd,) = _dev(g)
        mab.adam_step_bf16(pd, md, vd, gd, t, h, 1.0)
        ora.adam_step_bf16(p, m, v, g, t, ora.hyper(lr=0.05), 1.0)
    assert (host_bits16(pd) == p).all() and (host_bits16(md) == m).all() and (host_bits16(vd) == v).all()


# ------------------------------------------------------------------ full step
W_DT = {"bf16": torch.bfloat16, "f16": torch.float16}
G_DT = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}


def run_workload_on_gpu(n, steps, seed, g_kind, w_kind, subgroup, hyper, init_scale, growth,
                        faults, per_step_cb=None):
    p = torch.empty(n, dtype=torch.float32, device=DEV)
    m = torch.zeros(n, dtype=torch.float32, device=DEV)
    v = torch.zeros(n, dtype=torch.float32, device=DEV)
    w = torch.empty(n, dtype=W_DT[w_kind], device=DEV)
    g = torch.empty(n, dtype=G_DT[g_kind], device=DEV)
    mab.gen_seeded_weights(p, w, seed=seed)
    st = mab.Stepper(hyper, init_scale, growth, g_kind, w_kind)
    groups = [(p[o:o + subgroup], m[o:o + subgroup], v[o:o + subgroup], g[o:o + subgroup],
               w[o:o + subgroup]) for o in range(0, n, subgroup)]
    for s in range(steps):
        mab.gen_pseudo_grads(g, w, step=s, seed=seed, d_scale=st.scale_t)
        for fs, idx, bits in faults:
            if fs == s:
                mab.plant_bits(g, idx % n, bits)
        grads_fnv = fnv(g) if per_step_cb else None
        st.check(g)
        st.apply(groups)
        st.finish()
        if per_step_cb:
            per_step_cb(s, st, p, m, v, w, grads_fnv)
    return st, p, m, v, w


def test_stepper_workload_golden(golden):
    """The configs' workload end to end through the C ABI, per step, vs the
    reference's own composition (workload.json)."""
    for c in golden("workload.json")["cases"]:
        hyper = mab.AdamHyper(lr=u2f(c["lr"]), beta1=u2f(c["beta1"]), beta2=u2f(c["beta2"]),
                              eps=u2f(c["eps"]), weight_decay=u2f(c["wd"]))
        faults = [(f["step"], f["index"], f["bits"]) for f in c["faults"]]

        def cb(s, st, p, m, v, w, grads_fnv, c=c):
            want = c["per_step"][s]
            assert grads_fnv == want["grads_fnv"], (c["name"], s)
            state = st.state()
            assert bool(state["last_overflow"]) == want["overflow"], (c["name"], s)
            assert state["scale"] == want["scale_after"]
            for k, t in (("p", p), ("m", m), ("v", v), ("w", w)):
                assert fnv(t) == want[f"{k}_fnv"], (c["name"], s, k)

        st, *_ = run_workload_on_gpu(c["n"], c["steps"], c["seed"], c["g_kind"], c["w_kind"],
                                     c["subgroup"], hyper, c["init_scale"], c["growth_interval"],
                                     faults, cb)
        of, sc = st.history()
        assert of.tolist() == [s["overflow"] for s in c["per_step"]]
        assert sc.tolist() == [s["scale_after"] for s in c["per_step"]]
        assert st.state()["updates"] == c["updates"]


def test_stepper_toy_dense_digests(golden):
    """test_simulator.cpp:35-89: the reference simulator's digests (mixed mode:
    fp32 flat grads, fp16 shadows) reproduced on the GPU."""
    t = golden("trainer.json")
    for c in t["cases"]:
        if c["pure_bf16"]:
            continue
        faults = []
        if c["fault"]:
            faults = [(c["fault"]["step"], c["fault"]["index"], c["fault"]["bits"])]
        st, p, *_ = run_workload_on_gpu(t["n"], c["steps"], c["seed"], "f32", "f16", 1 << 30,
                                        mab.AdamHyper(), 65536.0, 2000, faults)
        assert fnv(p) == c["sim_digest"], c["name"]
        of, sc = st.history()
        assert np.nonzero(of)[0].tolist() == c["overflow_steps"]
        assert sc.tolist() == c["scale_after"]


def test_full_size_sampled_parity():
    """A 2^28+3 element partition (100M-element sub-groups), 4 steps with an
    injected NaN: decisions exact, and a random sample of 200k elements
    bit-exact against the oracle's elementwise replay."""
    n, steps, seed = (1 << 28) + 3, 4, 1
    faults = [(2, 123456789, 0x7FC1)]
    st, p, m, v, w = run_workload_on_gpu(n, steps, seed, "bf16", "bf16", 100_000_000,
                                         mab.AdamHyper(weight_decay=0.01), 65536.0, 2000, faults)
    of, _ = st.history()
    assert of.tolist() == [False, False, True, False]
    rs = np.random.default_rng(0)
    idx = np.unique(np.concatenate([rs.integers(0, n, 200_000), [0, 1, n - 1, 123456789]]))
    smp = ora.train_sample(idx, of.astype(np.uint8), steps, seed, g_kind="bf16", w_kind="bf16",
                           hyp=ora.hyper(weight_decay=0.01))
    it = torch.from_numpy(idx.astype(np.int64)).to(DEV)
    assert (host_f32(p[it]).view(np.uint32) == smp["p"].view(np.uint32)).all()
    assert (host_f32(m[it]).view(np.uint32) == smp["m"].view(np.uint32)).all()
    assert (host_f32(v[it]).view(np.uint32) == smp["v"].view(np.uint32)).all()
    assert (host_bits16(w[it]) == smp["w"]).all()


@pytest.mark.parametrize("slots,slot_elems", [(2, 8192), (3, 30000), (2, 1 << 20)])
def test_streamed_apply_workload_golden(golden, slots, slot_elems):
    """Configs 4/5 path: p/m/v in the registered host pool, sub-group slices
    staged H2D -> K2 -> D2H through device slots; per step vs the reference."""
    c = next(x for x in golden("workload.json")["cases"] if x["name"] == "cfg_bf16_n100003")
    n, sub, seed = c["n"], c["subgroup"], c["seed"]
    hyper = mab.AdamHyper(lr=u2f(c["lr"]), beta1=u2f(c["beta1"]), beta2=u2f(c["beta2"]),
                          eps=u2f(c["eps"]), weight_decay=u2f(c["wd"]))
    p = torch.empty(n, dtype=torch.float32, pin_memory=True)
    m = torch.zeros(n, dtype=torch.float32, pin_memory=True)
    v = torch.zeros(n, dtype=torch.float32, pin_memory=True)
    pd = torch.empty(n, dtype=torch.float32, device=DEV)
    w = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    g = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    mab.gen_seeded_weights(pd, w, seed=seed)
    p.copy_(pd)
    assert mab.pointer_kind(p) == 2
    st = mab.Stepper(hyper, c["init_scale"], c["growth_interval"], "bf16", "bf16")
    groups = [(p[o:o + sub], m[o:o + sub], v[o:o + sub], g[o:o + sub], w[o:o + sub])
              for o in range(0, n, sub)]
    staging = torch.empty(3 * slots * slot_elems, dtype=torch.float32, device=DEV)
    for s, want in enumerate(c["per_step"]):
        mab.gen_pseudo_grads(g, w, step=s, seed=seed, d_scale=st.scale_t)
        for f in c["faults"]:
            if f["step"] == s:
                mab.plant_bits(g, f["index"] % n, f["bits"])
        st.check(g)
        skipped = st.apply_streamed(groups, staging, slot_elems, slots)
        st.finish()
        torch.cuda.synchronize()
        assert skipped == want["overflow"]
        for k, t in (("p", p), ("m", m), ("v", v), ("w", w)):
            assert fnv(t) == want[f"{k}_fnv"], (s, k)


@pytest.mark.parametrize("sub", [1 << 30, 10007])
def test_stepper_pure_bf16_digest(golden, sub):
    """test_simulator.cpp:44-51: the pure-bf16 run (bf16 weights/m/v, fp32 flat
    grads) through K3 and the device-resident scaler, vs the reference digest."""
    t = golden("trainer.json")
    c = next(x for x in t["cases"] if x["pure_bf16"])
    n, seed = t["n"], c["seed"]
    w = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    m = torch.zeros(n, dtype=torch.int16, device=DEV)
    v = torch.zeros(n, dtype=torch.int16, device=DEV)
    g = torch.empty(n, dtype=torch.float32, device=DEV)
    mab.gen_seeded_weights(None, w, n=n, seed=seed)
    st = mab.Stepper(mab.AdamHyper(), 65536.0, 2000, "f32", "none")
    groups = [(w[o:o + sub], m[o:o + sub], v[o:o + sub], g[o:o + sub]) for o in range(0, n, sub)]
    for s in range(c["steps"]):
        mab.gen_pseudo_grads(g, w, step=s, seed=seed, d_scale=st.scale_t)
        st.check(g)
        st.apply_bf16(groups)
        st.finish()
    torch.cuda.synchronize()
    assert fnv(w) == c["sim_digest"]
    assert st.state()["scale"] == c["final_scale"]


def test_stepper_ingest_fused_check(golden):
    """§8(f) row 2: raw (unscaled) gradients scaled into the flat buffer with
    the overflow test fused into that store; no separate K1.  Decisions and
    the p/m/v/w trajectory must equal the reference composition."""
    c = next(x for x in golden("workload.json")["cases"] if x["name"] == "cfg_bf16_n100003")
    n, sub, seed = c["n"], c["subgroup"], c["seed"]
    hyper = mab.AdamHyper(lr=u2f(c["lr"]), beta1=u2f(c["beta1"]), beta2=u2f(c["beta2"]),
                          eps=u2f(c["eps"]), weight_decay=u2f(c["wd"]))
    p = torch.empty(n, dtype=torch.float32, device=DEV)
    m = torch.zeros(n, dtype=torch.float32, device=DEV)
    v = torch.zeros(n, dtype=torch.float32, device=DEV)
    w = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    g = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    raw = torch.empty(n, dtype=torch.float32, device=DEV)
    mab.gen_seeded_weights(p, w, seed=seed)
    st = mab.Stepper(hyper, c["init_scale"], c["growth_interval"], "bf16", "bf16")
    groups = [(p[o:o + sub], m[o:o + sub], v[o:o + sub], g[o:o + sub], w[o:o + sub])
              for o in range(0, n, sub)]
    for s, want in enumerate(c["per_step"]):
        mab.gen_pseudo_grads(raw, w, step=s, seed=seed, scale=1.0)  # the producer's raw grads
        mine = [f for f in c["faults"] if f["step"] == s]
        for f in mine:
            if (f["bits"] & 0x7F80) == 0x7F80:  # inf/NaN: planted in the source, stays non-finite
                mab.plant_bits(raw, f["index"] % n, f["bits"] << 16)
        st.ingest(raw, g)
        for f in mine:
            if (f["bits"] & 0x7F80) != 0x7F80:  # finite control: lands in the flat buffer as-is
                mab.plant_bits(g, f["index"] % n, f["bits"])
        st.apply(groups)
        st.finish()
        torch.cuda.synchronize()
        assert bool(st.state()["last_overflow"]) == want["overflow"], s
        if not want["overflow"]:
            assert fnv(g) == want["grads_fnv"], s
        for k, t in (("p", p), ("m", m), ("v", v), ("w", w)):
            assert fnv(t) == want[f"{k}_fnv"], (s, k)


def test_cfg2_full_size_sampled_parity():
    """BASELINE configs[1] at its full size: 8,030,261,248 params on one B200
    (81 sub-groups of 100M), 3 steps with a NaN planted past 2^32 at step 1.
    Decisions exact; 100k random elements plus the 2^32 boundary bit-exact
    against the oracle's elementwise replay."""
    torch.cuda.empty_cache()
    n, steps, seed = 8_030_261_248, 3, 1
    if torch.cuda.mem_get_info()[0] < n * 16 + (2 << 30):
        pytest.skip("needs 130 GB of free HBM")
    faults = [(1, (1 << 32) + 12345, 0x7FC0)]
    st, p, m, v, w = run_workload_on_gpu(n, steps, seed, "bf16", "bf16", 100_000_000,
                                         mab.AdamHyper(weight_decay=0.01), 65536.0, 2000, faults)
    of, _ = st.history()
    assert of.tolist() == [False, True, False]
    rs = np.random.default_rng(1)
    edge = [0, (1 << 31) - 1, 1 << 31, (1 << 32) - 1, 1 << 32, (1 << 32) + 1, n - 1,
            99_999_999, 100_000_000]
    idx = np.unique(np.concatenate([rs.integers(0, n, 100_000), edge]).astype(np.uint64))
    smp = ora.train_sample(idx, of.astype(np.uint8), steps, seed, g_kind="bf16", w_kind="bf16",
                           hyp=ora.hyper(weight_decay=0.01))
    it = torch.from_numpy(idx.astype(np.int64)).to(DEV)
    assert (host_f32(p[it]).view(np.uint32) == smp["p"].view(np.uint32)).all()
    assert (host_f32(m[it]).view(np.uint32) == smp["m"].view(np.uint32)).all()
    assert (host_f32(v[it]).view(np.uint32) == smp["v"].view(np.uint32)).all()
    assert (host_bits16(w[it]) == smp["w"]).all()
    del p, m, v, w, st
    torch.cuda.empty_cache()


def test_cfg2_full_size_pure_bf16_sampled_parity():
    """The pure-bf16 mode (OptimPrecision::pure_bf16, simulator.cpp:470-486)
    on configs[1]'s full partition — the `bench.py --precision pure_bf16`
    workload: 8,030,261,248 bf16 weights / m / v in HBM, 81 sub-groups, bf16
    gradients, K1 -> K3 -> scaler, a NaN planted past 2^32 at step 1, scale
    growth every 2 clean steps.  Decisions exact; 100k random elements plus
    the 2^32 / sub-group boundaries bit-exact against the oracle's
    elementwise replay."""
    torch.cuda.empty_cache()
    n, steps, seed, sub = 8_030_261_248, 4, 1, 100_000_000
    if torch.cuda.mem_get_info()[0] < n * 8 + (2 << 30):
        pytest.skip("needs 66 GB of free HBM")
    w = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    m = torch.zeros(n, dtype=torch.bfloat16, device=DEV)
    v = torch.zeros(n, dtype=torch.bfloat16, device=DEV)
    g = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    mab.gen_seeded_weights(None, w, seed=seed)
    h = mab.AdamHyper(weight_decay=0.01)
    st = mab.Stepper(h, 65536.0, 2, "bf16", "bf16")
    groups = [(w[o:o + sub], m[o:o + sub], v[o:o + sub], g[o:o + sub]) for o in range(0, n, sub)]
    for s in range(steps):
        mab.gen_pseudo_grads(g, w, step=s, seed=seed, d_scale=st.scale_t)
        if s == 1:
            mab.plant_bits(g, (1 << 32) + 12345, 0x7FC0)
        st.check(g)
        st.apply_bf16(groups)
        st.finish()
    torch.cuda.synchronize()
    of, sc = st.history()
    assert of.tolist() == [False, True, False, False]
    assert sc.tolist() == [65536.0, 32768.0, 32768.0, 65536.0]
    rs = np.random.default_rng(2)
    edge = [0, (1 << 31) - 1, 1 << 31, (1 << 32) - 1, 1 << 32, (1 << 32) + 1, (1 << 32) + 12345,
            n - 1, 99_999_999, 100_000_000]
    idx = np.unique(np.concatenate([rs.integers(0, n, 100_000), edge]).astype(np.uint64))
    smp = ora.train_sample(idx, of.astype(np.uint8), steps, seed, g_kind="bf16", w_kind="bf16",
                           hyp=ora.hyper(weight_decay=0.01), growth=2, mixed=False)
    it = torch.from_numpy(idx.astype(np.int64)).to(DEV)
    top = lambda x: (x.view(np.uint32) >> 16).astype(np.uint16)  # noqa: E731
    assert (host_bits16(w[it]) == smp["w"]).all()
    assert (host_bits16(m[it]) == top(smp["m"])).all()
    assert (host_bits16(v[it]) == top(smp["v"])).all()
    del w, m, v, g, st
    torch.cuda.empty_cache()


def test_empty_inputs():
    """n == 0 everywhere the reference accepts it: fused_overflow_check
    returns no overflow (overflow.cpp:77-79); adam_step_fp32 / _bf16 are
    no-ops but still reject t == 0 (optimizer.cpp:49-51); a stepper step over
    an empty partition is a clean step (t advances, the scaler counts it)."""
    for kind, dt in (("f32", torch.float32), ("bf16", torch.bfloat16), ("f16", torch.float16)):
        e = torch.empty(0, dtype=dt, device=DEV)
        r = mab.fused_overflow_check(e, track_first_index=True, kind=kind)
        assert r.overflow is False and r.first_offending_index is None
    z = torch.empty(0, dtype=torch.float32, device=DEV)
    z16 = torch.empty(0, dtype=torch.int16, device=DEV)
    mab.adam_step_fp32(z, z.clone(), z.clone(), z.clone(), 1, mab.AdamHyper(), 65536.0)
    mab.adam_step_fp32(z, z.clone(), z.clone(), z16.view(torch.bfloat16), 3, mab.AdamHyper(),
                       65536.0, w_out=z16.clone(), grad_kind="bf16", w_kind="bf16")
    with pytest.raises(mab.MemAscendError):
        mab.adam_step_fp32(z, z.clone(), z.clone(), z.clone(), 0, mab.AdamHyper(), 1.0)
    mab.adam_step_bf16(z16, z16.clone(), z16.clone(), z, 1, mab.AdamHyper(), 1.0)
    with pytest.raises(mab.MemAscendError):
        mab.adam_step_bf16(z16, z16.clone(), z16.clone(), z, 0, mab.AdamHyper(), 1.0)
    st = mab.Stepper(mab.AdamHyper(), 1024.0, 2, "bf16", "bf16")
    g = torch.empty(0, dtype=torch.bfloat16, device=DEV)
    for _ in range(3):
        st.check(g)
        st.ingest(torch.empty(0, dtype=torch.float32, device=DEV), g)   # producer-side check
        st.reduce_check([g, g.clone()], g.clone())                       # K4
        st.apply([])
        st.apply_bf16([])
        st.finish()
    torch.cuda.synchronize()
    s = st.state()
    assert s["updates"] == 3 and s["last_overflow"] == 0 and s["scale"] == 2048.0
    st.close()

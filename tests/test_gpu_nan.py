"""NaN parity: the B200 kernels against the UNMODIFIED reference (oracle/_ref)
when the optimizer state goes non-finite.

The reference computes on x86 SSE; its NaN results follow the operand order
of its compiled adam_range (pinned in tests/test_nan_semantics.py).  The
kernels' exact path reproduces that rule per operation, so p / m / v and the
cast working weights are equal BIT FOR BIT, NaN payloads included:

  * adversarial state (NaN payloads in every operand, infinities, signed
    zeros, subnormals, negative variance) under every loss-scale / eps case
    of tests/nan_inputs.py, through K2 (every working-weight kind) and K3;
  * repeated overflows push the device-resident loss scale
    below 1, after which FINITE scaled gradients overflow when unscaled —
    the step is not skipped (the check tests the stored gradients), m and v
    become infinite and p NaN, and the NaN state then propagates for several
    more steps;
  * eps = 0 with v = 0: 0/0 in mh / den;
  * the offloaded pipelines (configs[3] streamed from registered host memory,
    configs[4] through the O_DIRECT swap store) with non-finite and cold
    state: what lands back in host memory / the store equals the reference.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import nan_inputs as ni  # noqa: E402
import paper_2505_23254_b200 as mab  # noqa: E402
from oracle import oracle as ora  # noqa: E402

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ora.ref_available(), reason="oracle/_ref not built")]
DEV = "cuda:0"


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).copy()).to(DEV)


def u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("scale,eps", ni.CASES)
@pytest.mark.parametrize("w_kind", ["bf16", "f16"])
def test_k2_adversarial_state_equals_reference(scale, eps, w_kind):
    n = 50021
    p, m, v, g = ni.state(11 + int(scale * 100), n)
    h = ora.hyper(lr=1e-3, eps=eps, weight_decay=0.01)
    ref = [x.copy() for x in (p, m, v)]
    d = [dev(x) for x in (p, m, v)]
    dg = dev(g)
    w = torch.zeros(n, dtype=torch.int16, device=DEV)
    for t in range(1, 5):
        ora.ref_adam_step_fp32(*ref, g, t, h, scale, workers=4)
        mab.adam_step_fp32(d[0], d[1], d[2], dg, t, mab.AdamHyper(lr=1e-3, eps=eps,
                                                                   weight_decay=0.01),
                           scale, w_out=w, w_kind=w_kind)
        for got, want, name in zip(d, ref, "pmv"):
            diff = np.flatnonzero(u32(got) != want.view(np.uint32))
            assert diff.size == 0, (t, name, [(hex(u32(got)[i]), hex(want.view(np.uint32)[i]))
                                              for i in diff[:4]])
        assert np.array_equal(w.cpu().numpy().view(np.uint16), ora.cast_from_f32(ref[0], w_kind))
    assert np.isnan(ref[0]).sum() > n // 4


@pytest.mark.parametrize("scale,eps", ni.CASES)
def test_k3_adversarial_state_equals_reference(scale, eps):
    n = 50021
    p, m, v, g = ni.state(23 + int(scale * 100), n)
    h = ora.hyper(lr=1e-3, eps=eps, weight_decay=0.01)
    ref = [ni.bf16_bits(x) for x in (p, m, v)]
    d = [dev(x.view(np.int16)) for x in ref]
    dg = dev(g)
    hv = ora.ref_hyper_array(h)
    for t in range(1, 5):
        assert ora.ref().ref_adam_step_bf16(*(ora._ptr(x) for x in ref), ora._ptr(g), n, t,
                                            ora._ptr(hv), scale, 4) == 0
        mab.adam_step_bf16(d[0], d[1], d[2], dg, t,
                           mab.AdamHyper(lr=1e-3, eps=eps, weight_decay=0.01), scale)
        for got, want, name in zip(d, ref, "pmv"):
            assert np.array_equal(got.cpu().numpy().view(np.uint16), want), (t, name)


def _reference_steps(p, m, v, grads16, h, scale, growth):
    """The reference step composition (simulator.cpp:431-469) with the
    reference's own functions: one check of the stored bf16 gradients
    (fused_overflow_check over their fp32 widening), skip = halve the scale,
    else t += 1, adam_step_fp32 with the current scale, bf16 cast-back,
    LossScaler.  Returns per-step (skipped, scale_after) and the final w."""
    out, t, clean = [], 0, 0
    w = None
    for g16 in grads16:
        g = ora.widen(g16, "bf16")
        of, _ = ora.ref_fused_overflow_check(g)
        if of:
            scale *= np.float32(0.5)
            clean = 0
        else:
            t += 1
            ora.ref_adam_step_fp32(p, m, v, g, t, h, scale)
            w = ora.cast_from_f32(p, "bf16")
            clean += 1
            if clean >= growth:
                scale *= np.float32(2.0)
                clean = 0
        out.append((bool(of), float(scale)))
    return out, w


def test_scale_below_one_overflow_after_unscale():
    """SURVEY §7 item 6 through the device step driver: four injected +inf
    steps halve the scale 4 -> 0.25; then finite bf16 gradients near the
    bf16 maximum become infinite once divided by the scale, so m, v = inf and
    p = NaN (inf/inf in mh/den) on the reference; the NaN state is carried
    for four more steps.  Decisions, scales, p/m/v and the bf16 working
    weights equal the reference bit for bit."""
    n = 40009
    rng = np.random.default_rng(3)
    p0 = (rng.standard_normal(n) * 0.1).astype(np.float32)
    grads = []
    for s in range(10):
        g = rng.standard_normal(n).astype(np.float32) * 1e-3
        if s < 4:
            g[rng.integers(0, n)] = np.inf                      # overflow: skip, halve
        else:
            big = rng.integers(0, n, 3000)
            g[big] = rng.choice([-1, 1], big.size) * rng.uniform(5e37, 3.3e38, big.size)
        grads.append(ora.cast_from_f32(g, "bf16"))
    h = ora.hyper(lr=1e-3, weight_decay=0.01)
    ref = [p0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)]
    want, w_ref = _reference_steps(*ref, grads, h, np.float32(4.0), 2000)
    assert [s for s, _ in want] == [True] * 4 + [False] * 6
    assert want[3][1] == 0.25 and np.isnan(ref[0]).sum() > 1000

    st = mab.Stepper(mab.AdamHyper(lr=1e-3, weight_decay=0.01), 4.0, 2000, "bf16", "bf16")
    p, m, v = dev(p0), torch.zeros(n, device=DEV), torch.zeros(n, device=DEV)
    w = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    gd = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    groups = [(p[o:o + 10007], m[o:o + 10007], v[o:o + 10007], gd[o:o + 10007],
               w[o:o + 10007]) for o in range(0, n, 10007)]
    for g16 in grads:
        gd.view(torch.int16).copy_(torch.from_numpy(g16.view(np.int16)))
        st.step([gd], groups)
    of, sc = st.history()
    assert [(bool(a), float(b)) for a, b in zip(of, sc)] == want
    for got, exp, name in zip((p, m, v), ref, "pmv"):
        assert np.array_equal(u32(got), exp.view(np.uint32)), name
    assert np.array_equal(w.view(torch.int16).cpu().numpy().view(np.uint16), w_ref)
    st.close()


def test_eps_zero_zero_variance():
    """eps = 0, v = 0, g = 0 (and m = 0): 0/0 -> x86's default NaN 0xFFC00000
    in p on the reference, the same on the GPU (the canonical GPU NaN would be
    0x7FFFFFFF); the fp16 working weight is the reference's sign|0x7E00."""
    n = 4099
    p = np.linspace(-1, 1, n).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    g = np.zeros(n, np.float32)
    g[::3] = 1.0  # every third element takes the ordinary path
    h = ora.hyper(lr=1e-3, eps=0.0)
    ref = [p.copy(), m.copy(), v.copy()]
    ora.ref_adam_step_fp32(*ref, g, 1, h, 1.0)
    assert (ref[0].view(np.uint32)[1::3] == 0xFFC00000).all()
    d = [dev(x) for x in (p, m, v)]
    w = torch.zeros(n, dtype=torch.int16, device=DEV)
    mab.adam_step_fp32(d[0], d[1], d[2], dev(g), 1, mab.AdamHyper(lr=1e-3, eps=0.0), 1.0,
                       w_out=w, w_kind="f16")
    for got, exp in zip(d, ref):
        assert np.array_equal(u32(got), exp.view(np.uint32))
    assert np.array_equal(w.cpu().numpy().view(np.uint16), ora.cast_from_f32(ref[0], "f16"))
    assert (w.cpu().numpy().view(np.uint16)[1::3] == 0xFE00).all()


def _adversarial_state_finite_grads(seed, n):
    """Adversarial p/m/v (NaN payloads, infinities, negative v, cold zeros)
    with FINITE gradients, so the step is not skipped and the non-finite
    values reach K2 inside the offloaded pipelines."""
    p, m, v, _ = ni.state(seed, n, p_special=0.3)
    rng = np.random.default_rng(seed + 1)
    g = (rng.standard_normal(n) * 1024).astype(np.float32)
    g[rng.random(n) < 0.2] = 0.0
    return p, m, v, ora.cast_from_f32(g, "bf16")


@pytest.mark.parametrize("slots,slot_elems", [(2, 8192), (3, 30000)])
def test_streamed_path_adversarial_state_equals_reference(slots, slot_elems):
    """configs[3]'s path (p/m/v in registered host memory, staged through
    device slots) with non-finite / cold state: p/m/v and the bf16 working
    weights equal the reference bit for bit."""
    n, sub = 70_001, 30_000
    p, m, v, g16 = _adversarial_state_finite_grads(5, n)
    h = ora.hyper(lr=1e-3, weight_decay=0.01)
    ref = [x.copy() for x in (p, m, v)]
    ora.ref_adam_step_fp32(*ref, ora.widen(g16, "bf16"), 1, h, 65536.0)
    host = [torch.from_numpy(x.copy()).pin_memory() for x in (p, m, v)]
    gd = torch.from_numpy(g16.view(np.int16)).to(DEV).view(torch.bfloat16)
    w = torch.zeros(n, dtype=torch.bfloat16, device=DEV)
    st = mab.Stepper(mab.AdamHyper(lr=1e-3, weight_decay=0.01), 65536.0, 2000, "bf16", "bf16")
    groups = [(host[0][o:o + sub], host[1][o:o + sub], host[2][o:o + sub], gd[o:o + sub],
               w[o:o + sub]) for o in range(0, n, sub)]
    staging = torch.empty(3 * slots * slot_elems, dtype=torch.float32, device=DEV)
    assert not st.apply_streamed(groups, staging, slot_elems, slots)
    st.finish()
    torch.cuda.synchronize()
    for got, want, name in zip(host, ref, "pmv"):
        assert np.array_equal(got.numpy().view(np.uint32), want.view(np.uint32)), name
    assert np.array_equal(w.view(torch.int16).cpu().numpy().view(np.uint16),
                          ora.cast_from_f32(ref[0], "bf16"))


def test_swapped_path_adversarial_state_equals_reference(tmp_path):
    """configs[4]'s path (master/m/v in the O_DIRECT swap store, read ahead
    into registered host slots, through HBM, written back) with non-finite /
    cold state: what the store holds afterwards equals the reference."""
    n, sub, slot = 50_003, 20_000, 20_480
    p, m, v, g16 = _adversarial_state_finite_grads(9, n)
    h = ora.hyper(lr=1e-3, weight_decay=0.01)
    ref = [x.copy() for x in (p, m, v)]
    ora.ref_adam_step_fp32(*ref, ora.widen(g16, "bf16"), 1, h, 65536.0)
    store = mab.DirectIoEngine(mab.DirectIoEngine.create_virtual_devices(str(tmp_path), 2,
                                                                         8 << 20))
    buf = mab.aligned_host_buffer(slot * 4)
    gd = torch.from_numpy(g16.view(np.int16)).to(DEV).view(torch.bfloat16)
    w = torch.zeros(n, dtype=torch.bfloat16, device=DEV)
    groups = []
    for k, o in enumerate(range(0, n, sub)):
        ln = min(sub, n - o)
        keys = tuple(f"{t}.g{k}" for t in ("master", "m", "v"))
        for key, arr in zip(keys, (p, m, v)):
            buf.view(np.float32)[:ln] = arr[o:o + ln]
            store.write_tensor(key, buf, ln * 4)
        groups.append((keys, gd[o:o + ln], w[o:o + ln]))
    hstage = mab.aligned_host_buffer(2 * 3 * slot * 4, register=True)
    dstage = torch.empty(3 * 2 * slot, dtype=torch.float32, device=DEV)
    st = mab.Stepper(mab.AdamHyper(lr=1e-3, weight_decay=0.01), 65536.0, 2000, "bf16", "bf16")
    assert not st.apply_swapped(store, groups, hstage, 2, dstage, 2, slot)
    st.finish()
    torch.cuda.synchronize()
    for k, o in enumerate(range(0, n, sub)):
        ln = min(sub, n - o)
        for key, want, name in zip(groups[k][0], ref, "pmv"):
            store.read_tensor(key, buf)
            got = buf.view(np.float32)[:ln]
            assert np.array_equal(got.view(np.uint32), want[o:o + ln].view(np.uint32)), (k, name)
    assert np.array_equal(w.view(torch.int16).cpu().numpy().view(np.uint16),
                          ora.cast_from_f32(ref[0], "bf16"))
    store.close()

"""Cold parameters — no gradient for a while, or never — stay exact AND fast.

Elements with m = v = g = 0 (parameters that never received a gradient,
e.g. embedding rows no batch touched) or with moments decayed below the
fast path's 2^-50 bound take the cheap exact shortcuts of adam_cold
(ma_device.cuh) instead of the full IEEE / x86 sequence.  Checked bit for
bit against the UNMODIFIED reference (oracle/_ref) for K2 (fp32 state, bf16
and fp16 working weights) and K3 (bf16 state): signed zeros in every
operand, |m| from 2^-110 to 2^-45 over normal and huge variances (huge v
makes q = mh / den subnormal, which must fall back), several t, with and
without weight decay, scattered among ordinary elements.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2505_23254_b200 as mab  # noqa: E402
from oracle import oracle as ora  # noqa: E402

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ora.ref_available(), reason="oracle/_ref not built")]
f32 = np.float32


def cold_state(seed, n):
    rng = np.random.default_rng(seed)
    p = (rng.standard_normal(n) * 0.1).astype(f32)
    m = (rng.standard_normal(n) * 1e-3).astype(f32)
    v = (np.abs(rng.standard_normal(n)) * 1e-6).astype(f32)
    g = (rng.standard_normal(n) * 1024).astype(f32)
    cat = rng.integers(0, 6, n)
    z = cat == 0                                  # never touched: signed zeros
    sgn = lambda k: np.where(rng.integers(0, 2, k) == 0, f32(0.0), f32(-0.0))  # noqa: E731
    m[z], v[z], g[z] = sgn(z.sum()), np.zeros(z.sum(), f32), sgn(z.sum())
    d = cat == 1                                  # decayed: tiny m, ordinary v, g = 0
    m[d] = (rng.choice([-1, 1], d.sum()) * np.exp2(rng.uniform(-110, -45, d.sum()))).astype(f32)
    g[d] = 0
    h = cat == 2                                  # decayed m, huge v: q may be subnormal
    m[h] = (rng.choice([-1, 1], h.sum()) * np.exp2(rng.uniform(-110, -60, h.sum()))).astype(f32)
    v[h] = np.exp2(rng.uniform(40, 79, h.sum())).astype(f32)
    g[h] = 0
    zv = cat == 3                                 # m = 0 with v > 0 (g = 0)
    m[zv], g[zv] = sgn(zv.sum()), sgn(zv.sum())
    pz = (cat == 4) & (rng.random(n) < 0.5)       # zero p among cold elements
    p[pz] = sgn(pz.sum())
    m[pz], v[pz], g[pz] = 0, 0, 0
    return p, m, v, g


@pytest.mark.parametrize("t,wd", [(1, 0.0), (7, 0.01), (1000, 0.1)])
@pytest.mark.parametrize("w_kind", ["bf16", "f16"])
def test_k2_cold_elements_equal_reference(t, wd, w_kind):
    n = 100_003
    p, m, v, g = cold_state(t + int(wd * 100), n)
    h = ora.hyper(lr=1e-3, weight_decay=wd)
    ref = [x.copy() for x in (p, m, v)]
    ora.ref_adam_step_fp32(*ref, g, t, h, 65536.0)
    d = [torch.from_numpy(x.copy()).cuda() for x in (p, m, v, g)]
    w = torch.zeros(n, dtype=torch.int16, device="cuda")
    mab.adam_step_fp32(*d, t, mab.AdamHyper(lr=1e-3, weight_decay=wd), 65536.0, w_out=w,
                       w_kind=w_kind)
    for got, want, name in zip(d, ref, "pmv"):
        a = got.cpu().numpy().view(np.uint32)
        bad = np.flatnonzero(a != want.view(np.uint32))
        assert bad.size == 0, (name, [(hex(a[i]), hex(want.view(np.uint32)[i])) for i in bad[:4]])
    assert np.array_equal(w.cpu().numpy().view(np.uint16), ora.cast_from_f32(ref[0], w_kind))


@pytest.mark.parametrize("t", [1, 50])
def test_k3_cold_elements_equal_reference(t):
    n = 100_003
    p, m, v, g = cold_state(100 + t, n)
    b = [(x.view(np.uint32) >> 16).astype(np.uint16) for x in (p, m, v)]
    h = ora.hyper(lr=1e-3, weight_decay=0.01)
    hv = ora.ref_hyper_array(h)
    ref = [x.copy() for x in b]
    assert ora.ref().ref_adam_step_bf16(*(ora._ptr(x) for x in ref), ora._ptr(g), n, t,
                                        ora._ptr(hv), 65536.0, 1) == 0
    d = [torch.from_numpy(x.view(np.int16).copy()).cuda() for x in b]
    mab.adam_step_bf16(*d, torch.from_numpy(g).cuda(), t,
                       mab.AdamHyper(lr=1e-3, weight_decay=0.01), 65536.0)
    for got, want in zip(d, ref):
        assert np.array_equal(got.cpu().numpy().view(np.uint16), want)


@pytest.mark.parametrize("kernel", ["k2", "k3"])
def test_cold_rows_over_120_steps_equal_oracle(kernel):
    """An embedding-like table of 256 rows x 4096 over 120 steps: some rows
    never receive a gradient (m = v = 0 throughout), some only in the first
    step (their momentum decays through 2^-50 into the decayed-moment
    shortcut: beta1 = 0.5), the rest at random half of the steps.  State
    equal to the oracle (the reference's arithmetic) bit for bit at every
    10th step and at the end."""
    rows, cols, steps = 256, 4096, 120
    n = rows * cols
    rng = np.random.default_rng(11)
    kind = rng.integers(0, 3, rows)           # 0 never, 1 first step only, 2 intermittent
    h = ora.hyper(lr=1e-3, beta1=0.5, beta2=0.999, weight_decay=0.01)
    hd = mab.AdamHyper(lr=1e-3, beta1=0.5, beta2=0.999, weight_decay=0.01)
    p0 = (rng.standard_normal(n) * 0.1).astype(f32)
    if kernel == "k2":
        ref = [p0.copy(), np.zeros(n, f32), np.zeros(n, f32)]
        d = [torch.from_numpy(x.copy()).cuda() for x in ref]
    else:
        ref = [(p0.view(np.uint32) >> 16).astype(np.uint16), np.zeros(n, np.uint16),
               np.zeros(n, np.uint16)]
        d = [torch.from_numpy(x.view(np.int16).copy()).cuda() for x in ref]
    for t in range(1, steps + 1):
        live = np.where(kind == 2, rng.random(rows) < 0.5, (kind == 1) & (t == 1))
        g = (rng.standard_normal(n) * 64).astype(f32) * np.repeat(live, cols).astype(f32)
        gd = torch.from_numpy(g).cuda()
        if kernel == "k2":
            ora.adam_step(*ref, g, t, h, 65536.0)
            mab.adam_step_fp32(*d, gd, t, hd, 65536.0)
        else:
            ora.adam_step_bf16(*ref, g, t, h, 65536.0)
            mab.adam_step_bf16(*d, gd, t, hd, 65536.0)
        if t % 10 == 0 or t == steps:
            for got, want, name in zip(d, ref, "pmv"):
                a = got.cpu().numpy().view(want.dtype)
                assert np.array_equal(a, want), (t, name)
    # the decayed-moment route was exercised: first-step-only rows' m is tiny
    if kernel == "k2":
        m_once = np.abs(ref[1].reshape(rows, cols)[kind == 1])
        assert ((m_once > 0) & (m_once < 2.0 ** -50)).mean() > 0.5

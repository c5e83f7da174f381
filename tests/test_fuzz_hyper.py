"""Randomised hyper-parameters and state magnitudes: K2 (fp32 state) and K3
(bf16 state) against the oracle's restatement of optimizer.cpp, bit for
bit.  Exercises the fast path's admission guards (power-of-two vs other
loss scales, bias corrections from t = 1 to 10^6, eps down to 0, moments
spanning 2^-120..2^100, zeros, subnormals) and the exact fallback — with
NaN payloads, infinities and invalid operations mixed in (tests/nan_inputs.py),
compared bit for bit INCLUDING the NaN payloads (the kernels reproduce the
reference's x86 NaN rules, pinned in tests/test_nan_semantics.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import nan_inputs as ni  # noqa: E402
import paper_2505_23254_b200 as mab  # noqa: E402
from oracle import oracle as ora  # noqa: E402

pytestmark = pytest.mark.gpu
f32 = np.float32


def wide(rng, n, lo, hi, zero_frac=0.05, neg=True):
    mag = np.exp2(rng.uniform(lo, hi, n)).astype(f32)
    if neg:
        mag *= np.where(rng.random(n) < 0.5, f32(-1), f32(1))
    mag[rng.random(n) < zero_frac] = 0
    return mag.astype(f32)


def draw(seed):
    rng = np.random.default_rng(seed)
    hyp = dict(lr=float(f32(10 ** rng.uniform(-6, -1))), beta1=float(f32(rng.uniform(0.5, 0.99))),
               beta2=float(f32(1 - 10 ** rng.uniform(-5, -1))),
               eps=float(f32(rng.choice([1e-8, 1e-12, 1e-3, 0.0]))),
               weight_decay=float(f32(rng.choice([0.0, 0.01, 0.1]))))
    t = int(rng.choice([1, 2, 7, 100, 2000, 10 ** 5, 10 ** 6]))
    scale = float(rng.choice([1.0, 2.0 ** rng.integers(-4, 20), float(f32(rng.uniform(0.3, 3e4)))]))
    return rng, hyp, t, scale


@pytest.mark.parametrize("seed", range(24))
def test_k2_fuzz_vs_oracle(seed):
    rng, hyp, t, scale = draw(seed)
    n = 20011
    p = wide(rng, n, -20, 4)
    m = wide(rng, n, -120, 40)
    v = np.abs(wide(rng, n, -120, 100, neg=False))
    g = wide(rng, n, -140, 20)  # includes subnormals
    g[rng.integers(0, n, 8)] = f32(1e-45)
    if seed % 2:  # every other draw: adversarial specials in ~10% of each operand
        p, m, v, g = (ni.adversarial(rng, n, x, negative=(k == 2), p_special=0.1)
                      for k, x in enumerate((p, m, v, g)))
    w_kind = "bf16" if seed % 3 else "f16"
    dev = [torch.from_numpy(x.copy()).cuda() for x in (p, m, v, g)]
    w = torch.zeros(n, dtype=torch.int16, device="cuda")
    mab.adam_step_fp32(dev[0], dev[1], dev[2], dev[3], t, mab.AdamHyper(**hyp), scale, w_out=w,
                       w_kind=w_kind)
    po, mo, vo = p.copy(), m.copy(), v.copy()
    w_or = ora.adam_step(po, mo, vo, g.copy(), t, ora.hyper(**hyp), scale, g_kind="f32",
                         w_kind=w_kind)
    for got, want in ((dev[0], po), (dev[1], mo), (dev[2], vo)):
        a = got.cpu().numpy().view(np.uint32)
        assert np.array_equal(a, want.view(np.uint32))
    assert np.array_equal(w.cpu().numpy().view(np.uint16), w_or)


@pytest.mark.parametrize("seed", range(12))
def test_k3_fuzz_vs_oracle(seed):
    rng, hyp, t, scale = draw(1000 + seed)
    n = 20011
    p16 = ora.cast_from_f32(wide(rng, n, -20, 4), "bf16")
    m16 = ora.cast_from_f32(wide(rng, n, -100, 30), "bf16")
    v16 = ora.cast_from_f32(np.abs(wide(rng, n, -100, 60, neg=False)), "bf16")
    g = wide(rng, n, -130, 20)
    if seed % 2:
        p16, m16, v16 = (ni.bf16_bits(ni.adversarial(rng, n, ora.widen(x, "bf16"),
                                                     negative=(k == 2), p_special=0.1))
                         for k, x in enumerate((p16, m16, v16)))
        g = ni.adversarial(rng, n, g, p_special=0.1)
    dev = [torch.from_numpy(x.view(np.int16).copy()).cuda() for x in (p16, m16, v16)]
    gd = torch.from_numpy(g.copy()).cuda()
    mab.adam_step_bf16(dev[0], dev[1], dev[2], gd, t, mab.AdamHyper(**hyp), scale)
    po, mo, vo = p16.copy(), m16.copy(), v16.copy()
    ora.adam_step_bf16(po, mo, vo, g.copy(), t, ora.hyper(**hyp), scale)
    for got, want in zip(dev, (po, mo, vo)):
        assert np.array_equal(got.cpu().numpy().view(np.uint16), want)

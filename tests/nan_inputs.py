"""Adversarial optimizer state for the NaN-semantics parity tests (test
infrastructure).  Every element of p / m / v / g is drawn from a menu of
ordinary values, signed zeros, infinities, quiet and signalling NaNs with
random payloads and signs, subnormals, huge and tiny magnitudes and (for v)
negative values, so that Adam's intermediates hit every x86 NaN rule:
NaN operands in either position, inf - inf, 0 * inf, 0 / 0, inf / inf and
sqrt of a negative number."""
import numpy as np

f32 = np.float32


def _nan_bits(rng, n, quiet):
    mant = rng.integers(1, 1 << 22, n, dtype=np.uint32)
    sign = rng.integers(0, 2, n, dtype=np.uint32) << 31
    q = np.uint32(0x00400000) if quiet else np.uint32(0)
    return sign | np.uint32(0x7F800000) | q | mant


def adversarial(rng, n, base, negative=False, p_special=0.5):
    """`base` (float32 array of ordinary values) with about p_special of its
    elements replaced by special values."""
    x = np.ascontiguousarray(base.astype(f32)).copy()
    u = x.view(np.uint32)
    cat = rng.integers(0, 10 if negative else 9, n)
    special = rng.random(n) < p_special
    sel = lambda k: np.flatnonzero(special & (cat == k))  # noqa: E731
    u[sel(0)] = 0x00000000
    u[sel(1)] = 0x80000000
    i = sel(2)
    u[i] = np.where(rng.integers(0, 2, i.size) == 0, 0x7F800000, 0xFF800000).astype(np.uint32)
    i = sel(3)
    u[i] = _nan_bits(rng, i.size, quiet=True)
    i = sel(4)
    u[i] = _nan_bits(rng, i.size, quiet=False)
    i = sel(5)
    u[i] = rng.integers(1, 1 << 23, i.size, dtype=np.uint32) | (
        rng.integers(0, 2, i.size, dtype=np.uint32) << 31)                 # subnormal
    i = sel(6)
    x[i] = (rng.choice([-1, 1], i.size) * rng.uniform(1e37, 3.4e38, i.size)).astype(f32)
    i = sel(7)
    x[i] = (rng.choice([-1, 1], i.size) * rng.uniform(1e-38, 1e-30, i.size)).astype(f32)
    i = sel(8)
    x[i] = (rng.choice([-1, 1], i.size) * rng.uniform(1e15, 1e25, i.size)).astype(f32)
    if negative:
        i = sel(9)
        x[i] = -np.abs(x[i]) - f32(1e-6)
    return x


def state(seed, n, p_special=0.5):
    """(p, m, v, g) float32 arrays; v may be negative, g carries NaN payloads."""
    rng = np.random.default_rng(seed)
    p = adversarial(rng, n, rng.standard_normal(n), p_special=p_special)
    m = adversarial(rng, n, rng.standard_normal(n) * 1e-3, p_special=p_special)
    v = adversarial(rng, n, np.abs(rng.standard_normal(n)) * 1e-6, negative=True,
                    p_special=p_special)
    g = adversarial(rng, n, rng.standard_normal(n) * 1024, p_special=p_special)
    return p, m, v, g


def bf16_bits(x):
    """Upper halves of float32 values (keeps NaN payload bits 16..22)."""
    return (np.ascontiguousarray(x, f32).view(np.uint32) >> 16).astype(np.uint16)


# (loss scale, eps): power-of-two scales (the LossScaler's), scales below 1
# (finite scaled gradients that overflow after unscaling),
# a non-power-of-two scale (true division), eps = 0 (0/0 when v = 0)
CASES = [(65536.0, 1e-8), (2.0 ** -10, 1e-8), (0.3, 1e-8), (1.0, 0.0), (2.0 ** -3, 0.0)]

"""Producer-side fused check (ma_stepper_ingest_async):
dst = cast(src * scale) in the stepper's gradient kind with the overflow test
on the stored values — the reference's store into the flat buffer
(simulator.cpp:401-405: fp32 multiply, then the halfprec.hpp cast) fused
with its check (overflow.hpp:46-51).  Every dtype pair, 16-byte-misaligned
views (scalar head/tail CTAs), clean and planted buffers, bit for bit
against numpy + the oracle's reference casts."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2505_23254_b200 as mab  # noqa: E402
from oracle import oracle as ora  # noqa: E402

pytestmark = pytest.mark.gpu
KINDS = ["f32", "bf16", "f16"]
TD = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


def bits_tensor(bits, kind, offset):
    """Device tensor of `bits` starting `offset` elements into its allocation."""
    it = torch.int32 if kind == "f32" else torch.int16
    raw = np.ascontiguousarray(bits).view(np.int32 if kind == "f32" else np.int16)
    buf = torch.zeros(bits.size + offset, dtype=it, device="cuda")
    buf[offset:] = torch.from_numpy(raw).cuda()
    return buf[offset:].view(TD[kind])


def host_bits(t, kind):
    if kind == "f32":
        return t.view(torch.int32).cpu().numpy().view(np.uint32)
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def expected(src_bits, sk, dk, scale):
    x = src_bits.view(np.float32) if sk == "f32" else ora.widen(src_bits, sk)
    with np.errstate(invalid="ignore", over="ignore"):  # NaN/inf inputs are the point
        y = (x.astype(np.float32) * np.float32(scale)).astype(np.float32)
    if dk == "f32":
        out = y.view(np.uint32)
        bad = bool((out & 0x7F800000 == 0x7F800000).any())
    else:
        out = ora.cast_from_f32(y, dk)
        mask = 0x7F80 if dk == "bf16" else 0x7C00
        bad = bool(((out & mask) == mask).any())
    return out, bad


@pytest.mark.parametrize("sk", KINDS)
@pytest.mark.parametrize("dk", KINDS)
@pytest.mark.parametrize("n,soff,doff", [(1_000_003, 0, 0), (65_541, 1, 3), (13, 2, 0)])
@pytest.mark.parametrize("plant", [None, 0x7FC00000, 0x7F800000, 0xFF812345])
def test_ingest_matches_reference_store(sk, dk, n, soff, doff, plant):
    rng = np.random.default_rng(n + 7 * soff + doff)
    x = (rng.standard_normal(n) * 0.25).astype(np.float32)
    src_bits = x.view(np.uint32).copy() if sk == "f32" else ora.cast_from_f32(x, sk)
    if plant is not None:
        i = int(rng.integers(0, n))
        src_bits[i] = plant if sk == "f32" else (plant >> 16 if sk == "bf16" else
                                                 ((plant >> 16) & 0x8000) | 0x7C00 |
                                                 ((plant & 0x7FFFFF) >> 13))
    scale = 2.0
    st = mab.Stepper(mab.AdamHyper(), scale, 2000, dk, "none")
    src = bits_tensor(src_bits, sk, soff)
    dst = bits_tensor(np.zeros(n, np.uint32 if dk == "f32" else np.uint16), dk, doff)
    st.ingest(src, dst)
    torch.cuda.synchronize()
    want, bad = expected(src_bits, sk, dk, scale)
    got = host_bits(dst, dk)
    # bit for bit, NaN payloads included: a NaN gradient keeps its payload
    # (quieted) through x * scale, as on the reference's x86 host
    assert np.array_equal(got, want)
    assert bool(st.flag.item()) == bad
    st.close()

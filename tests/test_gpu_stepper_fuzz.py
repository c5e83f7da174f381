"""Randomised whole-step scenarios on the B200 against the oracle's
composition of the reference (proj/src/simulator.cpp:427-492,
proj/tests/reference_trainer.hpp:27-106), bit for bit.

Each case draws, from its own seed: the partition length, misaligned base
offsets, a random cut of the partition into sub-groups (size-1 groups
included), the gradient / working-weight kinds, AdamW hyper-parameters, the
initial loss scale (power of two or not) and growth interval, faults (f32 /
bf16 non-finite patterns and finite controls) at random steps, and one of the
driver modes:

  eager    check(g) -> apply -> finish
  split    one check per sub-group gradient view (the flag ORs across them)
  graph    check -> apply -> finish captured once, replayed every step
  resume   run, snapshot {scale, clean_steps, updates}, restore into a NEW
           stepper and continue
  pure     pure-bf16 state (K3), fp32 or bf16 gradients
  streamed p / m / v in pinned host memory, staged through a random number of
           device slots of random size (configs 4/5's path)

Every mode must end with p / m / v / w (or the bf16 w / m / v) identical to
the oracle's, the same per-step skip decisions and loss scales.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2505_23254_b200 as mab  # noqa: E402
from oracle import oracle as ora  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)
G_DT = {"bf16": torch.bfloat16, "f32": torch.float32}
W_DT = {"bf16": torch.bfloat16, "f16": torch.float16}
BAD = {"bf16": (0x7F80, 0xFF80, 0x7F81, 0x7FC0, 0xFFC1),
       "f32": (0x7F800000, 0xFF800000, 0x7F800001, 0x7FC00000, 0xFFC12345)}
CONTROL = {"bf16": (0x7F7F, 0x0001, 0x8000), "f32": (0x7F7FFFFF, 0x00000001, 0x80000000)}
MODES = ("eager", "split", "graph", "resume", "pure", "streamed")


def draw_case(case):
    rs = np.random.default_rng(1000 + case)
    mode = MODES[case % len(MODES)]
    n = int(rs.choice([1, 7, 8, 33, int(rs.integers(2, 5000)), int(rs.integers(5000, 60000))]))
    cuts = sorted(set(int(x) for x in rs.integers(1, max(2, n), int(rs.integers(0, 7)))
                      if 0 < x < n))
    if n > 3 and rs.random() < 0.5:
        cuts = sorted(set(cuts + [1, n - 1]))  # size-1 groups at both ends
    bounds = list(zip([0] + cuts, cuts + [n]))
    g_kind = "f32" if rs.random() < 0.4 else "bf16"
    w_kind = "bf16" if mode == "pure" or rs.random() < 0.6 else "f16"
    hyp = dict(lr=float(rs.choice([1e-5, 1e-3, 3e-2, 0.1])),
               beta1=float(rs.choice([0.9, 0.5, 0.0, 0.99])),
               beta2=float(rs.choice([0.999, 0.95, 0.5])),
               eps=float(rs.choice([1e-8, 1e-6, 1e-3])),
               weight_decay=float(rs.choice([0.0, 0.01, 0.1])))
    scale = float(rs.choice([2.0 ** int(rs.integers(0, 21)), 3000.0, 1.5, 65536.0]))
    growth = int(rs.choice([1, 2, 3, 2000]))
    steps = int(rs.integers(4, 11))
    faults = []
    for s in range(steps):
        r = rs.random()
        if r < 0.3:
            faults.append((s, int(rs.integers(0, n)), int(rs.choice(BAD[g_kind]))))
        elif r < 0.5:
            faults.append((s, int(rs.integers(0, n)), int(rs.choice(CONTROL[g_kind]))))
    offs = [int(x) for x in rs.integers(0, 4, 5)]
    return dict(mode=mode, n=n, bounds=bounds, g_kind=g_kind, w_kind=w_kind, hyp=hyp,
                scale=scale, growth=growth, steps=steps, faults=faults, offs=offs,
                seed=int(rs.integers(1, 1 << 30)), cut=int(rs.integers(1, steps)),
                slots=int(rs.integers(2, 4)), slot_elems=int(rs.choice([64, 1000, 4096, 1 << 16])))


def buf(n, dtype, off, zero=False, host=False):
    """A length-n view starting `off` elements into a fresh allocation (misaligned)."""
    kw = dict(pin_memory=True) if host else dict(device=DEV)
    b = (torch.zeros if zero else torch.empty)(n + off, dtype=dtype, **kw)
    return b[off:off + n]


def bits(t):
    torch.cuda.synchronize()
    if t.element_size() == 4:
        return t.view(torch.int32).cpu().numpy().view(np.uint32)
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


class Rig:
    def __init__(self, c):
        self.c = c
        n, o = c["n"], c["offs"]
        self.pure = c["mode"] == "pure"
        self.g = buf(n, G_DT[c["g_kind"]], o[3])
        if self.pure:
            self.w = buf(n, torch.bfloat16, o[0])
            self.m = buf(n, torch.int16, o[1], zero=True)
            self.v = buf(n, torch.int16, o[2], zero=True)
            mab.gen_seeded_weights(None, self.w, n=n, seed=c["seed"])
        else:
            host = c["mode"] == "streamed"
            self.p = buf(n, torch.float32, o[0], host=host)
            self.m = buf(n, torch.float32, o[1], zero=True, host=host)
            self.v = buf(n, torch.float32, o[2], zero=True, host=host)
            self.w = buf(n, W_DT[c["w_kind"]], o[4])
            pd = buf(n, torch.float32, 0) if host else self.p
            mab.gen_seeded_weights(pd, self.w, seed=c["seed"])
            if host:
                self.p.copy_(pd)
                self.staging = torch.empty(3 * c["slots"] * c["slot_elems"],
                                           dtype=torch.float32, device=DEV)
        self.st = self.new_stepper()

    def new_stepper(self):
        c = self.c
        st = mab.Stepper(mab.AdamHyper(**c["hyp"]), c["scale"], c["growth"], c["g_kind"],
                         "none" if self.pure else c["w_kind"])
        b = c["bounds"]
        if self.pure:
            self.groups = [(self.w[lo:hi], self.m[lo:hi], self.v[lo:hi], self.g[lo:hi])
                           for lo, hi in b]
        else:
            self.groups = mab.Stepper.subgroups(
                [(self.p[lo:hi], self.m[lo:hi], self.v[lo:hi], self.g[lo:hi], self.w[lo:hi])
                 for lo, hi in b], c["g_kind"], c["w_kind"])
        return st

    def produce(self, s, stream=None):
        c = self.c
        mab.gen_pseudo_grads(self.g, self.w, step=s, seed=c["seed"], d_scale=self.st.scale_t,
                             stream=stream)
        for fs, idx, b in c["faults"]:
            if fs == s:
                mab.plant_bits(self.g, idx, b, stream=stream)

    def chain(self, stream=None, split=False):
        if split:
            for lo, hi in self.c["bounds"]:
                self.st.check(self.g[lo:hi], stream=stream)
        else:
            self.st.check(self.g, stream=stream)
        if self.pure:
            self.st.apply_bf16(self.groups, stream=stream)
        elif self.c["mode"] == "streamed":
            self.st.apply_streamed(self.groups, self.staging, self.c["slot_elems"],
                                   self.c["slots"], stream=stream)
        else:
            self.st.apply(self.groups, stream=stream)
        self.st.finish(stream=stream)


def run(c):
    r = Rig(c)
    mode, steps = c["mode"], c["steps"]
    hist_of, hist_sc = [], []
    if mode == "graph":
        stream = torch.cuda.Stream(device=DEV)
        stream.wait_stream(torch.cuda.current_stream())
        graph = r.st.capture(lambda: r.chain(stream), stream, reserve_steps=64)
        for s in range(steps):
            r.produce(s, stream=stream)
            graph.launch(stream)
        stream.synchronize()
        graph.close()
    elif mode == "resume":
        for s in range(c["cut"]):
            r.produce(s)
            r.chain()
        of, sc = r.st.history()
        hist_of += of.tolist()
        hist_sc += sc.tolist()
        snap = r.st.state()
        r.st.close()
        r.st = r.new_stepper()
        r.st.set_state(snap["scale"], snap["clean_steps"], snap["updates"])
        for s in range(c["cut"], steps):
            r.produce(s)
            r.chain()
    else:
        for s in range(steps):
            r.produce(s)
            r.chain(split=mode == "split")
    of, sc = r.st.history()
    hist_of += of.tolist()
    hist_sc += sc.tolist()
    return r, hist_of, hist_sc


@pytest.mark.parametrize("case", range(120))
def test_random_scenario_vs_oracle(case):
    c = draw_case(case)
    r, of, sc = run(c)
    ref = ora.train(c["n"], c["steps"], c["seed"], mixed=c["mode"] != "pure",
                    g_kind=c["g_kind"], w_kind=c["w_kind"], hyp=ora.hyper(**c["hyp"]),
                    scale=c["scale"], growth=c["growth"], faults=c["faults"])
    info = {k: c[k] for k in ("mode", "n", "g_kind", "w_kind", "hyp", "scale", "growth",
                              "steps", "offs", "slots", "slot_elems")}
    assert of == ref["overflow"].astype(bool).tolist(), info
    assert sc == ref["scale_after"].tolist(), info
    assert r.st.state()["updates"] == ref["updates"], info
    if c["mode"] == "pure":
        assert np.array_equal(bits(r.w), ref["w"]), info
        assert np.array_equal(bits(r.m), ref["m16"]), info
        assert np.array_equal(bits(r.v), ref["v16"]), info
    else:
        for k in "pmv":
            assert np.array_equal(bits(getattr(r, k)), ref[k].view(np.uint32)), (k, info)
        assert np.array_equal(bits(r.w), ref["w"]), info
    r.st.close()


@pytest.mark.parametrize("mode", ["eager", "graph", "pure", "streamed"])
def test_more_subgroups_than_one_launch_holds(mode):
    """300 ragged sub-groups (a launch takes at most 96: the update is then
    split over four launches; the streamed path runs them slot by slot),
    misaligned views, faults and scale growth, vs the oracle bit for bit."""
    rs = np.random.default_rng(77)
    n = 300 * 137 + 5
    cuts = sorted(set(int(x) for x in rs.choice(np.arange(1, n), 299, replace=False)))
    assert len(cuts) == 299
    c = dict(mode=mode, n=n, bounds=list(zip([0] + cuts, cuts + [n])), g_kind="bf16",
             w_kind="bf16", hyp=dict(lr=1e-3, weight_decay=0.01), scale=65536.0, growth=3,
             steps=6, faults=[(1, 12345, 0x7FC0), (4, n - 1, 0x7F7F)], offs=[1, 2, 3, 0, 1],
             seed=4242, cut=3, slots=3, slot_elems=4096)
    r, of, sc = run(c)
    ref = ora.train(n, c["steps"], c["seed"], mixed=mode != "pure", g_kind="bf16", w_kind="bf16",
                    hyp=ora.hyper(**c["hyp"]), scale=c["scale"], growth=c["growth"],
                    faults=c["faults"])
    assert of == ref["overflow"].astype(bool).tolist()
    assert sc == ref["scale_after"].tolist()
    if mode == "pure":
        assert np.array_equal(bits(r.w), ref["w"])
        assert np.array_equal(bits(r.m), ref["m16"])
        assert np.array_equal(bits(r.v), ref["v16"])
    else:
        for k in "pmv":
            assert np.array_equal(bits(getattr(r, k)), ref[k].view(np.uint32)), k
        assert np.array_equal(bits(r.w), ref["w"])
    r.st.close()

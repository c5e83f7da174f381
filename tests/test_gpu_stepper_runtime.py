"""Step-driver runtime features on the B200, each against the oracle's
composition of the reference (bit for bit):

  * resume: LossScaler {scale, clean_steps} and OptimizerState::step_t
    restored into a NEW stepper (optimizer.hpp:19-35,60-66,
    optimizer.cpp:120-124) continue a run exactly — 5 steps, snapshot,
    5 more == 10 steps, including a skipped step on each side of the cut and
    a scale growth right after it;
  * CUDA graph: check -> apply -> finish captured once and replayed every
    step (the loss scale, flag and t stay on the device, so one graph serves
    all steps), gradients produced outside the graph;
  * NCCL in the library: a world-1 communicator's all-reduce(max) of the
    flag between K1 and K2, eager and inside the graph.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2505_23254_b200 as mab  # noqa: E402
from oracle import oracle as ora  # noqa: E402

pytestmark = pytest.mark.gpu
N, SUB, SEED = 100_003, 30_000, 1
HYP = dict(weight_decay=0.01)
FAULTS = [(2, 4242, 0x7FC0), (7, 99, 0xFF80)]


class Run:
    def __init__(self, growth=2000, init_scale=65536.0):
        dev = torch.device("cuda", 0)
        self.p = torch.empty(N, dtype=torch.float32, device=dev)
        self.m = torch.zeros(N, dtype=torch.float32, device=dev)
        self.v = torch.zeros(N, dtype=torch.float32, device=dev)
        self.w = torch.empty(N, dtype=torch.bfloat16, device=dev)
        self.g = torch.empty(N, dtype=torch.bfloat16, device=dev)
        mab.gen_seeded_weights(self.p, self.w, seed=SEED)
        self.growth = growth
        self.st = mab.Stepper(mab.AdamHyper(**HYP), init_scale, growth, "bf16", "bf16")
        self.groups = mab.Stepper.subgroups(
            [(self.p[o:o + SUB], self.m[o:o + SUB], self.v[o:o + SUB], self.g[o:o + SUB],
              self.w[o:o + SUB]) for o in range(0, N, SUB)], "bf16", "bf16")

    def produce(self, s, stream=None):
        mab.gen_pseudo_grads(self.g, self.w, step=s, seed=SEED, d_scale=self.st.scale_t,
                             stream=stream)
        for fs, idx, bits in FAULTS:
            if fs == s:
                mab.plant_bits(self.g, idx, bits, stream=stream)

    def bits(self):
        torch.cuda.synchronize()
        return {k: getattr(self, k).view(torch.int32 if k in "pmv" else torch.int16).cpu().numpy()
                for k in "pmvw"}


def oracle(steps, growth=2000, init_scale=65536.0):
    return ora.train(N, steps, SEED, g_kind="bf16", w_kind="bf16", hyp=ora.hyper(**HYP),
                     scale=init_scale, growth=growth, faults=FAULTS)


def same(run, ref):
    b = run.bits()
    for k in "pmv":
        assert np.array_equal(b[k].view(np.uint32), ref[k].view(np.uint32)), k
    assert np.array_equal(b["w"].view(np.uint16), ref["w"])


def test_resume_equals_uninterrupted_run():
    growth = 3  # the scale grows on the first step after the cut
    ref = oracle(10, growth=growth)
    a = Run(growth)
    for s in range(5):
        a.produce(s)
        a.st.step([a.g], a.groups)
    snap = a.st.state()
    assert snap["updates"] == 4 and snap["clean_steps"] == 2  # step 2 was skipped
    b = Run(growth)
    b.p.copy_(a.p), b.m.copy_(a.m), b.v.copy_(a.v), b.w.copy_(a.w)
    a.st.close()
    b.st.set_state(snap["scale"], snap["clean_steps"], snap["updates"])
    for s in range(5, 10):
        b.produce(s)
        b.st.step([b.g], b.groups)
    same(b, ref)
    st = b.st.state()
    assert st["updates"] == 8 and st["scale"] == float(ref["scale_after"][-1])
    of, sc = b.st.history()
    assert of.tolist() == ref["overflow"][5:].astype(bool).tolist()
    assert sc.tolist() == ref["scale_after"][5:].tolist()


def test_set_state_validation():
    r = Run()
    with pytest.raises(mab.MemAscendError):
        r.st.set_state(0.0, 0, 3)
    with pytest.raises(mab.MemAscendError):
        r.st.set_state(1024.0, 2000, 3)  # clean_steps must stay below growth_interval


def test_apply_bf16_validation():
    """apply_bf16 checks kinds and lengths before anything reaches the device."""
    st = mab.Stepper(mab.AdamHyper(), 65536.0, 2000, "bf16", "bf16")
    n = 4096
    b = lambda k=n: torch.zeros(k, dtype=torch.bfloat16, device="cuda")  # noqa: E731
    with pytest.raises(mab.MemAscendError):  # fp32 moments
        st.apply_bf16([(b(), torch.zeros(n, device="cuda"), b(), b())])
    with pytest.raises(mab.MemAscendError):  # short variance
        st.apply_bf16([(b(), b(), b(n - 8), b())])
    with pytest.raises(mab.MemAscendError):  # fp32 grads for a bf16 stepper
        st.apply_bf16([(b(), b(), b(), torch.zeros(n, device="cuda"))])
    with pytest.raises(mab.MemAscendError):  # non-contiguous
        st.apply_bf16([(b(2 * n)[::2], b(), b(), b())])
    st.apply_bf16([(b(), b(), b(), b())])  # well-formed: runs
    torch.cuda.synchronize()
    st.close()


@pytest.mark.parametrize("with_comm", [False, True])
def test_graph_replay_equals_eager(with_comm):
    ref = oracle(10)
    r = Run()
    stream = torch.cuda.Stream()
    comm = mab.NcclComm(1, 0, lambda b: b) if with_comm else None

    def chain():
        r.st.check(r.g, stream=stream)
        if comm is not None:
            r.st.allreduce_flag(comm, stream=stream)
        r.st.apply(r.groups, stream=stream)
        r.st.finish(stream=stream)

    stream.wait_stream(torch.cuda.current_stream())
    graph = r.st.capture(chain, stream, reserve_steps=64)
    for s in range(10):
        r.produce(s, stream=stream)
        graph.launch(stream)
    stream.synchronize()
    same(r, ref)
    of, sc = r.st.history()
    assert of.tolist() == ref["overflow"].astype(bool).tolist()
    assert sc.tolist() == ref["scale_after"].tolist()
    assert r.st.state()["steps"] == 10
    graph.close()
    if comm is not None:
        assert comm.info()["world"] == 1 and comm.info()["nccl_version"] > 0
        comm.close()


def test_graph_reserve_exhaustion_is_reported():
    r = Run()
    stream = torch.cuda.Stream()

    def chain():
        r.st.check(r.g, stream=stream)
        r.st.apply(r.groups, stream=stream)
        r.st.finish(stream=stream)

    graph = r.st.capture(chain, stream, reserve_steps=3)
    launched = 0
    with pytest.raises(mab.MemAscendError) as e:
        for s in range(100000):
            graph.launch(stream)
            launched += 1
    assert e.value.code == "lifecycle" and launched >= 3
    stream.synchronize()


def test_nccl_flag_allreduce_eager():
    ref = oracle(10)
    r = Run()
    comm = mab.NcclComm(1, 0, lambda b: b)
    for s in range(10):
        r.produce(s)
        r.st.check(r.g)
        r.st.allreduce_flag(comm)
        r.st.apply(r.groups)
        r.st.finish()
    same(r, ref)
    comm.close()


def test_subgroup_validation():
    r = Run()
    with pytest.raises(mab.MemAscendError):  # f32 grads for a bf16 stepper
        r.st.apply([(r.p, r.m, r.v, torch.zeros(N, device="cuda"), r.w)])
    with pytest.raises(mab.MemAscendError):  # length mismatch
        r.st.apply([(r.p, r.m, r.v[:-1], r.g, r.w)])
    with pytest.raises(mab.MemAscendError):  # missing working weights
        r.st.apply([(r.p, r.m, r.v, r.g, None)])


def test_shard_stepper_with_library_nccl():
    """shard.py's ShardStepper with the OR in the library's NCCL communicator
    (DeviceShard.comm, world 1) over cfg3's plan == the single-process oracle."""
    from paper_2505_23254_b200.shard import DeviceShard, FaultPlan, ShardStepper

    plan = FaultPlan(N, SUB, seed=7)
    be = DeviceShard(N, 0, SUB, seed=SEED, hyper=mab.AdamHyper(**HYP))
    be.comm = mab.NcclComm(1, 0, lambda b: b)
    drv = ShardStepper(be, 0, N, plan, allreduce=None)
    for s in range(8):
        drv.step(s)
    torch.cuda.synchronize()
    faults = [(p.step, p.index, p.bits) for s in range(8) for p in plan.at(s)]
    ref = ora.train(N, 8, SEED, g_kind="bf16", w_kind="bf16", hyp=ora.hyper(**HYP),
                    faults=faults)
    of, sc = be.st.history()
    assert of.tolist() == ref["overflow"].astype(bool).tolist()
    assert sc.tolist() == ref["scale_after"].tolist()
    for k in "pmv":
        got = getattr(be, k).cpu().numpy().view(np.uint32)
        assert np.array_equal(got, ref[k].view(np.uint32)), k
    be.comm.close()


def test_fused_exchange_single_rank_in_a_graph():
    """K1's fused flag exchange at world 1 (the last-CTA completion counter,
    the device-side epoch, the slot protocol) eager and replayed from a graph:
    decisions / state equal the oracle — in one process, so compute-sanitizer
    sees the protocol (tools/sanitize.sh)."""
    ref = oracle(10)
    r = Run()
    x = mab.api.FlagExchange(1, 0, lambda b: [b])
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())

    def chain():
        r.st.check(r.g, stream=stream, xchg=x)
        r.st.apply(r.groups, stream=stream)
        r.st.finish(stream=stream)

    for s in range(3):  # eager
        r.produce(s, stream=stream)
        chain()
    graph = r.st.capture(chain, stream, reserve_steps=64)
    for s in range(3, 10):
        r.produce(s, stream=stream)
        graph.launch(stream)
    stream.synchronize()
    same(r, ref)
    assert not x.timed_out()
    graph.close()
    x.close()


def test_registered_host_memory_sits_on_the_gpus_numa_node():
    """On a multi-socket host the pages of a registered buffer are placed on
    the NUMA node of the GPU's PCIe root (ma_host_register); on one node the
    query still answers."""
    import ctypes as C
    import os

    dev_node, page_node = C.c_int(), C.c_int()
    mab.capi.check(mab.capi.lib().ma_device_numa_node(C.byref(dev_node)))
    buf = mab.aligned_host_buffer(64 << 20, register=True)
    mab.capi.check(mab.capi.lib().ma_host_numa_node(buf.ctypes.data, C.byref(page_node)))
    nodes = len([d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")])
    if nodes > 1 and dev_node.value >= 0:
        assert page_node.value == dev_node.value
    else:
        assert page_node.value >= -1
    mab.host_unregister(buf)


def test_failed_capture_leaves_the_stepper_usable():
    """An exception inside the captured function ends the capture and drops
    the partial graph; the stepper then steps eagerly as before."""
    ref = oracle(3)
    r = Run()
    stream = torch.cuda.Stream()

    def bad():
        r.st.check(r.g, stream=stream)
        raise RuntimeError("user code failed mid-capture")

    with pytest.raises(RuntimeError):
        r.st.capture(bad, stream)
    for s in range(3):
        r.produce(s)
        r.st.step([r.g], r.groups)
    same(r, ref)


def test_resume_at_huge_t_keeps_a_small_window():
    """A run resumed at t = 10^9 (OptimizerState::step_t) continues exactly:
    the bias-correction window starts at the restored t instead of holding
    every t from 1 (which would be 8 GB here)."""
    n = 20_011
    rng = np.random.default_rng(2)
    p0 = (rng.standard_normal(n) * 0.1).astype(np.float32)
    m0 = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    v0 = (np.abs(rng.standard_normal(n)) * 1e-6).astype(np.float32)
    t0 = 10 ** 9
    h = ora.hyper(**HYP)
    ref = [p0.copy(), m0.copy(), v0.copy()]
    dev = torch.device("cuda", 0)
    p, m, v = (torch.from_numpy(x.copy()).to(dev) for x in (p0, m0, v0))
    w = torch.empty(n, dtype=torch.bfloat16, device=dev)
    g = torch.empty(n, dtype=torch.bfloat16, device=dev)
    st = mab.Stepper(mab.AdamHyper(**HYP), 1024.0, 2000, "bf16", "bf16")
    st.set_state(1024.0, 5, t0)
    for s in range(4):
        gs = ora.cast_from_f32((rng.standard_normal(n) * 1024).astype(np.float32), "bf16")
        g.view(torch.int16).copy_(torch.from_numpy(gs.view(np.int16)))
        st.step([g], [(p, m, v, g, w)])
        ora.adam_step(*ref, ora.widen(gs, "bf16"), t0 + s + 1, h, 1024.0)
    torch.cuda.synchronize()
    for got, want, name in zip((p, m, v), ref, "pmv"):
        assert np.array_equal(got.cpu().numpy().view(np.uint32), want.view(np.uint32)), name
    assert st.state()["updates"] == t0 + 4


def test_bias_window_rolls_over_past_65536_steps():
    """70 000 eager steps on a small partition: the bias-correction window
    (65 536 entries) is re-based once on the way; decisions, scales and the
    final state equal the oracle's 70 000-step run bit for bit."""
    n, steps = 4099, 70_000
    ref = ora.train(n, steps, SEED, g_kind="bf16", w_kind="bf16", hyp=ora.hyper(**HYP),
                    scale=65536.0, growth=2000)
    dev = torch.device("cuda", 0)
    p = torch.empty(n, dtype=torch.float32, device=dev)
    m = torch.zeros(n, dtype=torch.float32, device=dev)
    v = torch.zeros(n, dtype=torch.float32, device=dev)
    w = torch.empty(n, dtype=torch.bfloat16, device=dev)
    g = torch.empty(n, dtype=torch.bfloat16, device=dev)
    mab.gen_seeded_weights(p, w, seed=SEED)
    st = mab.Stepper(mab.AdamHyper(**HYP), 65536.0, 2000, "bf16", "bf16")
    groups = mab.Stepper.subgroups([(p, m, v, g, w)], "bf16", "bf16")
    for s in range(steps):
        mab.gen_pseudo_grads(g, w, step=s, seed=SEED, d_scale=st.scale_t)
        st.check(g)
        st.apply(groups)
        st.finish()
    torch.cuda.synchronize()
    of, sc = st.history(cap=steps)
    assert of.tolist() == ref["overflow"].astype(bool)[-of.size:].tolist()
    assert sc.tolist() == ref["scale_after"][-sc.size:].tolist()
    for k, t in zip("pmv", (p, m, v)):
        assert np.array_equal(t.cpu().numpy().view(np.uint32), ref[k].view(np.uint32)), k
    assert st.state()["updates"] == int(ref["updates"]) > 65_536

"""Multi-rank step (BASELINE configs[2]): per-rank K1, one
all-reduce(max) of the flag, identical skip decisions on every rank.

The world-size 2/4/8 runs use torch.distributed with the gloo backend on
127.0.0.1.  The CPU test drives the product's ShardStepper with an
oracle-backed shard (test infrastructure); the GPU test drives it with the
B200 kernels (DeviceShard, both ranks on cuda:0).  Both are compared with a
single-process oracle run over the whole partition with the same faults.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as ora
from paper_2505_23254_b200.shard import (FaultPlan, ShardStepper, shard_range, subgroup_bounds)

N_TOTAL, SUBGROUP, STEPS, SEED = 1_000_003, 100_000, 10, 1
WORLDS = [2, 4, 8]  # BASELINE configs[2]: the injection run at 2/4/8 ranks
HYP = dict(lr=1e-3, weight_decay=0.01)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleShard:
    """Test backend: the oracle (CPU) in the ShardStepper protocol."""

    def __init__(self, n, base):
        self.n, self.base = n, base
        self.p, self.w = ora.fill_weights(n, base=base, seed=SEED) if n else (
            np.zeros(0, np.float32), np.zeros(0, np.uint16))
        self.m = np.zeros(n, np.float32)
        self.v = np.zeros(n, np.float32)
        self.flag = torch.zeros(1, dtype=torch.int32)
        self.scaler = ora.Scaler(65536.0, 2000, 0)
        self.updates = 0
        self.history = []

    def produce_grads(self, step):
        self.g = (ora.fill_grads(self.w, step, base=self.base, seed=SEED,
                                 scale=self.scaler.scale, widened=False)[0]
                  if self.n else np.zeros(0, np.uint16))

    def plant(self, i, bits):
        self.g[i] = bits

    def check(self):
        self.flag[0] = int(ora.overflow_check(self.g, "bf16")[0]) if self.n else 0

    def apply(self):
        if int(self.flag[0]) or not self.n:
            return
        self.w[:] = ora.adam_step(self.p, self.m, self.v, self.g, self.updates + 1,
                                  ora.hyper(**HYP), self.scaler.scale, "bf16", "bf16")

    def finish(self):
        skip = bool(int(self.flag[0]))
        if skip:
            ora.lib().ora_scaler_on_overflow(ora.C.byref(self.scaler))
        else:
            self.updates += 1
            ora.lib().ora_scaler_on_clean_step(ora.C.byref(self.scaler))
        self.history.append((skip, self.scaler.scale))
        self.flag[0] = 0


def _worker(rank, port, out_dir, device_backend, p2p=False, WORLD=2):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        base, n = shard_range(N_TOTAL, WORLD, rank, SUBGROUP)
        plan = FaultPlan(N_TOTAL, SUBGROUP, seed=7)
        if device_backend:
            import paper_2505_23254_b200 as mab
            from paper_2505_23254_b200.shard import DeviceShard

            torch.cuda.set_device(0)
            be = DeviceShard(n, base, SUBGROUP, seed=SEED, hyper=mab.AdamHyper(**HYP))
            if p2p:
                # the OR rides on K1 over peer memory (CUDA IPC mappings)
                be.xchg = mab.api.FlagExchange(WORLD, rank, mab.api.torch_all_gather_bytes())
                allreduce = None
            else:
                def allreduce(flag):
                    dist.all_reduce(flag, op=dist.ReduceOp.MAX)  # gloo on a CUDA tensor
        else:
            be = OracleShard(n, base)

            def allreduce(flag):
                dist.all_reduce(flag, op=dist.ReduceOp.MAX)

        drv = ShardStepper(be, base, n, plan, allreduce)
        for s in range(STEPS):
            drv.step(s)
        if device_backend:
            torch.cuda.synchronize()
            if p2p:
                assert not be.xchg.timed_out()
            of, sc = be.st.history()
            res = dict(p=be.p.cpu().numpy(), m=be.m.cpu().numpy(), v=be.v.cpu().numpy(),
                       w=be.w.view(torch.int16).cpu().numpy().view(np.uint16),
                       overflow=of.astype(np.uint8), scale=sc)
        else:
            res = dict(p=be.p, m=be.m, v=be.v, w=be.w,
                       overflow=np.array([h[0] for h in be.history], np.uint8),
                       scale=np.array([h[1] for h in be.history], np.float32))
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), base=base, n=n, **res)
    finally:
        dist.destroy_process_group()


def _check_against_single_process(out_dir, WORLD):
    plan = FaultPlan(N_TOTAL, SUBGROUP, seed=7)
    faults = [(p.step, p.index, p.bits) for s in range(STEPS) for p in plan.at(s)]
    want = ora.train(N_TOTAL, STEPS, SEED, g_kind="bf16", w_kind="bf16", hyp=ora.hyper(**HYP),
                     faults=faults)
    expected = [plan.expected_skip(s) for s in range(STEPS)]
    assert want["overflow"].astype(bool).tolist() == expected
    assert any(expected) and not all(expected)  # the plan exercises both paths
    covered = 0
    for r in range(WORLD):
        d = np.load(os.path.join(out_dir, f"rank{r}.npz"))
        base, n = int(d["base"]), int(d["n"])
        assert d["overflow"].astype(bool).tolist() == expected, r
        assert d["scale"].tolist() == want["scale_after"].tolist(), r
        for k in "pmvw":
            a, b = d[k], want[k][base:base + n]
            assert a.view(np.uint8).tobytes() == b.view(np.uint8).tobytes(), (r, k)
        covered += n
    assert covered == N_TOTAL


def test_shard_ranges_cover_in_whole_subgroups():
    for world in (1, 2, 3, 4, 8):
        spans = [shard_range(N_TOTAL, world, r, SUBGROUP) for r in range(world)]
        assert sum(n for _, n in spans) == N_TOTAL
        pos = 0
        for base, n in spans:
            assert base == pos and (base % SUBGROUP == 0 or n == 0)
            pos += n
    assert subgroup_bounds(250, 100) == [(0, 100), (100, 100), (200, 50)]


def test_fault_plan_is_deterministic_and_rank_local():
    plan = FaultPlan(N_TOTAL, SUBGROUP, seed=7)
    assert [plan.at(s) for s in range(20)] == [FaultPlan(N_TOTAL, SUBGROUP, 7).at(s)
                                                 for s in range(20)]
    ks = {sum(not p.control for p in plan.at(s)) for s in range(60)}
    assert ks == {0, 1, 3}
    for world in WORLDS:
        for s in range(20):
            local = [p for r in range(world)
                     for p in plan.local(s, *shard_range(N_TOTAL, world, r, SUBGROUP))]
            assert (sorted(local, key=lambda p: p.index) ==
                    sorted(plan.at(s), key=lambda p: p.index))


@pytest.mark.parametrize("world", WORLDS)
def test_ranks_gloo_cpu_match_single_process(world):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(free_port(), d, False, False, world), nprocs=world, join=True)
        _check_against_single_process(d, world)


@pytest.mark.gpu
@pytest.mark.parametrize("world", WORLDS)
def test_ranks_on_b200_match_single_process(world):
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(free_port(), d, True, False, world), nprocs=world, join=True)
        _check_against_single_process(d, world)


@pytest.mark.gpu
@pytest.mark.parametrize("world", WORLDS)
def test_ranks_on_b200_peer_exchange_fused_in_k1(world):
    """Same run with the skip decision exchanged by K1's last CTA through
    peer memory (ma_stepper_check_xchg_async) instead of an all-reduce."""
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(free_port(), d, True, True, world), nprocs=world, join=True)
        _check_against_single_process(d, world)


def test_cfg3_plan_fixture_pins_decisions_and_scales(golden):
    """tests/golden/cfg3_plan.json (oracle/_ref golden_gen: the plan's draws
    + the reference's own LossScaler) is what bench.py --config cfg3 checks
    its ranks against: shard.FaultPlan's decision of every step equals it
    for any partition size, and the oracle's scaler reproduces its scales."""
    fx = golden("cfg3_plan.json")
    for n_total, sub in ((1_000_003, 100_000), (8_030_261_248 * 8, 100_000_000), (77, 10)):
        plan = FaultPlan(n_total, sub, seed=fx["seed"])
        assert [int(plan.expected_skip(s)) for s in range(fx["steps"])] == fx["overflow"]
    sc = ora.Scaler(fx["init_scale"], fx["growth_interval"], 0)
    got = []
    for of in fx["overflow"]:
        if of:
            ora.lib().ora_scaler_on_overflow(ora.C.byref(sc))
        else:
            ora.lib().ora_scaler_on_clean_step(ora.C.byref(sc))
        got.append(int(np.float32(sc.scale).view(np.uint32)))
    assert got == fx["scale_after_bits"]

"""ZeRO-style sharding of the optimizer partition and the cross-rank skip step.

The reference runs ONE fused check over the whole flat gradient buffer
(proj/src/simulator.cpp:431-436) and treats the rank count as a pure
parameter (ceil-division sharding in proj/src/model.cpp:85-94).
Here each rank owns a contiguous slice of whole sub-groups, checks only its
own gradients (K1), and the global decision is the OR of the per-rank flags —
one all-reduce(max) of a single int32 over NCCL — so every rank skips or
updates identically and its LossScaler / t evolve identically (SURVEY.md
§8(e)).  Nothing else crosses ranks.

The step driver is backend-agnostic so the same exchange logic is exercised
with the B200 kernels (``DeviceShard``) and, in tests, with any object that
implements the four-method backend protocol.  With ``DeviceShard`` the OR
runs in one of three places: a host-side ``allreduce`` callable
(torch.distributed), the library's own NCCL communicator
(``DeviceShard.comm = NcclComm(...)``, no Python on the step path) or K1's
last CTA over peer memory (``DeviceShard.xchg = FlagExchange(...)``).
"""
from __future__ import annotations

from dataclasses import dataclass

MASK64 = (1 << 64) - 1

# cfg3 (BASELINE.json configs[2]) bf16 patterns: +inf, -inf, sNaN, qNaN, -NaN
BAD_BF16 = (0x7F80, 0xFF80, 0x7F81, 0x7FC0, 0xFFC1)
CONTROL_BF16 = 0x7F7F  # largest finite bf16: must never trigger a skip


def ceil_div(a: int, b: int) -> int:
    return (a + b - 1) // b


def shard_range(n_total: int, world: int, rank: int, subgroup: int) -> tuple[int, int]:
    """(base, n) of `rank`'s slice: whole sub-groups, ceil-divided like
    model.cpp:87-94 so no shard undersizes; trailing ranks may be empty."""
    groups = ceil_div(n_total, subgroup)
    per = ceil_div(groups, world)
    lo = min(n_total, rank * per * subgroup)
    hi = min(n_total, (rank + 1) * per * subgroup)
    return lo, hi - lo


def subgroup_bounds(n: int, subgroup: int) -> list[tuple[int, int]]:
    return [(o, min(subgroup, n - o)) for o in range(0, n, subgroup)]


def splitmix64(x: int) -> int:
    """proj/include/memascend/simulator.hpp:23-28 (host copy for planning)."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


@dataclass(frozen=True)
class Plant:
    step: int
    index: int   # global element index
    bits: int    # bf16 pattern
    control: bool


class FaultPlan:
    """cfg3's seeded injection: every step picks k in {0, 1, 3} random
    sub-groups (anywhere in the global partition, hence on random ranks) and
    plants one of the five non-finite bf16 patterns in each, plus one
    max-finite control value that must not trigger.  Deterministic in
    (seed, step), so every rank derives the same plan without communication."""

    def __init__(self, n_total: int, subgroup: int, seed: int = 2505):
        self.n_total, self.subgroup, self.seed = n_total, subgroup, seed
        self.groups = ceil_div(n_total, subgroup)

    def at(self, step: int) -> list[Plant]:
        h = splitmix64(self.seed ^ splitmix64(step ^ 0xC0FFEE))

        def draw():
            nonlocal h
            h = splitmix64(h)
            return h

        k = (0, 1, 3)[draw() % 3]
        out = []
        for _ in range(k):
            g = draw() % self.groups
            lo = g * self.subgroup
            size = min(self.subgroup, self.n_total - lo)
            out.append(Plant(step, lo + draw() % size, BAD_BF16[draw() % len(BAD_BF16)], False))
        out.append(Plant(step, draw() % self.n_total, CONTROL_BF16, True))
        return out

    def expected_skip(self, step: int) -> bool:
        return any(not p.control for p in self.at(step))

    def local(self, step: int, base: int, n: int) -> list[Plant]:
        return [p for p in self.at(step) if base <= p.index < base + n]


class ShardStepper:
    """One rank's step: produce -> plant -> K1 -> all-reduce(max) -> K2 -> scaler.

    backend protocol:
      produce_grads(step)              gradients for this step (the producer)
      plant(local_index, bits)         fault injection (simulator.cpp:427-429)
      check()                          local overflow check into backend.flag
      apply() / finish()               update (skipped on flag) and scaler
    `allreduce(flag)` ORs the int32 flag across ranks (None on one rank).
    """

    def __init__(self, backend, base: int, n: int, plan: FaultPlan | None = None,
                 allreduce=None):
        self.backend, self.base, self.n = backend, base, n
        self.plan, self.allreduce = plan, allreduce

    def step(self, step: int) -> None:
        b = self.backend
        b.produce_grads(step)
        if self.plan is not None:
            for p in self.plan.local(step, self.base, self.n):
                b.plant(p.index - self.base, p.bits)
        b.check()
        if self.allreduce is not None:
            self.allreduce(b.flag)
        b.apply()
        b.finish()


class DeviceShard:
    """B200 backend: one rank's p/m/v/g/w in HBM, the device-resident step
    driver (ma_stepper_*) and the bit-exact workload generators."""

    def __init__(self, n: int, base: int, subgroup: int, seed: int = 1, hyper=None,
                 init_scale: float = 65536.0, growth_interval: int = 2000, device=None):
        import torch

        from .api import AdamHyper, Stepper, gen_seeded_weights

        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.n, self.base, self.seed = n, base, seed
        self.p = torch.empty(max(n, 1), dtype=torch.float32, device=dev)[:n]
        self.m = torch.zeros(max(n, 1), dtype=torch.float32, device=dev)[:n]
        self.v = torch.zeros(max(n, 1), dtype=torch.float32, device=dev)[:n]
        self.g = torch.empty(max(n, 1), dtype=torch.bfloat16, device=dev)[:n]
        self.w = torch.empty(max(n, 1), dtype=torch.bfloat16, device=dev)[:n]
        self.st = Stepper(hyper or AdamHyper(), init_scale, growth_interval, "bf16", "bf16",
                          device=dev)
        self.flag = self.st.flag
        if n:
            gen_seeded_weights(self.p, self.w, base=base, seed=seed)
        self.groups = Stepper.subgroups(
            [(self.p[o:o + k], self.m[o:o + k], self.v[o:o + k], self.g[o:o + k],
              self.w[o:o + k]) for o, k in subgroup_bounds(n, subgroup)]) if n else None

    def produce_grads(self, step: int) -> None:
        from .api import gen_pseudo_grads

        if self.n:
            gen_pseudo_grads(self.g, self.w, step=step, base=self.base, seed=self.seed,
                             d_scale=self.st.scale_t)

    def plant(self, local_index: int, bits: int) -> None:
        from .api import plant_bits

        plant_bits(self.g, local_index, bits)

    xchg = None  # FlagExchange: fuse the cross-rank OR into K1 (no all-reduce)
    comm = None  # NcclComm: the library's own ncclAllReduce(max) of the flag

    def check(self) -> None:
        if self.xchg is not None:
            self.st.check(self.g if self.n else None, xchg=self.xchg)
        elif self.n:
            self.st.check(self.g)
        if self.comm is not None:
            # the cross-rank OR inside the library (ma_stepper_allreduce_flag_async),
            # on the compute stream: pass allreduce=None to ShardStepper
            self.st.allreduce_flag(self.comm)

    def apply(self) -> None:
        if self.n:
            self.st.apply(self.groups)

    def finish(self) -> None:
        self.st.finish()

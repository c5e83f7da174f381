#!/usr/bin/env python
"""Optimizer-step benchmark for the B200 MemAscend hot path.

One step = the reference's per-step optimizer pass (simulator.cpp:427-492)
over one rank's flat partition: K1 fused overflow check over all scaled bf16
gradients -> (N>1: NCCL all-reduce(max) of the flag) -> K2 unscale + AdamW +
bf16 cast-back over every 100M-param sub-group -> device-side LossScaler.

Default workload = BASELINE.json configs[1]: Llama-3-8B-shaped optimizer
state, 8,030,261,248 params per GPU (model.cpp:233), resident in HBM
(fp32 master/m/v + bf16 grads + bf16 working weights = 128.5 GB), 81
sub-groups of 100,000,000 params.  Weak scaling under torchrun: every rank
owns one such partition (global element index = rank * n + i).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Rank 0 prints one JSON line.  Timing: CUDA events on the launching stream,
barrier + synchronize on both sides, max over ranks.  Inputs (128.5 GB) are
far larger than L2 (126 MB), so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "optimizer-step params/sec (overflow check+AdamW) and HBM GB/s vs B200 peak"
LLAMA3_8B = 8_030_261_248       # proj/src/model.cpp:233
QWEN25_14B = 14_770_033_664     # proj/src/model.cpp:239 (configs[3], sharded 8 ways)
LLAMA3_70B = 70_553_706_496     # configs[4] (V 128256, H 8192, I 28672, L 80, kv 1024), 8 ways
CFG1 = 67_108_864               # configs[0]: one 64M-param sub-group
SUBGROUP = 100_000_000          # optimizer sub-group
BYTES_PER_PARAM = 28            # 2 g + 12 pmv read + 12 pmv write + 2 w16
HYPER = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["cfg2", "cfg1", "cfg3", "cfg4", "cfg5"], default="cfg2",
                    help="BASELINE.json configs[n-1]; cfg3 = cfg2's partition per rank with "
                         "the seeded inf/NaN injection plan, decisions checked against the "
                         "committed oracle plan")
    ap.add_argument("--slots", type=int, default=3, help="cfg4 staging slots")
    ap.add_argument("--slot-params", type=int, default=1 << 24, help="cfg4 params per slot")
    ap.add_argument("--params", type=int, default=0, help="override params per GPU (debug)")
    ap.add_argument("--swap-dir", default="/tmp/memascend_swap",
                    help="cfg5: directory of the swap store's file-backed devices")
    ap.add_argument("--swap-gb", type=float, default=32.0,
                    help="cfg5: optimizer state kept on the swap device (the rest in pinned DRAM)")
    ap.add_argument("--host-slots", type=int, default=6, help="cfg5 registered host slots")
    ap.add_argument("--io-workers", type=int, default=4, help="cfg5 swap-store workers")
    ap.add_argument("--io-depth", type=int, default=32, help="cfg5 requests in flight per worker")
    ap.add_argument("--zero-fused", action="store_true",
                    help="the whole ZeRO step over peer memory: K4 reduce-scatter+check of "
                         "full-length gradients, K2 update + weight all-gather (per-rank "
                         "partition --params, default 1e9)")
    ap.add_argument("--precision", choices=["mixed", "pure_bf16"], default="mixed",
                    help="optimizer state: fp32 master/m/v (K2) or bf16 m/v + bf16 weights "
                         "(OptimPrecision::pure_bf16, K3) — in HBM for cfg1/cfg2/cfg3, "
                         "swapped for cfg5")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e-spec", action="store_true",
                    help="e2e without speculative updates during the gradient transfer")
    ap.add_argument("--flag-exchange", choices=["nccl", "torch", "p2p"], default="nccl",
                    help="N>1: all-reduce the skip flag with the library's own NCCL "
                         "communicator (ma_comm, default), with torch.distributed, or fuse "
                         "the exchange into K1 over peer memory")
    ap.add_argument("--graph", action="store_true",
                    help="capture check -> exchange -> apply -> finish into a CUDA graph once "
                         "and replay it every step (one launch per step)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=CFG1,
                    help="params in the CPU baseline's bounded sample")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        except Exception:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][2]),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit()),
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------- CPU arms
def cpu_reference_run(n, steps, warmup, threads):
    """The reference's own CPU path (oracle/_ref: fused_overflow_check +
    adam_step_fp32 per sub-group + cast, simulator.cpp:431-469 composition)
    on a bounded sample of the same workload.  Falls back to the restated
    oracle only if the reference library was not built."""
    from oracle import oracle as ora

    p, w = ora.fill_weights(n, seed=1, w_kind="bf16", threads=threads)
    _, g32 = ora.fill_grads(w, 0, seed=1, scale=65536.0, g_kind="bf16", w_kind="bf16",
                            threads=threads)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    h = ora.hyper(**HYPER)
    kind = "reference" if ora.ref_available() else "port"
    times = []
    for s in range(warmup + steps):
        if kind == "reference":
            of, secs = ora.ref_bench_step(g32, p, m, v, w, "bf16", SUBGROUP, s + 1, h, 65536.0,
                                          threads)
        else:
            t0 = time.perf_counter()
            of, _ = ora.overflow_check(g32, "f32")
            w[:] = ora.adam_step(p, m, v, g32, s + 1, h, 65536.0, "f32", "bf16")
            secs = time.perf_counter() - t0
        assert not of
        if s >= warmup:
            times.append(secs)
    t = float(np.median(times))
    return {"value": n / t, "unit": "params/s", "cores": threads, "kind": kind,
            "sample": f"{n} params (bf16-rounded grads widened to the reference's fp32 flat "
                      f"buffer), {SUBGROUP // 1_000_000}M sub-groups, median of {steps} steps "
                      f"after {warmup} warm-up, {threads} threads",
            "seconds_per_step": t}


def cpu_reference_run_bf16(n, steps, warmup, threads):
    """The reference's pure-bf16 step (OptimPrecision::pure_bf16,
    simulator.cpp:431-486: fused_overflow_check over the fp32 flat buffer,
    then adam_step_bf16 per sub-group on the bf16 weights / m / v) from
    oracle/_ref on a bounded sample, all `threads` host threads."""
    from oracle import oracle as ora

    if not ora.ref_available():
        raise SystemExit("cpu baseline: oracle/_ref (the compiled reference) is missing")
    _, w = ora.fill_weights(n, seed=1, w_kind="bf16", threads=threads)
    _, g32 = ora.fill_grads(w, 0, seed=1, scale=65536.0, g_kind="bf16", w_kind="bf16",
                            threads=threads)
    m = np.zeros(n, np.uint16)
    v = np.zeros(n, np.uint16)
    h = ora.hyper(**HYPER)
    times = []
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        of, _ = ora.ref_fused_overflow_check(g32, workers=threads)
        assert not of
        for o in range(0, n, SUBGROUP):
            e = min(n, o + SUBGROUP)
            ora.ref_adam_step_bf16(w[o:e], m[o:e], v[o:e], g32[o:e], s + 1, h, 65536.0, threads)
        if s >= warmup:
            times.append(time.perf_counter() - t0)
    t = float(np.median(times))
    return {"value": n / t, "unit": "params/s", "cores": threads, "kind": "reference",
            "sample": f"{n} params, pure-bf16 state (bf16 weights/m/v, bf16-rounded grads "
                      f"widened to the reference's fp32 flat buffer), fused_overflow_check + "
                      f"adam_step_bf16 per {SUBGROUP // 1_000_000}M sub-group, median of {steps} "
                      f"steps after {warmup} warm-up, {threads} threads",
            "seconds_per_step": t}


def cpu_model():
    """lscpu's model name and socket count (record both)."""
    model, sockets = "unknown", None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
            elif line.startswith("Socket(s)"):
                sockets = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return model if sockets is None else f"{model}, {sockets} socket(s)"


def reference_swapped_run(args, steps, warmup, threads, groups=2):
    """configs[4] reference arm: the reference's own swapped step
    (DirectIoEngine read master/m/v -> adam_step_fp32 -> write back,
    simulator.cpp:453-469) on `groups` 100 M sub-groups in --swap-dir."""
    import shutil

    from oracle import oracle as ora

    gs = np.random.default_rng(0).standard_normal(groups * SUBGROUP).astype(np.float32) * 8192
    rdir = os.path.join(args.swap_dir, "ref-arm")
    try:
        secs, io = ora.ref_swap_bench(rdir, 2, SUBGROUP, groups, steps, warmup, gs,
                                      ora.hyper(**HYPER), 65536.0, threads)
    finally:
        shutil.rmtree(rdir, ignore_errors=True)
    return {"value": groups * SUBGROUP / secs, "unit": "params/s", "cores": threads,
            "kind": "reference", "seconds_per_step": secs,
            "sample": f"{groups} swapped groups of {SUBGROUP} params in the reference "
                      f"DirectIoEngine: read master/m/v -> adam_step_fp32 -> write back "
                      f"(simulator.cpp:453-469), median of {steps} steps after {warmup} warm-up, "
                      f"{threads} threads, storage {io / secs / 1e9:.2f} GB/s"}


def reference_arm(args, n_per_gpu, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    if args.config == "cfg5":
        res = reference_swapped_run(args, max(1, min(args.steps, 3)), 1, threads)
    elif args.precision == "pure_bf16":
        sample = min(args.cpu_sample, n_per_gpu)
        res = cpu_reference_run_bf16(sample, max(1, args.steps), max(1, args.warmup), threads)
    else:
        sample = min(args.cpu_sample, n_per_gpu)
        res = cpu_reference_run(sample, max(1, args.steps), max(1, args.warmup), threads)
    line = {
        "metric": METRIC, "value": res["value"], "unit": "params/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": res["seconds_per_step"] * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args, n_per_gpu, world),
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": "params/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "host": {"cpu": cpu_model(), "nproc": threads},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, n, world):
    name = ("llama3-8b-optimizer-state-hbm" if args.config == "cfg2" and not args.params
            else "llama3-8b-optimizer-state-hbm-inf-nan-injection" if args.config == "cfg3"
            and not args.params
            else "cfg1-64M-subgroup" if args.config == "cfg1" and not args.params
            else "qwen2.5-14b-shard-streamed-from-host" if args.config == "cfg4"
            and not args.params
            else "llama3-70b-shard-swapped-nvme+dram" if args.config == "cfg5"
            and not args.params else f"custom-{n}")
    if args.precision == "pure_bf16" and args.config != "cfg5":
        name += "-pure-bf16"
    state = ("fp32 master/m/v in the registered host pool, staged H2D/D2H"
             if args.config == "cfg4" else
             "fp32 master/m/v split between the O_DIRECT swap store and the registered host pool"
             if args.config == "cfg5" else
             "bf16 weights/m/v in HBM (OptimPrecision::pure_bf16)" if args.precision == "pure_bf16"
             else "fp32 master/m/v in HBM")
    return {"workload": name, "params_per_gpu": n, "subgroup_params": min(SUBGROUP, n),
            "grads": "bf16", "working_weights": "bf16", "state": state,
            "optimizer": "AdamW lr=1e-3 b1=0.9 b2=0.999 eps=1e-8 wd=0.01, loss scale 65536",
            "parallelism": f"zero-partition x{world} (flag all-reduce only)",
            "l2": "inputs larger than L2 (no flush needed)" if n * 14 > 4 * 126e6
            else "L2 flushed between steps"}


# --------------------------------------------------------------- our arm
class Exchange:
    """The step's cross-rank skip decision (N > 1): the library's own NCCL
    communicator (ma_comm: ncclAllReduce(max) of the flag on the compute
    stream, capturable), torch.distributed's all-reduce, or the OR fused into
    K1's last CTA over peer memory (ma_xchg)."""

    def __init__(self, mode, world, rank):
        import paper_2505_23254_b200 as mab

        self.mode, self.world = mode, world
        self.comm = self.xchg = None
        self.fallback = None
        if world > 1 and mode == "nccl" and not self._library_nccl_everywhere(mab):
            # every rank must take the same path (the communicator's creation is
            # collective): all fall back to torch.distributed, and the line says so
            self.mode, self.fallback = "torch", "libnccl.so.2 not resolvable on every rank"
        if world > 1 and self.mode == "nccl":
            self.comm = mab.NcclComm(world, rank, mab.torch_broadcast_bytes())
        elif world > 1 and mode == "p2p":
            self.xchg = mab.api.FlagExchange(world, rank, mab.api.torch_all_gather_bytes())

    @staticmethod
    def _library_nccl_everywhere(mab):
        """Whether every rank resolves libnccl.so.2 for ma_comm (one MIN
        all-reduce over torch.distributed before any rank enters the
        communicator's collective creation)."""
        import ctypes

        import torch
        import torch.distributed as dist

        buf = (ctypes.c_ubyte * mab.capi.NCCL_ID_BYTES)()
        ok = mab.capi.lib().ma_comm_unique_id(buf) == 0
        dev = torch.cuda.current_device() if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    def after_check(self, st, stream):
        import torch
        import torch.distributed as dist

        if self.comm is not None:
            st.allreduce_flag(self.comm, stream=stream)
        elif self.world > 1 and self.mode == "torch":
            with torch.cuda.stream(stream):
                dist.all_reduce(st.flag, op=dist.ReduceOp.MAX)

    @property
    def capturable(self):
        # torch's all-reduce is not ours to capture (the library's NCCL call
        # and the fused p2p exchange, whose epoch lives on the device, are)
        return not (self.world > 1 and self.mode == "torch")

    def describe(self):
        if self.world == 1:
            return "none (1 rank)"
        d = {"nccl": "ma_comm ncclAllReduce(max) of the flag (library NCCL)",
             "torch": "torch.distributed all_reduce(max) of the flag",
             "p2p": "fused into K1's last CTA over peer memory (CUDA IPC)"}[self.mode]
        return d if self.fallback is None else f"{d} (fallback: {self.fallback})"

    def close(self):
        if self.comm is not None:
            self.comm.close()
        if self.xchg is not None:
            self.xchg.close()


def ours(args, n, rank, world, local_rank):
    """configs[1] (and [0] / [2]): the state of `n` params per GPU in HBM.
    A step = K1 over the step's gradients -> cross-rank OR of the flag ->
    K2 over every sub-group -> device-side LossScaler, on one stream; with
    --graph the chain is captured once and replayed (one launch per step).
    configs[2] (--config cfg3) regenerates the gradients every step and plants
    the seeded inf/NaN plan (outside the timed segments), and checks every
    rank's decisions and loss scales against the committed plan."""
    import torch
    import torch.distributed as dist

    import paper_2505_23254_b200 as mab
    from paper_2505_23254_b200.shard import FaultPlan

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    # --precision pure_bf16: OptimPrecision::pure_bf16 (simulator.cpp:470-486)
    # — the bf16 weights are the parameters, bf16 m/v, K3 instead of K2
    bf16_state = args.precision == "pure_bf16"
    bpp = 14 if bf16_state else BYTES_PER_PARAM
    free, total = torch.cuda.mem_get_info()
    need = n * (8 if bf16_state else 16) + (1 << 30)
    if need > free:
        raise SystemExit(f"rank {rank}: need {need / 1e9:.1f} GB of HBM, {free / 1e9:.1f} free")
    sdt = torch.bfloat16 if bf16_state else torch.float32
    w = torch.empty(n, dtype=torch.bfloat16, device=dev)
    p = w if bf16_state else torch.empty(n, dtype=torch.float32, device=dev)
    m = torch.zeros(n, dtype=sdt, device=dev)
    v = torch.zeros(n, dtype=sdt, device=dev)
    g = torch.empty(n, dtype=torch.bfloat16, device=dev)
    base = rank * n
    mab.gen_seeded_weights(None if bf16_state else p, w, base=base, seed=1)
    mab.gen_pseudo_grads(g, w, step=0, base=base, seed=1, scale=65536.0)
    st = mab.Stepper(mab.AdamHyper(**HYPER), 65536.0, 2000, "bf16", "bf16", device=dev)
    sub = min(SUBGROUP, n)
    if bf16_state:
        groups = [(p[o:o + sub], m[o:o + sub], v[o:o + sub], g[o:o + sub])
                  for o in range(0, n, sub)]

        def apply_step(stream):
            st.apply_bf16(groups, stream=stream)
    else:
        groups = mab.Stepper.subgroups(
            [(p[o:o + sub], m[o:o + sub], v[o:o + sub], g[o:o + sub], w[o:o + sub])
             for o in range(0, n, sub)], "bf16", "bf16")

        def apply_step(stream):
            st.apply(groups, stream=stream)
    stream = torch.cuda.Stream(device=dev)  # non-default: capturable
    stream.wait_stream(torch.cuda.current_stream(dev))
    inject = args.config == "cfg3"
    plan = FaultPlan(n * world, sub, seed=2505) if inject else None
    flush = flush_read = None
    if n * bpp < 4 * 126e6:  # small configs: flush L2 between steps
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        flush_read = torch.empty(1, dtype=torch.int64, device=dev)
    xc = Exchange(args.flag_exchange, world, rank)
    use_graph = args.graph and xc.capturable

    def chain(with_events=None):
        if with_events:
            with_events[0].record(stream)
        st.check(g, stream=stream, xchg=xc.xchg)
        if with_events:
            with_events[1].record(stream)
        xc.after_check(st, stream)
        if with_events:
            with_events[2].record(stream)
        apply_step(stream)
        st.finish(stream=stream)
        if with_events:
            with_events[3].record(stream)

    graph = st.capture(chain, stream, reserve_steps=1 << 20) if use_graph else None

    def prepare(s):
        """Outside the timed segments: this step's gradients (+ the cfg3
        plants) and the L2 flush (small configs: 256 MB written, then read
        back so the write-back of its dirty lines also completes here)."""
        with torch.cuda.stream(stream):
            # the reference's per-step gradients (simulator.cpp:401-405: the
            # generator over the current working weights, times the current
            # device-resident loss scale)
            mab.gen_pseudo_grads(g, w, step=s, base=base, seed=1, d_scale=st.scale_t,
                                 stream=stream)
            if inject:
                for pl in plan.local(s, base, n):
                    mab.plant_bits(g, pl.index - base, pl.bits, stream=stream)
            if flush is not None:
                flush.zero_()
                torch.sum(flush.view(torch.int64), dim=0, keepdim=True, out=flush_read)

    segmented = True  # the producer (and flush) run between the timed steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    seg = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]

    def one_step(s, k=None):
        prepare(s)
        if k is not None:
            seg[k][0].record(stream)
        if graph is not None:
            graph.launch(stream)
        else:
            chain(ev[k] if k is not None else None)
        if k is not None:
            seg[k][1].record(stream)

    for s in range(args.warmup):
        one_step(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(args.steps):
            one_step(args.warmup + k, k)
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    clocks = clk.summary()
    elapsed_ms = t0.elapsed_time(t1)
    if segmented:
        # gradients produced (and L2 flushed) between steps: time the steps
        elapsed_ms = float(sum(e[0].elapsed_time(e[1]) for e in seg))
        region_ms = t0.elapsed_time(t1)
    first = args.warmup
    if graph is None:
        timed_ev = ev
        kernel_timing = "CUDA events around K1 and K2 on the launching stream, timed region"
    else:
        # inside a graph replay the kernels cannot be bracketed: K1 / K2 are
        # timed over the same number of eager steps right after the region
        timed_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)]
                    for _ in range(args.steps)]
        for k in range(args.steps):
            prepare(args.warmup + args.steps + k)
            chain(timed_ev[k])
        torch.cuda.synchronize()
        first = args.warmup + args.steps
        kernel_timing = ("CUDA events around K1 and K2 over as many eager steps right after "
                         "the graph-timed region")
    # K2 of a skipped step returns at once: average K2 over the applied steps
    applied = list(range(args.steps))
    if inject:
        of_all, _ = st.history()
        applied = [k for k in range(args.steps) if not of_all[first + k]] or applied
        kernel_timing += "; K2 averaged over the steps that applied an update"
    k1_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in timed_ev]))
    k2_ms = float(np.mean([timed_ev[k][2].elapsed_time(timed_ev[k][3]) for k in applied]))
    total_steps = args.warmup + args.steps * (2 if graph is not None else 1)
    state = st.state()
    assert state["steps"] == total_steps, state
    check = None
    if inject:
        fx = json.load(open(os.path.join(ROOT, "tests", "golden", "cfg3_plan.json")))
        if total_steps > fx["steps"]:
            raise SystemExit(f"cfg3: the committed plan covers {fx['steps']} steps")
        of, sc = st.history()
        want_of = fx["overflow"][:total_steps]
        want_sc = np.array(fx["scale_after_bits"][:total_steps], np.uint32).view(np.float32)
        ok = (of.astype(int).tolist() == want_of and
              np.array_equal(sc.view(np.uint32), want_sc.view(np.uint32)))
        res = torch.tensor([0 if ok else 1], dtype=torch.int32, device=dev)
        if world > 1:
            dist.all_reduce(res, op=dist.ReduceOp.MAX)
        if res.item():
            raise SystemExit(f"rank {rank}: cfg3 decisions / scales differ from "
                             "tests/golden/cfg3_plan.json")
        check = {"plan": "tests/golden/cfg3_plan.json (FaultPlan seed 2505 + the reference's "
                         "LossScaler)", "steps_checked": total_steps, "skipped": int(of.sum()),
                 "decisions_match": True, "scales_match": True, "ranks_agree": True,
                 "planted_this_rank": sum(len(plan.local(s, base, n)) for s in range(total_steps))}
    else:
        assert state["last_overflow"] == 0

    # max over ranks
    t = torch.tensor([elapsed_ms, k1_ms, k2_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms, k1_ms, k2_ms = t.tolist()
    ms_per_step = elapsed_ms / args.steps

    # ---- e2e: gradients from pinned host memory through the public API
    e2e = None
    if args.e2e_steps > 0 and not inject:
        # the gradient flat buffer in alignment-free registered host memory
        # (§4.3; torch's pin_memory would round 16.06 GB up to 32 GiB)
        g_buf = mab.aligned_host_buffer(n * 2, register=True)
        g_host = torch.from_numpy(g_buf.view(np.int16))
        g_host.copy_(g.view(torch.int16), non_blocking=False)
        g_host = g_host.view(torch.bfloat16)
        res_host = torch.empty(16, dtype=torch.uint8, pin_memory=True)
        # speculative updates while the gradients stream in (fp32 state):
        # the leading sub-groups whose state fits a backup in the free HBM
        spec_groups, backup = 0, None
        if not args.no_e2e_spec:
            al = lambda b: (b + 255) // 256 * 256  # noqa: E731
            need = [3 * al(2 * min(sub, n - o)) if bf16_state else
                    3 * al(4 * min(sub, n - o)) + al(2 * min(sub, n - o))
                    for o in range(0, n, sub)][:96]
            room = torch.cuda.mem_get_info()[0] - (2 << 30)
            while spec_groups < len(need) and sum(need[:spec_groups + 1]) <= room:
                spec_groups += 1
            if spec_groups:
                backup = torch.empty(sum(need[:spec_groups]), dtype=torch.uint8, device=dev)

        spec_arr = st.subgroups_bf16(groups) if bf16_state else groups

        def e2e_step():
            if backup is not None and bf16_state:
                st.check_from_host_spec_bf16(g_host, g, spec_arr, backup, stream=stream)
            elif backup is not None:
                st.check_from_host_spec(g_host, g, spec_arr, backup, stream=stream)
            else:
                st.check_from_host(g_host, g, stream=stream)
            if xc.xchg is not None:
                st.check(None, stream=stream, xchg=xc.xchg)  # exchange-only K1 launch
            xc.after_check(st, stream)
            if backup is not None and bf16_state:
                st.apply_spec_bf16(spec_arr, stream=stream)
            elif backup is not None:
                st.apply_spec(spec_arr, stream=stream)
            else:
                apply_step(stream)
            st.finish(stream=stream)
            with torch.cuda.stream(stream):
                res_host.copy_(st.state_t[:16], non_blocking=True)  # flag/scale readback

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        e2e_ms = torch.tensor([a.elapsed_time(b) / args.e2e_steps], dtype=torch.float64,
                              device=dev)
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e_ms = float(e2e_ms.item())
        e2e = {"value": n * world / (e2e_ms / 1e3), "unit": "params/s",
               "h2d_bytes_per_step": n * 2, "d2h_bytes_per_step": 16,
               "ms_per_step": e2e_ms,
               "path": "pinned host bf16 grads -> chunked H2D overlapped with K1 "
                       + ("and with the speculative K2 of every landed sub-group whose state "
                          "fits the backup (ma_stepper_check_host_spec[_bf16]_async) -> flag "
                          f"exchange -> {'K3' if bf16_state else 'K2'} over the rest, restore on "
                          "a skip (ma_stepper_apply_spec[_bf16]_async)"
                          if backup is not None else
                          "(ma_stepper_check_host_async) -> flag exchange -> "
                          f"{'K3' if bf16_state else 'K2'} over HBM-resident state")
                       + " -> D2H of the step's flag/loss-scale",
               "speculated_subgroups": spec_groups, "subgroups": len(groups),
               "backup_bytes": 0 if backup is None else backup.numel()}
        del backup
        del g_host
        mab.host_unregister(g_buf)
    if graph is not None:
        graph.close()
    xc.close()

    if rank != 0:
        return
    peak, peak_kind = peaks()
    alg_bytes = bpp * n
    k2_gbs = alg_bytes / (k2_ms / 1e3) / 1e9
    # K1 + K2 launches (96 sub-groups per launch) + finish, plus the producer
    # (k_gen_grads) and cfg3's k_plant launches between the timed segments
    launches_per_step = 1 + (len(groups) + 95) // 96 + 1 + 1
    plants = (sum(len(plan.local(args.warmup + k, base, n)) for k in range(args.steps))
              if inject else 0)
    # DRAM bytes per launch of K2 = ncu's dram__bytes_{read,write}.sum per param
    # (one `ncu --set full` capture, profiles/*_ncu_summary.json) x params/launch
    traffic = None
    for name in sorted(os.listdir(os.path.join(ROOT, "profiles")), reverse=True):
        if name.endswith("_ncu_summary.json"):
            try:
                summ = json.load(open(os.path.join(ROOT, "profiles", name)))
                tag = "k3_" if bf16_state else "k2_"
                k2 = next(v for v in summ.values() if tag in v.get("Kernel Name", ""))
                traffic = k2["dram_bytes_per_param"] * n
                break
            except Exception:
                traffic = None
    cfg = workload_config(args, n, world)
    cfg.update(flag_exchange=xc.describe(), graph=graph is not None,
               gradients="regenerated every step outside the timed segments (the reference's "
                         "pseudo_gradient over the current weights x the device loss scale)")
    if flush is not None:
        cfg["l2"] = ("L2 flushed between steps (256 MB written then read back, outside the "
                     "timed segments)")
    line = {
        "metric": METRIC,
        "value": n * world / (ms_per_step / 1e3),
        "unit": "params/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "region_ms_incl_producer": region_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (reference generators seeded_weight/pseudo_gradient)",
        "config": cfg,
        "hbm_gbs_per_gpu": alg_bytes / (ms_per_step / 1e3) / 1e9,
        "roofline": {"bound": "hbm",
                     "kernel": ("k3_v2 (K3 fused unscale+AdamW on bf16 weights/m/v)" if bf16_state
                                else "k2_oneshot (K2 fused unscale+AdamW+cast)"),
                     "achieved": k2_gbs, "peak": peak, "unit": "GB/s",
                     "frac": k2_gbs / peak, "traffic": traffic,
                     "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                     "bytes_per_param": bpp, "params_per_launch": n,
                     "k2_ms": k2_ms, "k1_ms": k1_ms, "kernel_timing": kernel_timing,
                     "k1_gbs": 2 * n / (k1_ms / 1e3) / 1e9,
                     "step_frac": alg_bytes / (ms_per_step / 1e3) / 1e9 / peak},
        "gpu_launches": launches_per_step * args.steps + plants,
        "clocks": clocks,
        "e2e": e2e,
    }
    if check is not None:
        line["cfg3_check"] = check
    if world == 1 and not args.no_cpu_baseline and not inject and bf16_state:
        threads = os.cpu_count() or 1
        cb = cpu_reference_run_bf16(min(args.cpu_sample, n), 5, 1, threads)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        line["host"] = {"cpu": cpu_model(), "nproc": threads}
    elif world == 1 and not args.no_cpu_baseline and not inject:
        threads = os.cpu_count() or 1
        cb = cpu_reference_run(min(args.cpu_sample, n), 5, 1, threads)  # >= 5
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        # the reference's path at 1 worker too (the reference's
        # simulator calls adam_step_fp32 with its default workers = 1)
        one = cpu_reference_run(min(args.cpu_sample, n), 5, 1, 1)
        line["cpu_baseline"]["single_thread"] = {"value": one["value"], "unit": "params/s",
                                                 "cores": 1}
        line["host"] = {"cpu": cpu_model(), "nproc": threads}
    print(json.dumps(line), flush=True)


def host_grads_e2e(args, st, g, n, world, rank, dev, stream, step_rest):
    """The same step end to end through the public API: this step's bf16
    gradients come from registered (pinned) host memory —
    ma_stepper_check_host_async copies them in chunks with K1 overlapped —
    then `step_rest()` (exchange, update, scaler) and a D2H of the step's
    flag / loss scale.  Returns (ms per step, max over ranks)."""
    import torch
    import torch.distributed as dist

    import paper_2505_23254_b200 as mab

    g_buf = mab.aligned_host_buffer(n * 2, register=True)
    g_host = torch.from_numpy(g_buf.view(np.int16))
    g_host.copy_(g.view(torch.int16), non_blocking=False)
    g_host = g_host.view(torch.bfloat16)
    res_host = torch.empty(16, dtype=torch.uint8, pin_memory=True)

    def e2e_step():
        st.check_from_host(g_host, g, stream=stream)
        step_rest()
        with torch.cuda.stream(stream):
            res_host.copy_(st.state_t[:16], non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    b.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / args.e2e_steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    del g_host
    mab.host_unregister(g_buf)  # before the pages go back to the allocator
    return float(ms.item())


def ours_streamed(args, n, rank, world, local_rank):
    """configs[3]: Qwen2.5-14B-shaped state sharded 8 ways (1.85 B params per
    GPU); fp32 p/m/v live in the drop-in memascend::Pool (adaptive,
    alignment-free, cudaHostRegister'd: include/memascend/state_pool.h, one
    checked-out slot per sub-group tensor), grads and working weights in HBM;
    every 100 M sub-group is staged H2D -> K2 -> D2H through `--slots`
    device slots.  Bound: the host link, 24 B/param (12 in, 12 out)."""
    import torch
    import torch.distributed as dist

    import paper_2505_23254_b200 as mab

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    sub = min(SUBGROUP, n)
    t_init = time.perf_counter()
    pool = mab.StatePool(n, sub)
    pstats = pool.stats()
    pinned_pow2 = 3 * sum(1 << (min(sub, n - o) * 4 - 1).bit_length() for o in range(0, n, sub))
    g = torch.empty(n, dtype=torch.bfloat16, device=dev)
    w = torch.empty(n, dtype=torch.bfloat16, device=dev)
    base = rank * n
    tmp = torch.empty(sub, dtype=torch.float32, device=dev)
    groups = []
    for k, o in enumerate(range(0, n, sub)):
        ln = min(sub, n - o)
        (ph, _), (mh, _), (vh, _) = (pool.tensor(k, i) for i in range(3))
        mab.gen_seeded_weights(tmp[:ln], w[o:o + ln], base=base + o, seed=1)
        ph.copy_(tmp[:ln])  # m and v slots are zero (the allocator's fill)
        groups.append((ph, mh, vh, g[o:o + ln], w[o:o + ln]))
    del tmp
    t_init = time.perf_counter() - t_init
    st = mab.Stepper(mab.AdamHyper(**HYPER), 65536.0, 2000, "bf16", "bf16", device=dev)
    arr = mab.Stepper.subgroups(groups, "bf16", "bf16")
    slot = args.slot_params
    staging = torch.empty(3 * args.slots * slot, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    stream.wait_stream(torch.cuda.current_stream(dev))
    xc = Exchange(args.flag_exchange, world, rank)

    def rest():
        xc.after_check(st, stream)
        st.apply_streamed(arr, staging, slot, args.slots, stream=stream)
        st.finish(stream=stream)

    seg = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]

    def one_step(s, k=None):
        mab.gen_pseudo_grads(g, w, step=s, base=base, seed=1, d_scale=st.scale_t, stream=stream)
        if k is not None:
            seg[k][0].record(stream)
        st.check(g, stream=stream, xchg=xc.xchg)
        rest()
        if k is not None:
            seg[k][1].record(stream)

    for s in range(args.warmup):
        one_step(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            one_step(args.warmup + k, k)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = torch.tensor([sum(e[0].elapsed_time(e[1]) for e in seg) / args.steps],
                      dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    e2e = None
    if args.e2e_steps > 0:
        e2e_ms = host_grads_e2e(args, st, g, n, world, rank, dev, stream, rest)
        e2e = {"value": n * world / (e2e_ms / 1e3), "unit": "params/s",
               "h2d_bytes_per_step": n * 2 + 12 * n, "d2h_bytes_per_step": 12 * n + 16,
               "ms_per_step": e2e_ms,
               "path": "pinned host bf16 grads -> chunked H2D overlapped with K1 -> flag "
                       "exchange -> p/m/v slots of the registered memascend::Pool streamed "
                       "H2D -> K2 -> D2H (ma_stepper_apply_streamed) -> D2H of flag/scale"}

    # measured host-link ceiling: concurrent pinned H2D + D2H of 1 GiB each
    hb = torch.empty(1 << 28, dtype=torch.float32, pin_memory=True)
    hb2 = torch.empty(1 << 28, dtype=torch.float32, pin_memory=True)
    db = torch.empty(1 << 28, dtype=torch.float32, device=dev)
    db2 = torch.empty(1 << 28, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    best = 0.0
    for _ in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s1.wait_stream(stream)
        s2.wait_stream(stream)
        with torch.cuda.stream(s1):
            db.copy_(hb, non_blocking=True)
        with torch.cuda.stream(s2):
            hb2.copy_(db2, non_blocking=True)
        stream.wait_stream(s1)
        stream.wait_stream(s2)
        e1.record(stream)
        torch.cuda.synchronize()
        best = max(best, 2 * (1 << 30) / (e0.elapsed_time(e1) / 1e3) / 1e9)
    xc.close()
    if rank != 0:
        pool.close()
        return
    link = 24 * n / (ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": n * world / (ms / 1e3), "unit": "params/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generators seeded_weight/pseudo_gradient)",
        "config": dict(workload_config(args, n, world), slots=args.slots, slot_params=slot,
                       flag_exchange=xc.describe(),
                       state_pool="memascend::Pool (adaptive, alignment-free, registered), "
                                  f"{pstats['classes']} slot classes, every master/m/v "
                                  "sub-group tensor a checked-out slot"),
        "pinned_host_bytes": {"pool_backing": pstats["backing_bytes"],
                              "pool_payload": pstats["capacity_bytes"],
                              "torch_pin_memory_would_take": pinned_pow2},
        "roofline": {"bound": "host-link", "achieved": link, "unit": "GB/s", "peak": best,
                     "frac": link / best, "traffic": None, "bytes_per_param": 24,
                     "peak_source": "measured concurrent pinned H2D+D2H, 1 GiB each"},
        "init_seconds": t_init,
        "gpu_launches": (1 + ((n + slot - 1) // slot) + 1 + 1) * args.steps,  # + producer
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    pool.close()
    print(json.dumps(line), flush=True)


def storage_peak(store_dir, io_workers, io_depth, key_bytes=1 << 30, keys=4):
    """Measured O_DIRECT bandwidth of the swap device through the same engine
    and settings: `keys` keys written concurrently (write), read back
    concurrently (read), then half rewritten while the other half is read
    (mixed — the pipeline's own pattern, its bound).  Returns GB/s dict."""
    import shutil

    import paper_2505_23254_b200 as mab

    d = os.path.join(store_dir, "peak")
    devs = mab.DirectIoEngine.create_virtual_devices(d, 2, keys * key_bytes // 2 + (16 << 20))
    bufs = [mab.aligned_host_buffer(key_bytes) for _ in range(keys)]
    for b in bufs:
        b[:] = 7
    out = {}
    try:
        with mab.DirectIoEngine(devs, workers=io_workers, queue_depth=io_depth) as e:
            def timed(ops):
                t0 = time.perf_counter()
                for op in [f() for f in ops]:
                    op.wait()
                return keys * key_bytes / (time.perf_counter() - t0) / 1e9

            out["write"] = timed([lambda i=i: e.write_tensor_async(f"k{i}", bufs[i], key_bytes)
                                  for i in range(keys)])
            out["read"] = timed([lambda i=i: e.read_tensor_async(f"k{i}", bufs[i])
                                 for i in range(keys)])
            out["mixed"] = timed([(lambda i=i: e.write_tensor_async(f"k{i}", bufs[i], key_bytes))
                                  if i % 2 else (lambda i=i: e.read_tensor_async(f"k{i}", bufs[i]))
                                  for i in range(keys)])
    finally:
        shutil.rmtree(d, ignore_errors=True)
    return out


def ours_zero_fused(args, n, rank, world, local_rank):
    """Data-parallel ZeRO step with no collective call (tests/test_zero_step.py
    checks it bit for bit): every rank holds full-length bf16 gradients and
    the full working weights; per step K4 reduce-scatters the gradients with
    the overflow check in its epilogue (peers read over NVLink through CUDA
    IPC, the skip decision OR-ed by its last CTA), K2 updates this rank's
    partition and stores the new weights into every rank's buffer, the
    scaler advances.  Weak scaling: `n` params per rank.  Per rank and param:
    world x 2 B gradient reads (world-1 of them remote) + 2 B write (K4),
    28 B in HBM + (world-1) x 2 B remote weight stores (K2)."""
    import torch
    import torch.distributed as dist

    import paper_2505_23254_b200 as mab

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    total = n * world
    G = torch.empty(total, dtype=torch.bfloat16, device=dev)
    W = torch.empty(total, dtype=torch.bfloat16, device=dev)
    base = rank * n
    p = torch.empty(n, dtype=torch.float32, device=dev)
    m = torch.zeros(n, dtype=torch.float32, device=dev)
    v = torch.zeros(n, dtype=torch.float32, device=dev)
    gp = torch.empty(n, dtype=torch.bfloat16, device=dev)
    mab.gen_seeded_weights(None, W, n=total, seed=1)
    mab.gen_seeded_weights(p, W[base:base + n], base=base, seed=1)
    # this rank's micro-batch gradients: the generator seeded per rank
    mab.gen_pseudo_grads(G, W, step=0, seed=1 + rank, scale=65536.0)
    gather = (mab.api.torch_all_gather_bytes() if world > 1 else (lambda b: [b]))
    rs = mab.api.GradReduceScatter(world, rank, G, gather)
    ag = mab.api.GradReduceScatter(world, rank, W, gather)
    st = mab.Stepper(mab.AdamHyper(**HYPER), 65536.0, 2000, "bf16", "bf16", device=dev)
    sub = min(SUBGROUP, n)
    w = W[base:base + n]
    groups = mab.Stepper.subgroups(
        [(p[o:o + sub], m[o:o + sub], v[o:o + sub], gp[o:o + sub], w[o:o + sub])
         for o in range(0, n, sub)])
    stream = torch.cuda.current_stream(dev)

    def one_step():
        st.reduce_scatter(rs, base, n, gp, post_scale=1.0 / world)
        st.apply_allgather(groups, ag)
        st.finish()

    ms, _, clocks, _ = timed_swapped_steps(args, one_step, None, stream, dev, world, local_rank)
    skipped = bool(st.state()["last_overflow"])
    timed_out = rs.timed_out() or ag.timed_out()
    rs.close()
    ag.close()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": n * world / (ms / 1e3), "unit": "params/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generators seeded_weight/pseudo_gradient, per-rank seeds)",
        "config": dict(workload_config(args, n, world),
                       workload=f"zero-fused-{n}-per-rank",
                       parallelism=f"zero x{world}: K4 reduce-scatter+check, K2 update+all-gather "
                                   "over peer memory (no collective call)"),
        "hbm_bytes_per_param": {"k4": world * 2 + 2, "k2": 28},
        "remote_bytes_per_param": {"k4_reads": (world - 1) * 2, "k2_stores": (world - 1) * 2},
        "last_step_skipped": skipped, "peer_timeout": timed_out,
        "gpu_launches": 5 * args.steps,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def timed_swapped_steps(args, one_step, store, stream, dev, world, local_rank):
    """W warm-up steps, then K timed steps between barriers (CUDA events on
    the compute stream, max over ranks); returns (ms per step, swap-store
    bytes moved per step, clocks, backend)."""
    import torch
    import torch.distributed as dist

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    io0 = store.stats() if store else {}
    with ClockSampler(local_rank) as clk:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            one_step()
        b.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    io1 = store.stats() if store else {}
    ms = torch.tensor([a.elapsed_time(b) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    io_bytes = ((io1.get("bytes_read", 0) - io0.get("bytes_read", 0)) +
                (io1.get("bytes_written", 0) - io0.get("bytes_written", 0))) / args.steps
    return float(ms.item()), io_bytes, clk.summary(), (store.backend if store else None)


def storage_report(args, io_bytes, ms, bytes_per_swapped_param):
    """Swap-device rate of the step against the device's measured mixed
    read/write rate (equal bytes read and written concurrently bound it)."""
    pk = storage_peak(args.swap_dir, args.io_workers, args.io_depth)
    gbs = io_bytes / (ms / 1e3) / 1e9
    return {"bound": "swap-device", "achieved": gbs, "unit": "GB/s", "peak": pk["mixed"],
            "frac": gbs / pk["mixed"], "bytes_per_step": io_bytes,
            "bytes_per_swapped_param": bytes_per_swapped_param,
            "peak_read_gbs": pk["read"], "peak_write_gbs": pk["write"],
            "peak_source": "measured O_DIRECT through the engine, same settings: 4 x 1 GiB keys, "
                           "2 rewritten while 2 are read"}


def storage_roofline(sr):
    """The swapped step's roofline: the swap device (bytes moved per step
    from the store's own request counters) against its measured mixed
    read/write rate through the same engine and settings."""
    return {"bound": "swap-device", "achieved": sr["achieved"], "peak": sr["peak"],
            "unit": "GB/s", "frac": sr["frac"], "traffic": sr["bytes_per_step"],
            "bytes_per_swapped_param": sr["bytes_per_swapped_param"],
            "peak_source": sr["peak_source"]}


def ours_swapped(args, n, rank, world, local_rank):
    """configs[4]: Llama-3-70B-shaped state sharded 8 ways (8.82 B params per
    GPU).  fp32 master/m/v of `--swap-gb` worth of 100 M sub-groups live in
    the O_DIRECT swap store (memascend DirectIoEngine drop-in, io_uring
    backend, file-backed devices under --swap-dir), the rest in the
    registered host pool; grads and working weights in HBM.
    ma_stepper_apply_swapped reads swapped groups into registered host slots
    ahead of use, streams every group H2D -> K2 -> D2H and writes swapped
    groups back from a writer thread.  Bound: the swap device (24 B per
    swapped param) and the host link (24 B per param)."""
    import shutil

    import torch
    import torch.distributed as dist

    import paper_2505_23254_b200 as mab

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    sub = min(SUBGROUP, n)
    tb = (sub * 4 + 4095) // 4096 * 4096
    offs = list(range(0, n, sub))
    G = len(offs)
    S = min(G, int(args.swap_gb * 1e9 // (3 * tb)))
    swapped = set(int(i * G / S) for i in range(S)) if S else set()
    base = rank * n
    sdir = os.path.join(args.swap_dir, f"rank{rank}")
    shutil.rmtree(sdir, ignore_errors=True)
    per_dev = ((3 * tb * len(swapped)) // 2 + (64 << 20)) // 4096 * 4096
    devs = mab.DirectIoEngine.create_virtual_devices(sdir, 2, per_dev) if swapped else []
    store = (mab.DirectIoEngine(devs, workers=args.io_workers, queue_depth=args.io_depth)
             if swapped else None)
    host_ids = [k for k in range(G) if k not in swapped]
    n_host = sum(min(sub, n - offs[k]) for k in host_ids)
    pool = {}
    for name in ("p", "m", "v"):  # the DRAM tier: one registered region per tensor
        buf = mab.aligned_host_buffer(max(4, n_host * 4), register=True)
        pool[name] = buf.view(np.float32)
    pool["m"][:] = 0
    pool["v"][:] = 0
    g = torch.empty(n, dtype=torch.bfloat16, device=dev)
    w = torch.empty(n, dtype=torch.bfloat16, device=dev)
    hslots = args.host_slots
    hstage = mab.aligned_host_buffer(hslots * 3 * tb, register=True)
    dstage = torch.empty(3 * args.slots * sub, dtype=torch.float32, device=dev)
    tmp = torch.empty(sub, dtype=torch.float32, device=dev)
    zeros = mab.aligned_host_buffer(tb)
    zeros[:] = 0
    groups = []
    at = 0
    t_init = time.perf_counter()
    for k, o in enumerate(offs):
        ln = min(sub, n - o)
        mab.gen_seeded_weights(tmp[:ln], w[o:o + ln], base=base + o, seed=1)
        if k in swapped:
            pslot = hstage[:tb].view(np.float32)
            pslot[:ln] = tmp[:ln].cpu().numpy()
            keys = tuple(f"{t}.g{k}" for t in ("master", "m", "v"))
            store.write_tensor(keys[0], hstage[:tb], ln * 4)
            store.write_tensor(keys[1], zeros, ln * 4)
            store.write_tensor(keys[2], zeros, ln * 4)
            groups.append((keys, g[o:o + ln], w[o:o + ln]))
        else:
            pool["p"][at:at + ln] = tmp[:ln].cpu().numpy()
            groups.append(((pool["p"][at:at + ln], pool["m"][at:at + ln],
                            pool["v"][at:at + ln]), g[o:o + ln], w[o:o + ln]))
            at += ln
    del tmp
    t_init = time.perf_counter() - t_init
    mab.gen_pseudo_grads(g, w, step=0, base=base, seed=1, scale=65536.0)
    st = mab.Stepper(mab.AdamHyper(**HYPER), 65536.0, 2000, "bf16", "bf16", device=dev)
    stream = torch.cuda.current_stream(dev)

    xc = Exchange(args.flag_exchange, world, rank)

    def rest():
        xc.after_check(st, stream)
        st.apply_swapped(store, groups, hstage, hslots, dstage, args.slots, sub, stream=stream)
        st.finish(stream=stream)

    def one_step():
        st.check(g, stream=stream, xchg=xc.xchg)
        rest()

    try:
        ms, io_bytes, clocks, backend = timed_swapped_steps(args, one_step, store, stream, dev,
                                                            world, local_rank)
        e2e = None
        if args.e2e_steps > 0:
            e2e_ms = host_grads_e2e(args, st, g, n, world, rank, dev, stream, rest)
            n_sw_ = n - n_host
            e2e = {"value": n * world / (e2e_ms / 1e3), "unit": "params/s",
                   "h2d_bytes_per_step": n * 2 + 12 * n, "d2h_bytes_per_step": 12 * n + 16,
                   "storage_bytes_per_step": 24 * n_sw_, "ms_per_step": e2e_ms,
                   "path": "pinned host bf16 grads -> chunked H2D overlapped with K1 -> flag "
                           "exchange -> swapped groups read from the O_DIRECT store into "
                           "registered host slots, every group H2D -> K2 -> D2H, swapped groups "
                           "written back (ma_stepper_apply_swapped) -> D2H of flag/scale"}
        if store:
            store.close()
    finally:
        shutil.rmtree(sdir, ignore_errors=True)
        xc.close()
    if rank != 0:
        return
    n_sw = n - n_host
    line = {
        "metric": METRIC, "value": n * world / (ms / 1e3), "unit": "params/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generators seeded_weight/pseudo_gradient)",
        "config": dict(workload_config(args, n, world), swapped_params=n_sw,
                       dram_params=n_host, swapped_groups=len(swapped), groups=G,
                       host_slots=hslots, dev_slots=args.slots, io_backend=backend,
                       io_workers=args.io_workers, io_depth=args.io_depth),
        "storage": storage_report(args, io_bytes, ms, 24),
        "host_link": {"achieved": 24 * n / (ms / 1e3) / 1e9, "unit": "GB/s",
                      "bytes_per_param": 24},
        "init_seconds": t_init,
        "gpu_launches": (1 + G + 1) * args.steps,
        "clocks": clocks,
        "e2e": e2e,
    }
    line["roofline"] = storage_roofline(line["storage"])
    if world == 1 and not args.no_cpu_baseline:
        res = reference_swapped_run(args, 2, 1, os.cpu_count() or 1)
        line["cpu_baseline"] = {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")}
    print(json.dumps(line), flush=True)


def ours_swapped_bf16(args, n, rank, world, local_rank):
    """configs[4] in the reference's pure-bf16 mode (SURVEY §8(f) row 1,
    simulator.cpp:470-486): bf16 weights in HBM updated in place by K3, bf16
    m/v of `--swap-gb` worth of sub-groups in the swap store, the rest in the
    registered DRAM pool.  8 B per swapped parameter on the storage device
    instead of 24."""
    import shutil

    import torch
    import torch.distributed as dist

    import paper_2505_23254_b200 as mab

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    sub = min(SUBGROUP, n)
    tb = (sub * 2 + 4095) // 4096 * 4096
    offs = list(range(0, n, sub))
    G = len(offs)
    S = min(G, int(args.swap_gb * 1e9 // (2 * tb)))
    swapped = set(int(i * G / S) for i in range(S)) if S else set()
    base = rank * n
    sdir = os.path.join(args.swap_dir, f"rank{rank}")
    shutil.rmtree(sdir, ignore_errors=True)
    per_dev = ((2 * tb * len(swapped)) // 2 + (64 << 20)) // 4096 * 4096
    devs = mab.DirectIoEngine.create_virtual_devices(sdir, 2, per_dev) if swapped else []
    store = (mab.DirectIoEngine(devs, workers=args.io_workers, queue_depth=args.io_depth)
             if swapped else None)
    host_ids = [k for k in range(G) if k not in swapped]
    n_host = sum(min(sub, n - offs[k]) for k in host_ids)
    pool = {}
    for name in ("m", "v"):
        buf = mab.aligned_host_buffer(max(8, n_host * 2), register=True)
        buf[:] = 0
        pool[name] = buf.view(np.uint16)
    w = torch.empty(n, dtype=torch.bfloat16, device=dev)
    g = torch.empty(n, dtype=torch.bfloat16, device=dev)
    mab.gen_seeded_weights(None, w, n=n, base=base, seed=1)
    zeros = mab.aligned_host_buffer(tb)
    zeros[:] = 0
    groups = []
    at = 0
    t_init = time.perf_counter()
    for k, o in enumerate(offs):
        ln = min(sub, n - o)
        if k in swapped:
            keys = (f"m.g{k}", f"v.g{k}")
            for key in keys:
                store.write_tensor(key, zeros, ln * 2)
            groups.append((keys, w[o:o + ln], g[o:o + ln]))
        else:
            groups.append(((pool["m"][at:at + ln], pool["v"][at:at + ln]), w[o:o + ln],
                           g[o:o + ln]))
            at += ln
    t_init = time.perf_counter() - t_init
    mab.gen_pseudo_grads(g, w, step=0, base=base, seed=1, scale=65536.0)
    st = mab.Stepper(mab.AdamHyper(**HYPER), 65536.0, 2000, "bf16", "none", device=dev)
    hslots = args.host_slots
    hstage = mab.aligned_host_buffer(hslots * 2 * tb, register=True)
    dstage = torch.empty(2 * args.slots * sub, dtype=torch.int16, device=dev)
    stream = torch.cuda.current_stream(dev)

    xc = Exchange(args.flag_exchange, world, rank)

    def rest():
        xc.after_check(st, stream)
        st.apply_swapped_bf16(store, groups, hstage, hslots, dstage, args.slots, sub,
                              stream=stream)
        st.finish(stream=stream)

    def one_step():
        st.check(g, stream=stream, xchg=xc.xchg)
        rest()

    try:
        ms, io_bytes, clocks, backend = timed_swapped_steps(args, one_step, store, stream, dev,
                                                            world, local_rank)
        e2e = None
        if args.e2e_steps > 0:
            e2e_ms = host_grads_e2e(args, st, g, n, world, rank, dev, stream, rest)
            e2e = {"value": n * world / (e2e_ms / 1e3), "unit": "params/s",
                   "h2d_bytes_per_step": n * 2 + 4 * n, "d2h_bytes_per_step": 4 * n + 16,
                   "ms_per_step": e2e_ms,
                   "path": "pinned host bf16 grads -> chunked H2D overlapped with K1 -> flag "
                           "exchange -> bf16 m/v streamed from the store / DRAM tier, K3 on "
                           "HBM-resident bf16 weights (ma_stepper_apply_swapped_bf16) -> D2H "
                           "of flag/scale"}
        if store:
            store.close()
    finally:
        shutil.rmtree(sdir, ignore_errors=True)
        xc.close()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": n * world / (ms / 1e3), "unit": "params/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (reference generators seeded_weight/pseudo_gradient)",
        "config": dict(workload_config(args, n, world), optimizer_precision="pure_bf16",
                       state="bf16 weights in HBM; bf16 m/v split between the O_DIRECT swap "
                             "store and the registered host pool",
                       swapped_params=n - n_host, dram_params=n_host,
                       swapped_groups=len(swapped), groups=G, host_slots=hslots,
                       dev_slots=args.slots, io_backend=backend, io_workers=args.io_workers,
                       io_depth=args.io_depth),
        "storage": storage_report(args, io_bytes, ms, 8),
        "host_link": {"achieved": 8 * n / (ms / 1e3) / 1e9, "unit": "GB/s",
                      "bytes_per_param": 8},
        "init_seconds": t_init,
        "gpu_launches": (1 + G + 1) * args.steps,
        "clocks": clocks,
        "e2e": e2e,
    }
    line["roofline"] = storage_roofline(line["storage"])
    print(json.dumps(line), flush=True)


def launch_ranks(args):
    """`bench.py --gpus N` without a launcher: re-execute under
    torch.distributed.run with N ranks (one per GPU) on 127.0.0.1 and exit
    with its status.  Guards: N must not exceed the visible GPUs (our arm;
    the MA_BENCH_DEVICE test hook puts every rank on one device)."""
    import socket

    if args.impl == "ours" and "MA_BENCH_DEVICE" not in os.environ:
        import torch

        have = torch.cuda.device_count()
        if args.gpus > have:
            print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) are visible",
                  file=sys.stderr, flush=True)
            sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        launch_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr, flush=True)
        sys.exit(2)
    # the NCCL communicators log their init (incl. "nranks N") unless the
    # caller chose otherwise
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    # test hooks for the N>1 path on a single GPU (tests/ only): every rank on
    # MA_BENCH_DEVICE, collectives over MA_BENCH_BACKEND (gloo); default nccl
    hook = "MA_BENCH_DEVICE" in os.environ
    local_rank = int(os.environ.get("MA_BENCH_DEVICE", local_rank))
    backend = os.environ.get("MA_BENCH_BACKEND", "nccl")
    n = args.params or {"cfg2": LLAMA3_8B, "cfg1": CFG1, "cfg3": LLAMA3_8B,
                        "cfg4": (QWEN25_14B + 7) // 8, "cfg5": (LLAMA3_70B + 7) // 8}[args.config]
    if args.impl == "reference":
        reference_arm(args, n, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        if not hook and world > torch.cuda.device_count():
            print(f"bench.py: {world} ranks but {torch.cuda.device_count()} CUDA device(s)",
                  file=sys.stderr, flush=True)
            sys.exit(2)
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
        if hook and args.flag_exchange == "nccl":
            # NCCL cannot put two ranks on one GPU: the single-GPU test hook
            # exchanges the flag through torch.distributed instead
            args.flag_exchange = "torch"
    try:
        if args.zero_fused:
            ours_zero_fused(args, args.params or 1_000_000_000, rank, world, local_rank)
        elif args.config == "cfg4":
            ours_streamed(args, n, rank, world, local_rank)
        elif args.config == "cfg5" and args.precision == "pure_bf16":
            ours_swapped_bf16(args, n, rank, world, local_rank)
        elif args.config == "cfg5":
            ours_swapped(args, n, rank, world, local_rank)
        else:
            ours(args, n, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()

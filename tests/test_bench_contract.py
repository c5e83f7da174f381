"""bench.py contract: one JSON line from rank 0 with the required keys.

The CPU test exercises the reference arm (the reference's CPU path on a tiny
sample) at N=1 and under torchrun N=2 (rank 0 prints, rank 1 exits quietly).
The GPU test runs our arm at N=1 and the N=2 path on one GPU with gloo
(MA_BENCH_BACKEND / MA_BENCH_DEVICE test hooks)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return str(s.getsockname()[1])


def run(args, nproc=1, env=None, timeout=600):
    e = dict(os.environ, **(env or {}))
    if nproc == 1:
        cmd = [sys.executable, "bench.py"] + args
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1", "--master-port",
               port(), "bench.py", "--gpus", str(nproc)] + args
    p = subprocess.run(cmd, cwd=ROOT, env=e, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("nproc", [1, 2])
def test_reference_arm_line(nproc):
    j = run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--cpu-sample", "1000000"],
            nproc=nproc)
    assert REQUIRED <= set(j)
    assert j["impl"] == "reference" and j["value"] > 0
    assert j["cpu_baseline"]["kind"] in ("reference", "port") and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_line_n1():
    j = run(["--params", "200000000", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
             "--cpu-sample", "1000000"])
    assert REQUIRED <= set(j) and {"roofline", "cpu_baseline", "clocks", "gpu_launches"} <= set(j)
    r = j["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.2 and r["unit"] == "GB/s"
    assert j["e2e"]["h2d_bytes_per_step"] == 2 * 200000000 and j["gpu_launches"] > 0


@pytest.mark.gpu
def test_our_arm_two_ranks_one_gpu_gloo():
    j = run(["--params", "100000000", "--steps", "3", "--warmup", "3", "--e2e-steps", "1"],
            nproc=2, env={"MA_BENCH_BACKEND": "gloo", "MA_BENCH_DEVICE": "0"})
    assert j["n_gpus"] == 2 and j["scaling"] == "weak" and j["value"] > 0


@pytest.mark.gpu
def test_our_arm_two_ranks_one_gpu_p2p_exchange():
    j = run(["--params", "100000000", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
             "--flag-exchange", "p2p"],
            nproc=2, env={"MA_BENCH_BACKEND": "gloo", "MA_BENCH_DEVICE": "0"})
    assert j["n_gpus"] == 2 and j["value"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("nproc", [1, 2])
def test_zero_fused_line(nproc):
    """--zero-fused: the ZeRO step over peer memory (K4 + K2-AG), every rank
    as a process on one GPU for nproc 2."""
    env = {"MA_BENCH_BACKEND": "gloo", "MA_BENCH_DEVICE": "0"} if nproc > 1 else None
    j = run(["--zero-fused", "--params", "50000000", "--steps", "3", "--warmup", "3"],
            nproc=nproc, env=env)
    assert REQUIRED - {"e2e"} <= set(j) and j["n_gpus"] == nproc and j["value"] > 0
    assert not j["peer_timeout"] and j["remote_bytes_per_param"]["k2_stores"] == 2 * (nproc - 1)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["mixed", "pure_bf16"])
def test_cfg5_line(precision, tmp_path):
    """configs[4] at a small size: a swap store under tmp, part of the groups
    swapped, the storage and host-link objects present."""
    j = run(["--config", "cfg5", "--precision", precision, "--params", "300000000",
             "--swap-gb", "1.3", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
             "--swap-dir", str(tmp_path)])
    assert j["value"] > 0 and j["config"]["swapped_groups"] >= 1
    assert j["storage"]["bytes_per_step"] > 0 and 0 < j["storage"]["frac"] < 5
    assert j["storage"]["bytes_per_swapped_param"] == (24 if precision == "mixed" else 8)

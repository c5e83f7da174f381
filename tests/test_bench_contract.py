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


def test_reference_arm_line_pure_bf16():
    """The reference arm in the pure-bf16 mode times the reference's own
    fused_overflow_check + adam_step_bf16 (oracle/_ref)."""
    j = run(["--impl", "reference", "--precision", "pure_bf16", "--steps", "1", "--warmup", "1",
             "--cpu-sample", "1000000"])
    assert REQUIRED <= set(j) and j["value"] > 0
    assert j["config"]["workload"].endswith("-pure-bf16")
    assert "adam_step_bf16" in j["cpu_baseline"]["sample"]


def run_plain(args, env=None, timeout=600):
    """bench.py WITHOUT a launcher (the driver's `python bench.py --gpus N`)."""
    e = dict(os.environ, **(env or {}))
    e.pop("WORLD_SIZE", None)
    return subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, env=e,
                          capture_output=True, text=True, timeout=timeout)


def test_gpus_flag_launches_ranks_itself():
    """`python bench.py --gpus 2` with no torchrun re-executes itself under
    torch.distributed.run with two ranks; rank 0 alone prints, n_gpus: 2."""
    p = run_plain(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1",
                   "--cpu-sample", "1000000"])
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["impl"] == "reference"


def test_gpus_beyond_visible_devices_fails_loudly():
    import torch

    want = torch.cuda.device_count() + 2  # >= 2: the launcher path
    p = run_plain(["--gpus", str(want), "--steps", "1", "--warmup", "1"])
    assert p.returncode != 0
    assert "CUDA device" in p.stderr and not [ln for ln in p.stdout.splitlines()
                                               if ln.startswith("{")]


def test_world_size_mismatch_fails_loudly():
    e = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=300)
    assert p.returncode != 0 and "WORLD_SIZE" in p.stderr


@pytest.mark.gpu
def test_gpus_flag_two_ranks_on_one_gpu_without_torchrun():
    p = run_plain(["--gpus", "2", "--params", "100000000", "--steps", "3", "--warmup", "3",
                   "--e2e-steps", "0"], env={"MA_BENCH_BACKEND": "gloo", "MA_BENCH_DEVICE": "0"})
    assert p.returncode == 0, p.stderr[-3000:]
    j = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][0])
    assert j["n_gpus"] == 2 and j["value"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("nproc,precision", [(1, "mixed"), (2, "mixed"), (2, "pure_bf16")])
def test_cfg3_injection_line(nproc, precision):
    """configs[2]: the seeded inf/NaN plan over nproc ranks; bench.py itself
    asserts every rank's decisions and scales against the committed plan (the
    decisions depend only on the gradients, so the pure-bf16 mode — K3 on bf16
    weights — must meet the same plan)."""
    env = {"MA_BENCH_BACKEND": "gloo", "MA_BENCH_DEVICE": "0"} if nproc > 1 else None
    j = run(["--config", "cfg3", "--params", "100000000", "--steps", "12", "--warmup", "3",
             "--no-cpu-baseline", "--precision", precision], nproc=nproc, env=env)
    c = j["cfg3_check"]
    assert c["decisions_match"] and c["scales_match"] and c["steps_checked"] == 15
    assert 0 < c["skipped"] < 15 and j["n_gpus"] == nproc


@pytest.mark.gpu
def test_cfg3_p2p_exchange_inside_a_graph_two_ranks():
    """The fused K1 flag exchange keeps its epoch on the device, so the
    captured step replays correctly: two ranks (one GPU), the injection plan,
    decisions and scales checked against the committed plan by bench.py."""
    j = run(["--config", "cfg3", "--flag-exchange", "p2p", "--graph", "--params", "50000000",
             "--steps", "10", "--warmup", "3", "--no-cpu-baseline"], nproc=2,
            env={"MA_BENCH_BACKEND": "gloo", "MA_BENCH_DEVICE": "0"})
    assert j["config"]["graph"] is True and "peer memory" in j["config"]["flag_exchange"]
    assert j["cfg3_check"]["decisions_match"] and j["cfg3_check"]["steps_checked"] == 23


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["cfg1", "cfg3"])
def test_graph_replay_line(cfg):
    j = run(["--config", cfg, "--graph", "--params", "67108864", "--steps", "8", "--warmup", "3",
             "--no-cpu-baseline", "--e2e-steps", "0"])
    assert j["config"]["graph"] is True and j["value"] > 0
    assert j["roofline"]["k2_ms"] > 0
    if cfg == "cfg3":
        assert j["cfg3_check"]["steps_checked"] == 3 + 8 + 8  # + the eager K1/K2 calibration


@pytest.mark.gpu
def test_our_arm_line_n1():
    j = run(["--params", "200000000", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
             "--cpu-sample", "1000000"])
    assert REQUIRED <= set(j) and {"roofline", "cpu_baseline", "clocks", "gpu_launches"} <= set(j)
    r = j["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.2 and r["unit"] == "GB/s"
    assert j["e2e"]["h2d_bytes_per_step"] == 2 * 200000000 and j["gpu_launches"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("graph", [False, True])
def test_our_arm_line_pure_bf16(graph):
    j = run(["--precision", "pure_bf16", "--params", "200000000", "--steps", "3", "--warmup",
             "3", "--e2e-steps", "1", "--cpu-sample", "1000000"] + (["--graph"] if graph else []))
    assert REQUIRED <= set(j) and {"roofline", "cpu_baseline", "gpu_launches"} <= set(j)
    r = j["roofline"]
    assert r["bytes_per_param"] == 14 and "k3_v2" in r["kernel"] and 0 < r["frac"] < 1.2
    assert j["config"]["state"].startswith("bf16 weights/m/v in HBM")
    assert "adam_step_bf16" in j["cpu_baseline"]["sample"]


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
             "--e2e-steps", "1", "--swap-dir", str(tmp_path)])
    assert j["roofline"]["bound"] == "swap-device" and j["roofline"]["frac"] > 0
    assert j["e2e"]["value"] > 0 and j["e2e"]["d2h_bytes_per_step"] > 0
    assert j["value"] > 0 and j["config"]["swapped_groups"] >= 1
    assert j["storage"]["bytes_per_step"] > 0 and 0 < j["storage"]["frac"] < 5
    assert j["storage"]["bytes_per_swapped_param"] == (24 if precision == "mixed" else 8)


@pytest.mark.gpu
def test_cfg4_line_pool_roofline_e2e():
    """configs[3] at a small size: p/m/v in the drop-in memascend::Pool
    (registered, adaptive), the host-link roofline and the e2e object."""
    j = run(["--config", "cfg4", "--params", "250000000", "--slot-params", "16777216",
             "--steps", "3", "--warmup", "3", "--e2e-steps", "1"])
    r = j["roofline"]
    assert r["bound"] == "host-link" and 0 < r["frac"] < 1.3 and r["bytes_per_param"] == 24
    assert "memascend::Pool" in j["config"]["state_pool"]
    assert j["pinned_host_bytes"]["pool_payload"] == 12 * 250000000
    assert j["e2e"]["h2d_bytes_per_step"] == 14 * 250000000 and j["e2e"]["value"] > 0


@pytest.mark.gpu
def test_library_nccl_agreement_world1():
    """The N>1 guard of bench.py's NCCL exchange (every rank must resolve
    libnccl before any enters the communicator's collective creation), run
    on a world-1 NCCL process group."""
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import bench
    import paper_2505_23254_b200 as mab

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port()}", world_size=1, rank=0,
                            device_id=torch.device("cuda", 0))
    try:
        assert bench.Exchange._library_nccl_everywhere(mab) is True
        x = bench.Exchange("nccl", 1, 0)
        assert x.describe() == "none (1 rank)" and x.fallback is None
        x.close()
    finally:
        dist.destroy_process_group()

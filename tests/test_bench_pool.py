"""bench-pool (the reference CLI's pool report, memascend_cli.cpp:186-268;
SURVEY §8(f) row 4): tools/bench_pool.cpp built against the reference's own
Pool/model library and against ours prints identical host rows — capacity,
backing, live replay of the trainer's prefetch/hold pattern (peak live,
fragmentation, checkouts) or the analytic prediction above the backing
budget.  Host-only, runs on CPU (the device rows need a GPU)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


def report(which, *args):
    exe = os.path.join(REF, f"bench_pool_{which}")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/bench_pool_* not built (needs /root/reference at build time)")
    p = subprocess.run([exe, *args], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    return json.loads(p.stdout)


@pytest.mark.parametrize("model,inflight,budget", [("toy-dense", "1", "8"), ("toy-dense", "2", "8"),
                                                   ("toy-dense", "4", "8"),
                                                   ("qwen2.5-7b", "2", "3"),
                                                   ("llama3.1-8b", "3", "0.5")])
def test_bench_pool_host_rows_match_reference(model, inflight, budget):
    ref = report("ref", model, inflight, budget)
    ours = report("ours", model, inflight, budget)
    host = [r for r in ours["rows"] if r["tier"] == "host"]
    assert host == ref["rows"] and ours["model"] == ref["model"]
    modes = {r["mode"]: r for r in host}
    assert modes["adaptive"]["capacity_bytes"] <= modes["monolithic"]["capacity_bytes"]

"""Drop-in proof: the reference's OWN test suites for the hot path
(proj/tests/test_overflow.cpp, test_optimizer.cpp, test_pinned.cpp, test_pool.cpp,
test_model.cpp), compiled
unmodified against our headers (include/memascend/*.hpp) and linked against
our library (libmemascend.so -> libmemascend_b200.so).  Built by
`make -C oracle dropin` in the build container (needs /root/reference); the
binary travels to the GPU box."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_tests")


def run():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_tests not built (needs /root/reference at build time)")
    p = subprocess.run([BIN], capture_output=True, text=True, cwd="/tmp", timeout=600)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", p.stdout)
    assert m, p.stdout + p.stderr
    return int(m.group(1)), int(m.group(2)), int(m.group(3)), p


def test_dropin_without_gpu_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present: see test_dropin_reference_suites_gpu")
    total, passed, failed, p = run()
    assert total == 44
    # pure host logic (capacity rules, scaler, conversions, ...) passes; every
    # failure is the loud no-device error, never a silent CPU result
    errs = [ln for ln in p.stderr.splitlines() if "threw:" in ln]
    assert failed == len(errs) and failed > 0
    assert all("no CPU fallback" in ln for ln in errs), errs


@pytest.mark.gpu
def test_dropin_reference_suites_gpu():
    total, passed, failed, p = run()
    assert (total, failed) == (44, 0), p.stdout + p.stderr


SIM = os.path.join(ROOT, "oracle", "_ref", "dropin_simulator")


@pytest.mark.gpu
def test_reference_simulator_on_b200_hot_path():
    """The reference's unmodified offloaded trainer (simulator.cpp +
    direct_io.cpp) linked to our hot path, run by its own test_simulator.cpp:
    digests bitwise equal to its in-memory reference trainer, fault skip,
    I/O accounting, pool fragmentation (13 cases)."""
    if not os.path.exists(SIM):
        pytest.skip("oracle/_ref/dropin_simulator not built")
    p = subprocess.run([SIM], capture_output=True, text=True, cwd="/tmp", timeout=900)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", p.stdout)
    assert m and (int(m.group(1)), int(m.group(3))) == (13, 0), p.stdout + p.stderr

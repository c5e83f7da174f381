"""Launch options of the step chain, each through the
stepper suites in a subprocess (the variables are latched at the library's
first launch): the L2-tail option of K1 (MA_K1_KEEP_MB, off by default —
a stepper check loads the gradients' last MiB under an L2 evict_last policy
and the next update demotes those lines) and plain instead of programmatic
launches (MA_PDL=0).  None may change a bit."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("ldk", ["1", "2"])
def test_stepper_suites_with_the_l2_tail_on(ldk):
    env = dict(os.environ, MA_K1_KEEP_MB="1", MA_K1_LDK=ldk)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        "tests/test_gpu_stepper_runtime.py", "tests/test_gpu_stepper_fuzz.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def test_stepper_suites_with_plain_launches():
    """MA_PDL=0: K2 / K3 / the scaler launched plainly instead of as
    programmatic dependents — the same bits."""
    env = dict(os.environ, MA_PDL="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        "tests/test_gpu_stepper_runtime.py", "tests/test_gpu_stepper_fuzz.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout

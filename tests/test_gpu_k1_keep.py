"""The L2-tail option of K1 (MA_K1_KEEP_MB, off by default):
with it on, a stepper check loads the gradients' last MiB under an L2
evict_last policy and the next update demotes those lines.  Neither may
change a bit.  The variables are latched at the library's first launch, so
the stepper suites run in a subprocess with the option on."""
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

"""Input draws of the reference known-answer tests, on the restated std::mt19937_64."""
import numpy as np

from oracle import oracle as ora

f32 = np.float32


def kat_random100_inputs(r):
    """test_optimizer.cpp:61-98 input draws on the restated engine."""
    rng = ora.MT19937_64(r["seed"])
    n = r["n"]
    p0 = np.array([rng() % 2048 for _ in range(n)], np.uint64).astype(f32) / f32(256.0) - f32(4.0)
    grads = []
    for _ in range(r["steps"]):
        u = np.array([rng() % 65536 for _ in range(n)], np.uint64).astype(f32)
        grads.append((u / f32(32768.0) - f32(1.0)) * f32(r["scale"]))
    return p0, grads

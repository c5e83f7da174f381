import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, torch
import paper_2505_23254_b200 as mab
n = 100_000_000
arrs = {}
for k in ("p", "m", "v"):
    b = mab.aligned_host_buffer(n * 4, register=True).view(np.float32); b[:] = 0.01; arrs[k] = b
g = mab.aligned_host_buffer(n * 4, register=True).view(np.float32); g[:] = 1.0
h = mab.AdamHyper(weight_decay=0.01)
for it in range(3):
    t0 = time.perf_counter()
    mab.adam_step_fp32(arrs["p"], arrs["m"], arrs["v"], g, it + 1, h, 1.0)
    dt = time.perf_counter() - t0
    print(f"registered zero-copy: {n/dt/1e9:.2f} G params/s ({dt*1e3:.1f} ms), PCIe bytes/param 28 -> {28*n/dt/1e9:.1f} GB/s")
# pageable
pp = {k: np.full(n, 0.01, np.float32) for k in "pmv"}
gg = np.ones(n, np.float32)
for it in range(2):
    t0 = time.perf_counter()
    mab.adam_step_fp32(pp["p"], pp["m"], pp["v"], gg, it + 1, h, 1.0)
    dt = time.perf_counter() - t0
    print(f"pageable staged: {n/dt/1e9:.2f} G params/s ({dt*1e3:.1f} ms)")

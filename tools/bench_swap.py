#!/usr/bin/env python
"""Swap-store backend comparison: O_DIRECT write and
read throughput of the DirectIoEngine drop-in per backend (pread/pwrite,
POSIX AIO = the reference's lio_listio path, io_uring), worker count and
queue depth, on file-backed devices under --dir.  Each point writes --keys
tensors of --mib MiB concurrently (async ops), then reads them back and
checks them.  One JSON line per point, then a summary line.

    python tools/bench_swap.py --dir /tmp/ma_swapbench [--mib 1024 --keys 4]
"""
import argparse
import json
import os
import shutil
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_23254_b200 as mab  # noqa: E402


def point(d, backend, workers, depth, keys, nbytes, bufs):
    devs = mab.DirectIoEngine.create_virtual_devices(d, 2, keys * nbytes // 2 + (16 << 20))
    try:
        with mab.DirectIoEngine(devs, workers=workers, queue_depth=depth, backend=backend) as e:
            t0 = time.perf_counter()
            ops = [e.write_tensor_async(f"k{i}", bufs[i], nbytes) for i in range(keys)]
            for op in ops:
                op.wait()
            t1 = time.perf_counter()
            outs = [mab.aligned_host_buffer(nbytes) for _ in range(keys)]
            t2 = time.perf_counter()
            ops = [e.read_tensor_async(f"k{i}", outs[i]) for i in range(keys)]
            for op in ops:
                op.wait()
            t3 = time.perf_counter()
            ok = all((outs[i][::4096] == bufs[i][::4096]).all() for i in range(keys))
    finally:
        shutil.rmtree(d, ignore_errors=True)
    total = keys * nbytes
    return {"backend": backend, "workers": workers, "queue_depth": depth,
            "write_gbs": total / (t1 - t0) / 1e9, "read_gbs": total / (t3 - t2) / 1e9,
            "bytes": total, "verified": bool(ok)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", default="/tmp/ma_swapbench")
    ap.add_argument("--mib", type=int, default=1024)
    ap.add_argument("--keys", type=int, default=4)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    nbytes = a.mib << 20
    bufs = []
    for i in range(a.keys):
        b = mab.aligned_host_buffer(nbytes)
        b[:] = np.random.default_rng(i).integers(0, 256, nbytes, dtype=np.uint8)
        bufs.append(b)
    backends = ["sync", "aio"] + (["uring"] if mab.uring_available() else [])
    rows = []
    for backend in backends:
        for workers in (1, 2, 4, 8):
            for depth in (1, 8, 32):
                if backend == "sync" and depth > 1:
                    continue  # depth does not apply to positional I/O
                r = point(os.path.join(a.dir, "p"), backend, workers, depth, a.keys, nbytes, bufs)
                rows.append(r)
                print(json.dumps(r), flush=True)
    best = {b: max((r for r in rows if r["backend"] == b),
                   key=lambda r: 2 / (1 / r["read_gbs"] + 1 / r["write_gbs"])) for b in backends}
    ref_default = next(r for r in rows if r["backend"] == "aio" and r["workers"] == 2
                       and r["queue_depth"] == 8)
    summary = {"summary": True, "best": best, "reference_default_aio_w2_qd8": ref_default}
    print(json.dumps(summary), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"points": rows, **summary}, f, indent=1)


if __name__ == "__main__":
    main()

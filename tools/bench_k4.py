"""K4 (reduce-scatter epilogue check) and K3 (bf16-state Adam) kernel
measurements on one B200 (run on the GPU box).  Writes
profiles/<tag>_k4_k3_bench.json.

K4 with `nsrc` HBM-resident sources stands in for the reduction half of the
reduce-scatter (on a multi-GPU node the nsrc-1 remote sources arrive over
NVLink instead); algorithmic bytes per element = nsrc * 2 (bf16 in) + 2
(bf16 out).  The unfused alternative (sum, then K1 over the result) moves
2 more bytes per element.  K3: 2 (bf16 g) + 6 read + 6 write = 14 B/param.

    python tools/bench_k4.py [--tag r1] [--n 268435456]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps, warm=3):
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch

    import paper_2505_23254_b200 as mab

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    peak = float(peaks.get("hbm_gbs", 6550.4))
    n = args.n
    out = {"n": n, "peak_gbs": peak, "k4": [], "k3": None}
    st = mab.Stepper(mab.AdamHyper(weight_decay=0.01), 65536.0, 2000, "bf16", "bf16")
    srcs = [torch.randn(n, device="cuda").to(torch.bfloat16) for _ in range(8)]
    dst = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    # one source measured first and again last: its first figure carries
    # whatever state the allocations above left (clocks, dirty L2 lines)
    for k in (1, 2, 4, 8, 1):
        ms = timed(lambda: st.reduce_check(srcs[:k], dst, post_scale=1.0 / k), args.reps)
        byts = (2 * k + 2) * n
        out["k4"].append({"nsrc": k, "ms": ms, "gbs": byts / ms / 1e6,
                          "frac": byts / ms / 1e6 / peak, "bytes_per_elem": 2 * k + 2})
        print(out["k4"][-1], flush=True)
    # producer-side check (k_ingest): dst = cast(src * scale) + the check
    out["ingest"] = []
    for skind, sdt in (("f32", torch.float32), ("bf16", torch.bfloat16)):
        src = srcs[0].to(sdt)
        ms = timed(lambda: st.ingest(src, dst), args.reps)
        byts = (src.element_size() + 2) * n
        out["ingest"].append({"src": skind, "ms": ms, "gbs": byts / ms / 1e6,
                              "frac": byts / ms / 1e6 / peak,
                              "bytes_per_elem": src.element_size() + 2})
        print(out["ingest"][-1], flush=True)
        del src
    del srcs, dst
    torch.cuda.empty_cache()

    # K3: pure-bf16 state over n params (bf16 g), 100M sub-groups
    p = torch.randn(n, device="cuda").to(torch.bfloat16)
    m = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    v = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    g = (torch.randn(n, device="cuda") * 1024).to(torch.bfloat16)
    sub = 100_000_000
    groups = [(p[o:o + sub], m[o:o + sub], v[o:o + sub], g[o:o + sub])
              for o in range(0, n, sub)]
    st3 = mab.Stepper(mab.AdamHyper(weight_decay=0.01), 65536.0, 2000, "bf16", "bf16")

    def k3():
        st3.apply_bf16(groups)

    ms = timed(k3, args.reps)
    out["k3"] = {"ms": ms, "gbs": 14 * n / ms / 1e6, "frac": 14 * n / ms / 1e6 / peak,
                 "bytes_per_param": 14}
    print(out["k3"], flush=True)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", f"{args.tag}_k4_k3_bench.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

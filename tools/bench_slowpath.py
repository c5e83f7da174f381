"""How much the exact (out-of-line) path costs when a workload sends slots to
it: K2 and K3 over 268 M params where a fraction of the 4- / 8-element slots
hold parameters that never received a gradient (m = v = g = 0, e.g.
embedding rows a batch does not touch) — such elements fail the fast-path
guard (|m| >= 2^-50) and are recomputed exactly.  CUDA events, warm, median.

    python tools/bench_slowpath.py [--n 268435456] [--fracs 0,0.01,0.05,0.2,1]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=10, warm=3):
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
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--fracs", default="0,0.01,0.05,0.2,1")
    ap.add_argument("--tag", default="r2")
    ap.add_argument("--layout", choices=["blocks", "rows"], default="blocks",
                    help="cold 8-element blocks scattered at random, or cold rows of 4096 "
                         "contiguous params (an embedding table's untouched rows)")
    ap.add_argument("--decayed", action="store_true",
                    help="cold elements keep tiny decayed moments (|m| ~ 2^-70) instead of 0")
    args = ap.parse_args()
    import torch

    import paper_2505_23254_b200 as mab

    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.4))
    n, sub = args.n, 100_000_000
    out = {"n": n, "peak_gbs": peak, "k2": [], "k3": []}
    gen = torch.Generator(device="cuda").manual_seed(1)
    for frac in (float(x) for x in args.fracs.split(",")):
        # K2: fp32 state, bf16 grads / working weights
        p = torch.randn(n, device="cuda") * 0.1
        m = torch.randn(n, device="cuda") * 1e-3
        v = torch.rand(n, device="cuda") * 1e-6
        g = (torch.randn(n, device="cuda") * 1024).to(torch.bfloat16)
        w = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        blk = 8 if args.layout == "blocks" else 4096
        cold = torch.rand((n + blk - 1) // blk, device="cuda", generator=gen) < frac
        cold = cold.repeat_interleave(blk)[:n]
        m[cold] = 2.0 ** -70 if args.decayed else 0.0
        if not args.decayed:
            v[cold] = 0
        g[cold] = 0
        st = mab.Stepper(mab.AdamHyper(weight_decay=0.01), 65536.0, 2000, "bf16", "bf16")
        groups = mab.Stepper.subgroups([(p[o:o + sub], m[o:o + sub], v[o:o + sub], g[o:o + sub],
                                         w[o:o + sub]) for o in range(0, n, sub)], "bf16", "bf16")
        # m / v stay zero on the cold elements from step to step (g = 0)
        ms = timed(lambda: st.apply(groups))
        out["k2"].append({"cold_frac": frac, "ms": ms, "frac": 28 * n / ms / 1e6 / peak})
        del p, m, v, w, groups
        st.close()
        # K3: bf16 state
        p16 = (torch.randn(n, device="cuda") * 0.1).to(torch.bfloat16)
        m16 = (torch.randn(n, device="cuda") * 1e-3).to(torch.bfloat16)
        v16 = (torch.rand(n, device="cuda") * 1e-6).to(torch.bfloat16)
        m16[cold] = 2.0 ** -70 if args.decayed else 0.0
        if not args.decayed:
            v16[cold] = 0
        st3 = mab.Stepper(mab.AdamHyper(weight_decay=0.01), 65536.0, 2000, "bf16", "bf16")
        g3 = [(p16[o:o + sub], m16[o:o + sub], v16[o:o + sub], g[o:o + sub])
              for o in range(0, n, sub)]
        ms = timed(lambda: st3.apply_bf16(g3))
        out["k3"].append({"cold_frac": frac, "ms": ms, "frac": 14 * n / ms / 1e6 / peak})
        print(frac, out["k2"][-1], out["k3"][-1], flush=True)
        del p16, m16, v16, g, g3, cold
        st3.close()
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    out.update(layout=args.layout, decayed=args.decayed)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out",
                                     f"{args.tag}_slowpath_{args.layout}{'_decayed' if args.decayed else ''}.json"), "w"),
              indent=1)


if __name__ == "__main__":
    main()

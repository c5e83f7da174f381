"""Does K1's evict_last gradient tail linger in L2 and slow
down the kernels that run after the optimizer step?

One process per setting (the K1 policy is latched at first launch): a
stepper step over `--n` params (check -> apply -> finish), then a "victim"
that re-reads an L2-sized buffer (`--victim-mb`) `--reps` times with
default caching (torch.sum), timed with CUDA events; repeated `--trials`
times.  Compared: MA_K1_KEEP_MB=0 (no evict_last lines) vs the default.

    python tools/l2_pollution_probe.py [--victim-mb 96] [--out gpurun_out/l2_pollution.json]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(n, victim_mb, reps, trials):
    import numpy as np
    import torch

    import paper_2505_23254_b200 as mab

    dev = torch.device("cuda", 0)
    p = torch.empty(n, dtype=torch.float32, device=dev)
    m = torch.zeros(n, dtype=torch.float32, device=dev)
    v = torch.zeros(n, dtype=torch.float32, device=dev)
    g = torch.empty(n, dtype=torch.bfloat16, device=dev)
    w = torch.empty(n, dtype=torch.bfloat16, device=dev)
    mab.gen_seeded_weights(p, w, seed=1)
    mab.gen_pseudo_grads(g, w, step=0, seed=1, scale=65536.0)
    st = mab.Stepper(mab.AdamHyper(weight_decay=0.01), 65536.0, 2000, "bf16", "bf16")
    groups = mab.Stepper.subgroups([(p, m, v, g, w)], "bf16", "bf16")
    victim = torch.ones(victim_mb << 18, dtype=torch.float32, device=dev)  # MiB / 4 B
    out = torch.empty((), dtype=torch.float32, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    times = []
    for t in range(trials + 2):
        flush.zero_()                       # L2 starts from the same state
        torch.sum(victim, dim=0, out=out)          # victim lines resident (normal priority)
        st.check(g)
        st.apply(groups)
        st.finish()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            torch.sum(victim, dim=0, out=out)
        b.record()
        torch.cuda.synchronize()
        if t >= 2:
            times.append(a.elapsed_time(b) / reps * 1e3)
    st.close()
    return {"victim_us": float(np.median(times)), "victim_us_all": times,
            "victim_gbs": (victim_mb << 20) / (np.median(times) * 1e-6) / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64 << 20)
    ap.add_argument("--victim-mb", type=int, default=96)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--trials", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "l2_pollution.json"))
    ap.add_argument("--child", action="store_true")
    args = ap.parse_args()
    if args.child:
        print(json.dumps(child(args.n, args.victim_mb, args.reps, args.trials)), flush=True)
        return
    rows = []
    for keep in ("0", "32", "0", "32"):
        env = dict(os.environ, MA_K1_KEEP_MB=keep)
        r = subprocess.run([sys.executable, __file__, "--child", "--n", str(args.n),
                            "--victim-mb", str(args.victim_mb), "--reps", str(args.reps),
                            "--trials", str(args.trials)], env=env, capture_output=True,
                           text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("{")]
        row = json.loads(line[-1]) if line else {"error": r.stderr[-800:]}
        row["keep_mb"] = int(keep)
        rows.append(row)
        print({k: row.get(k) for k in ("keep_mb", "victim_us", "victim_gbs", "error")}, flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

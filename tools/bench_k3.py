"""K3 (pure-bf16 Adam) A/B over MA_K3_VARIANT on one B200: each variant in
its own process (the variant is latched at first launch), bit-exact check
against the oracle on 1 M params (adversarial state included), then CUDA-
event timing over --n params (bf16 g, 100 M sub-groups, 14 B/param).

    python tools/bench_k3.py [--variants 0,9,10] [--n 268435456] [--tag r2]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def one(n, reps):
    import numpy as np
    import torch

    import nan_inputs as ni
    import paper_2505_23254_b200 as mab
    from oracle import oracle as ora

    # parity: 1 M params, a tenth of them adversarial, t = 3
    k = 1 << 20
    p, m, v, g = ni.state(5, k, p_special=0.1)
    p16, m16, v16 = (ni.bf16_bits(x) for x in (p, m, v))
    g16 = ni.bf16_bits(g)
    h = ora.hyper(lr=1e-3, weight_decay=0.01)
    want = [x.copy() for x in (p16, m16, v16)]
    ora.adam_step_bf16(*want, ora.widen(g16, "bf16"), 3, h, 65536.0)
    st = mab.Stepper(mab.AdamHyper(lr=1e-3, weight_decay=0.01), 65536.0, 2000, "bf16", "bf16")
    for _ in range(2):  # t = 3 at the third apply
        st.finish()
    d = [torch.from_numpy(x.view(np.int16).copy()).cuda() for x in (p16, m16, v16, g16)]
    st.apply_bf16([(d[0], d[1], d[2], d[3].view(torch.bfloat16))])
    torch.cuda.synchronize()
    exact = all(np.array_equal(a.cpu().numpy().view(np.uint16), b) for a, b in zip(d, want))
    st.close()

    pp = torch.randn(n, device="cuda").to(torch.bfloat16)
    mm = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    vv = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    gg = (torch.randn(n, device="cuda") * 1024).to(torch.bfloat16)
    sub = 100_000_000
    groups = [(pp[o:o + sub], mm[o:o + sub], vv[o:o + sub], gg[o:o + sub])
              for o in range(0, n, sub)]
    st3 = mab.Stepper(mab.AdamHyper(weight_decay=0.01), 65536.0, 2000, "bf16", "bf16")
    for _ in range(3):
        st3.apply_bf16(groups)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st3.apply_bf16(groups)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    ms = ts[len(ts) // 2]
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.4))
    return {"variant": int(os.environ.get("MA_K3_VARIANT", "0")), "ms": ms,
            "gbs": 14 * n / ms / 1e6, "frac": 14 * n / ms / 1e6 / peak, "exact": exact}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="0,9,10,11,12,13,14")
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tag", default="r2")
    ap.add_argument("--child", action="store_true")
    args = ap.parse_args()
    if args.child:
        print(json.dumps(one(args.n, args.reps)), flush=True)
        return
    rows = []
    for var in args.variants.split(","):
        env = dict(os.environ, MA_K3_VARIANT=var)
        r = subprocess.run([sys.executable, __file__, "--child", "--n", str(args.n), "--reps",
                            str(args.reps)], env=env, capture_output=True, text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("{")]
        rows.append(json.loads(line[-1]) if line else {"variant": int(var), "error": r.stderr[-800:]})
        print(rows[-1], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(rows, open(os.path.join(ROOT, "gpurun_out", f"{args.tag}_k3_ab.json"), "w"), indent=1)


if __name__ == "__main__":
    main()

# Final bench lines of the production code (GPU box): default (configs[1]),
# configs[0] and 8 Mi eager/graph, the pure-bf16 step, the reference arm.
set -u
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/final_cfg2.log 2>&1; tail -1 gpurun_out/final_cfg2.log > gpurun_out/final_cfg2.json
: > gpurun_out/final_cfg1.jsonl; : > gpurun_out/final_8mi.jsonl
for g in "" "--graph"; do
  timeout 120 python bench.py --config cfg1 --steps 50 --warmup 5 $g --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 >> gpurun_out/final_cfg1.jsonl
  timeout 120 python bench.py --params 8388608 --steps 50 --warmup 5 $g --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 >> gpurun_out/final_8mi.jsonl
done
timeout 400 python bench.py --precision pure_bf16 > gpurun_out/final_cfg2_bf16.log 2>&1; tail -1 gpurun_out/final_cfg2_bf16.log > gpurun_out/final_cfg2_bf16.json
timeout 300 python bench.py --impl reference > gpurun_out/final_ref.log 2>&1; tail -1 gpurun_out/final_ref.log > gpurun_out/final_ref.json
python - <<'PY'
import json
for f in ("final_cfg2.json", "final_cfg1.jsonl", "final_8mi.jsonl", "final_cfg2_bf16.json"):
    for line in open("gpurun_out/" + f):
        d = json.loads(line)
        print(f, d["config"]["workload"], "graph" if d["config"].get("graph") else "eager",
              round(d["ms_per_step"] * 1000, 2), "us", round(d["value"] / 1e9, 2), "G/s frac",
              round(d["roofline"]["frac"], 4), "step", round(d["roofline"]["step_frac"], 4),
              "e2e", (d.get("e2e") or {}).get("value"), "cpu", (d.get("cpu_baseline") or {}).get("value"))
d = json.load(open("gpurun_out/final_ref.json")); print("reference", d["value"])
PY

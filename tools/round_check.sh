# Full GPU check of HEAD (run on the GPU box from the repo root): the GPU
# test suite, smoke, the default bench line and the configs[0] lines.
set -u
mkdir -p gpurun_out
timeout 1100 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 400 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_cfg2.log > gpurun_out/bench_cfg2.json
for g in "" "--graph"; do
  timeout 120 python bench.py --config cfg1 --steps 50 --warmup 5 $g --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 >> gpurun_out/bench_cfg1.jsonl
  timeout 120 python bench.py --params 8388608 --steps 50 --warmup 5 $g --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 >> gpurun_out/bench_8mi.jsonl
done
python - <<'PY'
import json
for f in ("gpurun_out/bench_cfg2.json", "gpurun_out/bench_cfg1.jsonl", "gpurun_out/bench_8mi.jsonl"):
    for line in open(f):
        try:
            d = json.loads(line)
            print(f, d["config"]["workload"], "graph" if d["config"].get("graph") else "eager",
                  round(d["ms_per_step"] * 1000, 2), "us", round(d["value"] / 1e9, 2), "G/s",
                  "frac", round(d["roofline"]["frac"], 4), "step", round(d["roofline"]["step_frac"], 4),
                  "e2e", (d.get("e2e") or {}).get("value"))
        except Exception as e:
            print(f, "unparsed", line[:200])
PY

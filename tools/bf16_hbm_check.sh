# The pure-bf16 step in HBM (bench.py --precision pure_bf16 on configs[1] /
# configs[0]) with and without the programmatic K3 launch, plus the GPU
# tests that exercise K1/K2/K3 and the stepper runtime.  GPU box.
set -u
mkdir -p gpurun_out
out=gpurun_out/bf16_hbm.txt
: > $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stepper_runtime.py tests/test_gpu_stepper_fuzz.py tests/test_gpu_cold.py tests/test_gpu_nan.py -x -q > gpurun_out/bf16_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/bf16_tests.log)" >> $out
summ() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], "graph" if d["config"].get("graph") else "eager", round(d["ms_per_step"]*1000,2),"us", round(d["value"]/1e9,2), "G/s frac", round(d["roofline"]["frac"],4), "step", round(d["roofline"]["step_frac"],4), "k2_us", round(d["roofline"]["k2_ms"]*1000,1), "k1_us", round(d["roofline"]["k1_ms"]*1000,1), "e2e", (d.get("e2e") or {}).get("value"), "cpu", (d.get("cpu_baseline") or {}).get("value"))' 2>&1 | tail -1; }
for rep in 1 2; do
for k3 in 0 1; do
  for g in "" "--graph"; do
    echo "pdl_k3=$k3 $(MA_PDL_K3=$k3 timeout 120 python bench.py --precision pure_bf16 --config cfg1 --steps 50 --warmup 5 $g --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | summ)" >> $out
  done
  echo "pdl_k3=$k3 $(MA_PDL_K3=$k3 timeout 300 python bench.py --precision pure_bf16 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | summ)" >> $out
done
done
timeout 400 python bench.py --precision pure_bf16 > gpurun_out/bench_cfg2_bf16.log 2>&1
tail -1 gpurun_out/bench_cfg2_bf16.log > gpurun_out/bench_cfg2_bf16.json
echo "full: $(summ < gpurun_out/bench_cfg2_bf16.json)" >> $out
timeout 400 python bench.py > gpurun_out/bench_cfg2.log 2>&1
tail -1 gpurun_out/bench_cfg2.log > gpurun_out/bench_cfg2.json
echo "full mixed: $(summ < gpurun_out/bench_cfg2.json)" >> $out
timeout 200 python bench.py --impl reference --precision pure_bf16 > gpurun_out/bench_ref_bf16.log 2>&1
tail -1 gpurun_out/bench_ref_bf16.log > gpurun_out/bench_ref_bf16.json
echo "reference bf16: $(cut -c1-300 gpurun_out/bench_ref_bf16.json)" >> $out
cat $out

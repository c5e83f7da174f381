# K1's kept L2 tail demoted by the update: pollution probe
# (keep 0 vs 32 MiB), the seam A/B lines, the pure-bf16 step, GPU tests of
# the stepper paths.  GPU box.
set -u
mkdir -p gpurun_out
out=gpurun_out/demote_check.txt
: > $out
for mb in 96 48; do
  python tools/l2_pollution_probe.py --victim-mb $mb --out gpurun_out/l2_pollution_demoted_$mb.json >> $out 2>&1
done
summ() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], "graph" if d["config"].get("graph") else "eager", round(d["ms_per_step"]*1000,2),"us", round(d["value"]/1e9,2), "G/s frac", round(d["roofline"]["frac"],4), "step", round(d["roofline"]["step_frac"],4), "k2_us", round(d["roofline"]["k2_ms"]*1000,1), "k1_us", round(d["roofline"]["k1_ms"]*1000,1))' 2>&1 | tail -1; }
for rep in 1 2; do
  for g in "" "--graph"; do
    echo "$(timeout 120 python bench.py --config cfg1 --steps 50 --warmup 5 $g --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | summ)" >> $out
    echo "$(MA_K1_KEEP_MB=0 timeout 120 python bench.py --config cfg1 --steps 50 --warmup 5 $g --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | summ) [keep 0]" >> $out
  done
  echo "$(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | summ)" >> $out
  echo "$(timeout 300 python bench.py --precision pure_bf16 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | summ)" >> $out
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stepper_runtime.py tests/test_gpu_stepper_fuzz.py tests/test_gpu_swapped.py tests/test_zero_step.py tests/test_allgather.py -x -q > gpurun_out/demote_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/demote_tests.log)" >> $out
cat $out

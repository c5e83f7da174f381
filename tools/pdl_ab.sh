set -u
mkdir -p gpurun_out
out=gpurun_out/pdl_ab.txt
: > $out
for rep in 1 2; do
for cfg in "--config cfg1" "--params 8388608"; do
for g in "" "--graph"; do
for v in "14 0" "20 0" "20 1" "21 1"; do
  set -- $v
  line=$(MA_K1_LDK=0 MA_K2_VARIANT=$1 MA_PDL_FINISH=$2 timeout 120 python bench.py $cfg --steps 50 --warmup 5 $g --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1)
  echo "$rep|$cfg|$g|v=$1 fin=$2|$(echo "$line" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,2),"us", round(d["roofline"]["step_frac"],4), "k2_ms", round(d["roofline"]["k2_ms"]*1000,1), "k1", round(d["roofline"]["k1_ms"]*1000,1))' 2>&1 | tail -1)" >> $out
done; done; done; done
MA_K2_VARIANT=21 MA_PDL_FINISH=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stepper_runtime.py tests/test_gpu_stepper_fuzz.py -x -q > gpurun_out/pdl_tests.log 2>&1; echo "tests rc=$?" >> $out
tail -2 gpurun_out/pdl_tests.log >> $out
MA_K2_VARIANT=21 MA_PDL_FINISH=1 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 > gpurun_out/pdl_cfg2.json
cat $out

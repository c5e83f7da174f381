# K3 vector second chance (variant 25) vs production (21) on cold layouts +
# correctness under 25; cfg4 streamed line with K2 variant 14 vs 20 (PDL).
set -u
mkdir -p gpurun_out
out=gpurun_out/k3v25_cfg4_ab.txt
: > $out
python tools/bench_k3.py --variants 21,25,21,25 --tag k3v25 >> $out 2>&1
for var in 21 25; do
  for lay in "--layout blocks" "--layout rows" "--layout rows --decayed"; do
    MA_K3_VARIANT=$var timeout 600 python tools/bench_slowpath.py $lay --tag w$var > /dev/null 2>&1
    echo "v$var $lay: $(python -c "
import json,glob,os
fs=sorted(glob.glob('gpurun_out/w${var}_slowpath_*.json'),key=os.path.getmtime)
d=json.load(open(fs[-1])); print(fs[-1], [(r['cold_frac'], round(r['frac'],3)) for r in d['k3']])" 2>&1 | tail -1)" >> $out
  done
done
MA_K3_VARIANT=25 timeout 900 python -m pytest tests/test_gpu_cold.py tests/test_gpu_nan.py tests/test_gpu_parity.py tests/test_gpu_stepper_fuzz.py -x -q > gpurun_out/k3v25_tests.log 2>&1
echo "tests v25 rc=$? $(tail -1 gpurun_out/k3v25_tests.log)" >> $out
for rep in 1 2 3; do for v in 14 20; do
  echo "cfg4 v$v: $(MA_K2_VARIANT=$v timeout 900 python bench.py --config cfg4 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), round(d["roofline"]["frac"],4), d["roofline"].get("achieved"))')" >> $out
done; done
cat $out

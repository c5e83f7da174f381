# K3 split drain (variant 27: two threads per listed slot) vs production 21:
# live state (bench_k3, bit-exact check), cold layouts, tests under 27.
set -u
mkdir -p gpurun_out
out=gpurun_out/k3_split_ab.txt
: > $out
python tools/bench_k3.py --variants 21,27,21,27 --tag k3split >> $out 2>&1
for var in 21 27; do
  for lay in "--layout blocks" "--layout rows" "--layout rows --decayed"; do
    MA_K3_VARIANT=$var timeout 600 python tools/bench_slowpath.py $lay --tag s$var > /dev/null 2>&1
    echo "v$var $lay: $(python -c "
import json,glob,os
fs=sorted(glob.glob('gpurun_out/s${var}_slowpath_*.json'),key=os.path.getmtime)
d=json.load(open(fs[-1])); print(fs[-1], [(r['cold_frac'], round(r['frac'],3)) for r in d['k3']])" 2>&1 | tail -1)" >> $out
  done
done
MA_K3_VARIANT=27 timeout 900 python -m pytest tests/test_gpu_cold.py tests/test_gpu_nan.py tests/test_gpu_parity.py tests/test_gpu_stepper_fuzz.py tests/test_fuzz_hyper.py -x -q > gpurun_out/k3split_tests.log 2>&1
echo "tests v27 rc=$? $(tail -1 gpurun_out/k3split_tests.log)" >> $out
cat $out

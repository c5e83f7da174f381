# K3 cold-slot A/B (MA_K3_VARIANT 0 = production (when run: the deferred kernel without
# cold routes, now variant 24), 21 = early warp reject +
# vectorised cold route in the deferred phase, 22 = cold route only, 23 =
# early reject only): normal-case speed + bit-exactness (bench_k3.py), cold
# layouts (bench_slowpath.py), and the cold / NaN / parity tests per variant.
set -u
mkdir -p gpurun_out
out=gpurun_out/k3_cold_ab.txt
: > $out
python tools/bench_k3.py --variants 0,21,22,23,0,21 --tag k3cold >> $out 2>&1
for var in 0 21 22 23; do
  for lay in "--layout blocks" "--layout rows" "--layout rows --decayed"; do
    MA_K3_VARIANT=$var timeout 600 python tools/bench_slowpath.py $lay --tag v$var > gpurun_out/slow_v${var}.log 2>&1
    echo "v$var $lay: $(python -c "
import json,glob,os
fs=sorted(glob.glob('gpurun_out/v${var}_slowpath_*.json'),key=os.path.getmtime)
d=json.load(open(fs[-1])); print(fs[-1], [(r['cold_frac'], round(r['frac'],3)) for r in d['k3']])" 2>&1 | tail -1)" >> $out
  done
done
for var in 21; do
  MA_K3_VARIANT=$var timeout 900 python -m pytest tests/test_gpu_cold.py tests/test_gpu_nan.py tests/test_gpu_parity.py tests/test_gpu_stepper_fuzz.py -x -q > gpurun_out/k3v${var}_tests.log 2>&1
  echo "tests v$var rc=$? $(tail -1 gpurun_out/k3v${var}_tests.log)" >> $out
done
cat $out

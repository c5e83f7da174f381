# After a K3 production change: the GPU suite, the K3 ncu capture (merged
# into profiles/r2_ncu_summary.json on the box) and K3 live-state A/B.
set -u
mkdir -p gpurun_out
timeout 1100 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest.log
timeout 400 ncu --clock-control none --set full --import-source on -c 1 -k regex:k3_v2 --launch-skip 3 -o gpurun_out/r2_k3 \
    python tools/bench_k3.py --child --reps 2 > /dev/null 2>&1; echo "k3 ncu rc=$?"
python tools/ncu_summary.py r2k3 gpurun_out/r2_k3.ncu-rep:268435456:14 > /dev/null 2>&1; echo "summary rc=$?"
cp profiles/r2k3_ncu_summary.json gpurun_out/ 2>/dev/null
python tools/bench_k3.py --variants 0,24,0,24 --tag k3final 2>&1 | tail -4
timeout 400 python bench.py --precision pure_bf16 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 > gpurun_out/bench_cfg2_bf16_final.json
python -c "import json; d=json.load(open('gpurun_out/bench_cfg2_bf16_final.json')); print(d['value'], d['roofline']['frac'], d['roofline']['step_frac'])"

# Final bench lines of configs[2..4] on the production code (GPU box).
set -u
mkdir -p gpurun_out
timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final_cfg3.log 2>&1; echo "cfg3 rc=$?"; tail -1 gpurun_out/final_cfg3.log > gpurun_out/final_cfg3.json
timeout 900 python bench.py --config cfg4 --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/final_cfg4.log 2>&1; echo "cfg4 rc=$?"; tail -1 gpurun_out/final_cfg4.log > gpurun_out/final_cfg4.json
timeout 1500 python bench.py --config cfg5 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/final_cfg5.log 2>&1; echo "cfg5 rc=$?"; tail -1 gpurun_out/final_cfg5.log > gpurun_out/final_cfg5.json
timeout 1500 python bench.py --config cfg5 --precision pure_bf16 --swap-gb 36 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/final_cfg5_bf16.log 2>&1; echo "cfg5 bf16 rc=$?"; tail -1 gpurun_out/final_cfg5_bf16.log > gpurun_out/final_cfg5_bf16.json
timeout 900 python bench.py --impl reference --config cfg5 > gpurun_out/final_ref_cfg5.log 2>&1; echo "ref cfg5 rc=$?"; tail -1 gpurun_out/final_ref_cfg5.log > gpurun_out/final_ref_cfg5.json
for f in final_cfg3 final_cfg4 final_cfg5 final_cfg5_bf16 final_ref_cfg5; do echo "$f: $(cut -c1-400 gpurun_out/$f.json)"; done

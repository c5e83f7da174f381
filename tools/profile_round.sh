#!/bin/bash
# Profiles for profiles/ (run on the GPU box from the repo root):
#   launch list of the default bench (per-launch device time, cold/serialised)
#   + one `ncu --set full` capture per hot kernel.
# Summarise afterwards with tools/ncu_summary.py (see profiles/README.md).
set -u
TAG=${1:-r2}
mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/${TAG}_launches_bench_default.csv \
    python bench.py > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
echo "launch list rc=$?"
FULL="$NCU --set full --import-source on -c 1"
timeout 400 $FULL -k regex:k2_oneshot --launch-skip 3 -o gpurun_out/${TAG}_k2 \
    python bench.py --params 268435456 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
echo "k2 rc=$?"
timeout 400 $FULL -k regex:k1_oneshot --launch-skip 3 -o gpurun_out/${TAG}_k1 \
    python bench.py --params 1000000000 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
echo "k1 rc=$?"
MA_K3_VARIANT=0 timeout 400 $FULL -k regex:k3_v2 --launch-skip 3 -o gpurun_out/${TAG}_k3 \
    python tools/bench_k3.py --child --reps 2 > /dev/null 2>&1
echo "k3 rc=$?"
timeout 400 $FULL -k regex:k4_reduce_check --launch-skip 3 -o gpurun_out/${TAG}_k4_1src \
    python tools/bench_k4.py --n 268435456 --reps 1 > /dev/null 2>&1
echo "k4 1-src rc=$?"
timeout 400 $FULL -k regex:k4_reduce_check --launch-skip 12 -o gpurun_out/${TAG}_k4 \
    python tools/bench_k4.py --n 134217728 --reps 1 > /dev/null 2>&1
echo "k4 rc=$?"
timeout 400 $FULL -k regex:k_ingest --launch-skip 7 -o gpurun_out/${TAG}_ingest_bf16 \
    python tools/bench_k4.py --n 268435456 --reps 1 > /dev/null 2>&1
echo "ingest rc=$?"
# summaries on the box (the .ncu-rep files are ~10-20 MB each; gpurun
# copies back at most 64 MiB): keep K2's and K3's reports, drop the rest
python tools/ncu_summary.py ${TAG} gpurun_out/${TAG}_k2.ncu-rep:268435456:28 \
    gpurun_out/${TAG}_k1.ncu-rep:1000000000:2 gpurun_out/${TAG}_k3.ncu-rep:268435456:14 \
    gpurun_out/${TAG}_k4_1src.ncu-rep:268435456:4 gpurun_out/${TAG}_k4.ncu-rep:134217728:18 \
    gpurun_out/${TAG}_ingest_bf16.ncu-rep:268435456:4 && cp profiles/${TAG}_ncu_summary.json gpurun_out/
rm -f gpurun_out/${TAG}_k1.ncu-rep gpurun_out/${TAG}_k4_1src.ncu-rep gpurun_out/${TAG}_k4.ncu-rep \
    gpurun_out/${TAG}_ingest_bf16.ncu-rep
du -sh gpurun_out

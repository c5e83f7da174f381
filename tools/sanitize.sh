#!/bin/bash
# compute-sanitizer over the hot path (run on the GPU box from the repo root):
#   memcheck  — K1/K2/K3 parity suite (minus the exhaustive 2^32 sweeps and
#               the 8 B-param full-size runs, which take hours under the
#               tool), the NaN-semantics suite, the step-driver runtime
#               (graphs, NCCL, resume, the fused exchange at world 1), the
#               producer-side check, the hyper-parameter fuzz and the whole
#               peer-memory ZeRO step at world 1 (entry barrier, K4 + exit
#               barrier, K2 all-gather + barriers), all in ONE process;
#   racecheck + synccheck — the last-CTA completion-counter protocols (K1's
#               fused exchange, K4's exit barrier) in the same single-process
#               tests; memcheck + racecheck over the cold-parameter suite (K3's
#               shared-memory deferred-slot list and its drains);
#   ranks     — two ranks on one GPU where EACH rank process runs under the
#               tool (torchrun launches compute-sanitizer as the rank
#               program): bench.py with the fused p2p exchange inside a
#               graph, and the peer-memory ZeRO step (--zero-fused).
# Logs land in gpurun_out/<tag>_sanitize_<what>.txt (+ one log per rank
# process); the summary lines go to stdout.
set -u
TAG=${1:-r2}
mkdir -p gpurun_out
CS="compute-sanitizer --error-exitcode 99"
HEAVY="not mask_exhaustive and not cast_exhaustive and not fast_path_sqrt and not fast_path_division and not fast_path_general and not full_size and not megabuffer and not large_positions"
SINGLE="tests/test_gpu_stepper_runtime.py::test_fused_exchange_single_rank_in_a_graph tests/test_zero_step.py::test_fused_zero_step_single_process"
run() {
    local name=$1; shift
    local t0=$(date +%s)
    timeout 1500 "$@" > gpurun_out/${TAG}_sanitize_${name}.txt 2>&1
    local rc=$?
    echo "$name rc=$rc $(( $(date +%s) - t0 ))s $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/${TAG}_sanitize_${name}.txt | sort | uniq -c | tr '\n' ' ') $(grep -hE '[0-9]+ (passed|failed)' gpurun_out/${TAG}_sanitize_${name}.txt | tail -1)"
}
run memcheck_parity $CS --tool memcheck python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_nan.py tests/test_gpu_stepper_runtime.py tests/test_ingest.py tests/test_zero_step.py::test_fused_zero_step_single_process -k "$HEAVY"
run memcheck_fuzz $CS --tool memcheck python -m pytest -x -q -p no:cacheprovider tests/test_fuzz_hyper.py
# the cold routes: K3's shared-memory deferred list (atomicAdd + __syncthreads)
# and its vector / per-element drains, K2's inline second chance
run memcheck_cold $CS --tool memcheck python -m pytest -x -q -p no:cacheprovider tests/test_gpu_cold.py
run racecheck_cold $CS --tool racecheck --racecheck-report all python -m pytest -x -q -p no:cacheprovider tests/test_gpu_cold.py
# the speculative update during the transfer: backups, the applied-count
# marker and the restore kernel's last-CTA re-arm
run memcheck_spec $CS --tool memcheck python -m pytest -x -q -p no:cacheprovider tests/test_gpu_spec.py
run racecheck_spec $CS --tool racecheck --racecheck-report all python -m pytest -x -q -p no:cacheprovider tests/test_gpu_spec.py
run synccheck_spec $CS --tool synccheck python -m pytest -x -q -p no:cacheprovider tests/test_gpu_spec.py
run racecheck_protocols $CS --tool racecheck --racecheck-report all python -m pytest -x -q -p no:cacheprovider $SINGLE
run synccheck_protocols $CS --tool synccheck python -m pytest -x -q -p no:cacheprovider $SINGLE
ranks() {
    local name=$1 tool=$2; shift 2
    local t0=$(date +%s)
    MA_BENCH_BACKEND=gloo MA_BENCH_DEVICE=0 timeout 1500 python -m torch.distributed.run --nnodes=1 \
        --nproc-per-node=2 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) --no-python \
        compute-sanitizer --error-exitcode 99 --tool $tool --log-file gpurun_out/${TAG}_cs_${name}_rank%p.log \
        python bench.py --gpus 2 --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3 "$@" \
        > gpurun_out/${TAG}_sanitize_${name}.txt 2>&1
    local rc=$?
    echo "$name rc=$rc $(( $(date +%s) - t0 ))s $(cat gpurun_out/${TAG}_cs_${name}_rank*.log | grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' | sort | uniq -c | tr '\n' ' ') rank logs: $(ls gpurun_out/${TAG}_cs_${name}_rank*.log | wc -l)"
}
ranks memcheck_p2p_graph memcheck --config cfg3 --flag-exchange p2p --graph --params 20000000
ranks memcheck_zero memcheck --zero-fused --params 20000000
ranks racecheck_zero racecheck --zero-fused --params 20000000
ranks synccheck_p2p synccheck --config cfg3 --flag-exchange p2p --params 20000000

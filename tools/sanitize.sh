#!/bin/bash
# compute-sanitizer over the hot path (run on the GPU box from the repo root):
#   memcheck  — K1/K2/K3 parity suite (minus the exhaustive 2^32 sweeps and
#               the 8 B-param full-size runs, which take hours under the
#               tool), the NaN-semantics suite, the step-driver runtime
#               (graphs, NCCL, resume), the producer-side check and the
#               hyper-parameter fuzz;
#   racecheck + synccheck — the last-CTA completion-counter protocols: K1's
#               fused flag exchange and K4's exit barrier (2 processes on one
#               GPU, every child process tracked).
# Logs land in gpurun_out/sanitize_<tool>_<what>.txt; summarise into
# profiles/ with the ERROR SUMMARY lines.
set -u
TAG=${1:-r2}
mkdir -p gpurun_out
CS="compute-sanitizer --target-processes all --error-exitcode 99"
HEAVY="not mask_exhaustive and not cast_exhaustive and not fast_path_sqrt and not fast_path_division and not fast_path_general and not full_size and not megabuffer and not large_positions"
run() {
    local name=$1; shift
    local t0=$(date +%s)
    timeout 1500 "$@" > gpurun_out/${TAG}_sanitize_${name}.txt 2>&1
    local rc=$?
    echo "$name rc=$rc $(( $(date +%s) - t0 ))s $(grep -h 'ERROR SUMMARY' gpurun_out/${TAG}_sanitize_${name}.txt | sort | uniq -c | tr '\n' ' ') $(grep -hE '[0-9]+ (passed|failed)' gpurun_out/${TAG}_sanitize_${name}.txt | tail -1)"
}
run memcheck_parity $CS --tool memcheck python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_nan.py tests/test_gpu_stepper_runtime.py tests/test_ingest.py -k "$HEAVY"
run memcheck_fuzz $CS --tool memcheck python -m pytest -x -q -p no:cacheprovider tests/test_fuzz_hyper.py
run memcheck_xchg $CS --tool memcheck --log-file gpurun_out/${TAG}_cs_memcheck_xchg_%p.log python -m pytest -x -q -p no:cacheprovider "tests/test_multirank.py::test_ranks_on_b200_peer_exchange_fused_in_k1[2]" tests/test_reduce_scatter.py::test_two_ranks_reduce_scatter_over_peer_memory "tests/test_allgather.py" tests/test_peer_timeout.py::test_late_peer_inside_timeout_completes_identically
run racecheck_xchg $CS --tool racecheck --racecheck-report all --log-file gpurun_out/${TAG}_cs_racecheck_xchg_%p.log python -m pytest -x -q -p no:cacheprovider "tests/test_multirank.py::test_ranks_on_b200_peer_exchange_fused_in_k1[2]" tests/test_reduce_scatter.py::test_two_ranks_reduce_scatter_over_peer_memory
run synccheck_xchg $CS --tool synccheck --log-file gpurun_out/${TAG}_cs_synccheck_xchg_%p.log python -m pytest -x -q -p no:cacheprovider "tests/test_multirank.py::test_ranks_on_b200_peer_exchange_fused_in_k1[2]" tests/test_reduce_scatter.py::test_two_ranks_reduce_scatter_over_peer_memory
# per-process logs of the multi-process runs: one per tracked process
for f in gpurun_out/${TAG}_cs_*_%p.log gpurun_out/${TAG}_cs_*.log; do
    [ -f "$f" ] && echo "$f: $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' "$f" | tr '\n' ' ')"
done

# A/B round 2: K1 tail load flavour (1 = evict_last policy, 2 = default
# caching) x kept MiB, with K2 variant 20 (PDL) + PDL finish.  GPU box.
set -u
mkdir -p gpurun_out
out=gpurun_out/l2_ab2.txt
: > $out
run() {
  local label=$1; shift
  local envs=()
  while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  line=$(env "${envs[@]}" timeout 300 python bench.py "$@" --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1)
  echo "$label|$*|$(echo "$line" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,2),"us", round(d["roofline"]["step_frac"],4), "k2_us", round(d["roofline"]["k2_ms"]*1000,1), "k1_us", round(d["roofline"]["k1_ms"]*1000,1))' 2>&1 | tail -1)" >> $out
}
for rep in 1 2; do
for g in "" "--graph"; do
  run "v14 ldk0" MA_K2_VARIANT=14 MA_K1_LDK=0 MA_PDL_FINISH=0 -- --config cfg1 --steps 50 --warmup 5 $g
  for l in 1 2; do for mb in 16 32 48; do
    run "v20 fin ldk$l keep$mb" MA_K2_VARIANT=20 MA_PDL_FINISH=1 MA_K1_LDK=$l MA_K1_KEEP_MB=$mb -- --config cfg1 --steps 50 --warmup 5 $g
  done; done
done
done
for rep in 1 2; do
  run "cfg2 v14 ldk0" MA_K2_VARIANT=14 MA_K1_LDK=0 MA_PDL_FINISH=0 -- --steps 10 --warmup 3
  run "cfg2 v20 fin ldk2 keep32" MA_K2_VARIANT=20 MA_PDL_FINISH=1 MA_K1_LDK=2 MA_K1_KEEP_MB=32 -- --steps 10 --warmup 3
  run "cfg2 v20 fin ldk1 keep32" MA_K2_VARIANT=20 MA_PDL_FINISH=1 MA_K1_LDK=1 MA_K1_KEEP_MB=32 -- --steps 10 --warmup 3
done
cat $out

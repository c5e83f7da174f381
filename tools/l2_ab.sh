# A/B: L2 reuse of the gradients between K1 and K2 (MA_K1_LDK=1 keeps the
# last MA_K1_KEEP_MB of K1's gradients under an evict_last policy; K2
# variants 22/23 sweep the tiles back to front).  Run on the GPU box.
set -u
mkdir -p gpurun_out
out=gpurun_out/l2_ab.txt
: > $out
run() {  # label env... -- bench args
  local label=$1; shift
  local envs=()
  while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  line=$(env "${envs[@]}" timeout 300 python bench.py "$@" --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1)
  echo "$label|$*|$(echo "$line" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,2),"us", round(d["roofline"]["step_frac"],4), "k2_us", round(d["roofline"]["k2_ms"]*1000,1), "k1_us", round(d["roofline"]["k1_ms"]*1000,1))' 2>&1 | tail -1)" >> $out
}
for rep in 1 2; do
for g in "" "--graph"; do
  run "v14 ldk0" MA_K2_VARIANT=14 MA_K1_LDK=0 MA_PDL_FINISH=0 -- --config cfg1 --steps 50 --warmup 5 $g
  run "v22 ldk0" MA_K2_VARIANT=22 MA_K1_LDK=0 MA_PDL_FINISH=0 -- --config cfg1 --steps 50 --warmup 5 $g
  for mb in 32 64 96; do
    run "v22 ldk1 keep$mb" MA_K2_VARIANT=22 MA_K1_LDK=1 MA_K1_KEEP_MB=$mb MA_PDL_FINISH=0 -- --config cfg1 --steps 50 --warmup 5 $g
  done
  run "v14 ldk1 keep64" MA_K2_VARIANT=14 MA_K1_LDK=1 MA_K1_KEEP_MB=64 MA_PDL_FINISH=0 -- --config cfg1 --steps 50 --warmup 5 $g
  run "v20 ldk1 keep64 fin" MA_K2_VARIANT=20 MA_K1_LDK=1 MA_K1_KEEP_MB=64 MA_PDL_FINISH=1 -- --config cfg1 --steps 50 --warmup 5 $g
done
done
for v in "14 0" "22 1"; do
  set -- $v
  run "cfg2 v$1 ldk$2" MA_K2_VARIANT=$1 MA_K1_LDK=$2 MA_PDL_FINISH=0 -- --steps 10 --warmup 3
done
cat $out

# bench.py at edge partition sizes (1, 3, 4097, 100000001 params), both
# precisions, eager and graph: every line must parse (GPU box).
set -u
mkdir -p gpurun_out
out=gpurun_out/edge_sizes.txt
: > $out
for n in 1 3 4097 100000001; do
  for prec in mixed pure_bf16; do
    for g in "" "--graph"; do
      line=$(timeout 300 python bench.py --params $n --precision $prec --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 $g 2>&1 | tail -1)
      echo "n=$n $prec $g: $(echo "$line" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("ok", d["config"]["workload"], round(d["ms_per_step"],4), "ms", d["e2e"]["value"] > 0)' 2>&1 | tail -1)" >> $out
    done
  done
done
cat $out

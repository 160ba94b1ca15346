# time library variants on the Wide / HighRes configs: bash tools/var_cfg.sh
A="--steps 10 --warmup 3 --no-cpu-baseline --no-stream --no-flow --no-eval --no-densify --no-e2e"
for v in paper_1801_04720_b200/lib/var/*.so; do
  cp $v paper_1801_04720_b200/lib/libsgmsf.so
  for c in "wide 8" "highres 4"; do set -- $c
    timeout 600 python bench.py $A --config $1 --quads-per-gpu $2 > gpurun_out/bc.log 2>&1
    echo "$v $c $(tail -1 gpurun_out/bc.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), {k: round(v,3) for k, v in d["stage_ms"].items()})')"
  done
done

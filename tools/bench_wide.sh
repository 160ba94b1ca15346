#!/bin/bash
mkdir -p gpurun_out
A="--steps 10 --warmup 3 --no-cpu-baseline --no-stream --no-flow --no-eval --no-densify --no-e2e"
for c in "wide 8" "highres 4" "batch 8"; do
  set -- $c
  timeout 600 python bench.py $A --config $1 --quads-per-gpu $2 > gpurun_out/bc.log 2>&1
  tail -1 gpurun_out/bc.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"][:30], "| ms", round(d["ms_per_step"],3), {k: round(v,3) for k,v in d["stage_ms"].items()}, d["geometry"])' || tail -3 gpurun_out/bc.log
done

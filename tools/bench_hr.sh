#!/bin/bash
mkdir -p gpurun_out
A="--steps 10 --warmup 3 --no-cpu-baseline --no-stream --no-flow --no-eval --no-densify --no-e2e"
for c in "highres 2" "highres 4"; do
  set -- $c
  timeout 600 python bench.py $A --config $1 --quads-per-gpu $2 > gpurun_out/bc.log 2>&1
  tail -1 gpurun_out/bc.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"][:40], "| ms", round(d["ms_per_step"],3), d["stage_ms"], d["geometry"])' || tail -3 gpurun_out/bc.log
done

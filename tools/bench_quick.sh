#!/bin/bash
# quick main-step timing, twice: bash tools/bench_quick.sh
mkdir -p gpurun_out
A="--steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-stream --no-flow --no-eval --no-densify"
for k in 1 2; do
  timeout 300 python bench.py $A > gpurun_out/bq.log 2>&1
  tail -1 gpurun_out/bq.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), {k: round(v,3) for k, v in d["stage_ms"].items()})'
done

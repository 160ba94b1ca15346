#!/bin/bash
# main-step throughput / latency on the other BASELINE configs
mkdir -p gpurun_out
A="--steps 10 --warmup 3 --no-cpu-baseline --no-stream --no-flow --no-eval --no-densify"
for c in "driving 1" "driving 8" "wide 8" "highres 2" "highres 4" "tiny 64"; do
  set -- $c
  timeout 600 python bench.py $A --config $1 --quads-per-gpu $2 > gpurun_out/bc.log 2>&1
  tail -1 gpurun_out/bc.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"][:60], "| ms", round(d["ms_per_step"],3), "| frames/s", round(d["frames_per_s"],1), "| cells/s %.3g" % d["value"], "| e2e ms", round(d["e2e"]["ms_per_step"],3), "| frac", round(d["roofline"]["frac"],3))'
done

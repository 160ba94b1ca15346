#!/bin/bash
# upper bound of removing inter-warp / inter-band waits (results are wrong in that mode)
mkdir -p gpurun_out
A="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-stream --no-flow --no-eval --no-densify"
for f in 0 1 2; do
  SGM_DEBUG_FLAGS=$f timeout 300 python bench.py $A > gpurun_out/nd.log 2>&1
  echo "flags=$f $(tail -1 gpurun_out/nd.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), {k: round(v,3) for k,v in d["stage_ms"].items()})')"
done

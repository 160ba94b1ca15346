#!/bin/bash
mkdir -p gpurun_out
B="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-stream --no-eval"
timeout 600 python bench.py $B > gpurun_out/d1.log 2>&1
tail -1 gpurun_out/d1.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("with flow:", d["densify"]["ms_per_step"])'
timeout 600 python bench.py $B --no-flow > gpurun_out/d2.log 2>&1
tail -1 gpurun_out/d2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("no flow:", d["densify"]["ms_per_step"])'

#!/bin/bash
# ncu --set full of one forward + one backward sweep launch (8 Driving quads)
mkdir -p gpurun_out
A="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-stream --no-flow --no-eval --no-densify"
timeout 300 python bench.py $A > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 2 \
    -o gpurun_out/prof_sweep_x -f python bench.py $A > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?"

#!/bin/bash
# Round profile (run under gpurun from the repo root):
#   1. full bench.py (JSON line -> gpurun_out/bench_full.json)
#   2. ncu launch list of the same command (gpu__time_duration, cold, serialised)
#   3. ncu --set full on the two sweep kernels (one forward, one backward launch)
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
echo "bench exit $?"
tail -1 gpurun_out/bench_full.log > gpurun_out/bench_full.json
A="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
timeout 300 python bench.py $A > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py $A > gpurun_out/ncu_list.log 2>&1
echo "ncu list exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 2 \
    -o gpurun_out/prof_sweep_round python bench.py $A > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?"

#!/bin/bash
# Round profile (run under gpurun from the repo root):
#   1. full bench.py (JSON line -> gpurun_out/bench_full.json)
#   2. ncu launch list of the main step (gpu__time_duration, cold, serialised)
#   3. ncu --set full on the two sweep kernels (one forward, one backward launch)
#   4. ncu --set full on the evaluation kernel (row f1)
#   5. ncu launch list + --set full of the optical-flow kernels (row f2)
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
echo "bench exit $?"
tail -1 gpurun_out/bench_full.log > gpurun_out/bench_full.json
A="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-stream --no-flow --no-eval --no-densify"
timeout 300 python bench.py $A > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py $A > gpurun_out/ncu_list.log 2>&1
echo "ncu list exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 2 \
    -o gpurun_out/prof_sweep_round python bench.py $A > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?"
E="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-stream --no-flow --no-densify"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -c 1 \
    -o gpurun_out/prof_eval_round python bench.py $E > gpurun_out/ncu_eval.log 2>&1
echo "ncu eval exit $?"
timeout 300 python tools/flow_timing.py 8 3 > gpurun_out/flow_plain.log 2>&1 || { echo "flow run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/flow_launches.csv python tools/flow_timing.py 8 3 > gpurun_out/ncu_flow_list.log 2>&1
echo "ncu flow list exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"ff_prop_kernel|ff_knn_mma_kernel" -s 20 -c 3 \
    -o gpurun_out/prof_flow_round python tools/flow_timing.py 8 3 > gpurun_out/ncu_flow_full.log 2>&1
echo "ncu flow full exit $?"

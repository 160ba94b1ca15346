#!/bin/bash
# Round-2 profile (run under gpurun from the repo root):
#   1. the default bench.py line (64-quad configs[4] step + side sections) -> gpurun_out/r02_bench.json
#   2. ncu launch list of the main step (gpu__time_duration, cold, serialised)
#   3. ncu --set full of the two sweep kernels for every single-GPU config and the batch
#      (one forward + one backward launch each) -> gpurun_out/r02_sweep_<cfg>.ncu-rep
set -u
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/r02_bench.log 2> gpurun_out/r02_bench.err
echo "bench exit $?"
tail -1 gpurun_out/r02_bench.log > gpurun_out/r02_bench.json
A="--minimal --no-e2e --no-graph --steps 2 --warmup 3"
timeout 600 ncu -f --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02_launches.csv python bench.py $A > gpurun_out/r02_ncu_list.log 2>&1
echo "ncu list exit $?"
# the reports themselves are large: keep the raw-page CSV of each (what tools/ncu_traffic.py
# reads) and the full report of the 8-quad Driving step only (gpurun_out/ must stay < 64 MiB)
for spec in "batch 64" "driving 8" "driving 1" "wide 8" "highres 4" "tiny 64"; do
    set -- $spec
    timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:sweep_kernel -c 2 \
        -o gpurun_out/r02_sweep_$1x$2 python tools/sweep_time.py $1 $2 2 > gpurun_out/r02_ncu_$1x$2.log 2>&1
    echo "ncu $1x$2 exit $?"
    ncu -i gpurun_out/r02_sweep_$1x$2.ncu-rep --page raw --csv > gpurun_out/r02_sweep_$1x$2.raw.csv 2>/dev/null
    [ "$1x$2" = "drivingx8" ] || rm -f gpurun_out/r02_sweep_$1x$2.ncu-rep
done

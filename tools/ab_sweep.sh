#!/bin/bash
# A/B of sweep variants selected through the environment (run under gpurun)
for spec in "0 0 driving 8" "32 0 driving 8" "0 0 batch 64" "32 0 batch 64" "0 256 batch 64" "32 256 batch 64"; do
    set -- $spec
    if [ "$2" = "0" ]; then SGM_DEBUG_FLAGS=$1 python tools/sweep_time.py $3 $4 10 "flags$1-vg-default"
    else SGM_DEBUG_FLAGS=$1 SGM_VIEW_GROUP=$2 python tools/sweep_time.py $3 $4 10 "flags$1-vg$2"; fi
done

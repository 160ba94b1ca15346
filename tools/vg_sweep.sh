#!/bin/bash
# view-group sweep: timing then ncu DRAM bytes
for spec in "batch 64 10" "driving 8 20" "wide 8 20" "highres 4 10"; do
  for vg in 0 4 8 12 16 24 32; do
    set -- $spec
    SGM_VIEW_GROUP=$vg python tools/sweep_time.py $1 $2 $3 vg$vg 2>&1 | tail -1
  done
done
for vg in 0 8 16; do
  SGM_VIEW_GROUP=$vg timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sweep_kernel -c 2 --csv python tools/sweep_time.py batch 64 1 2>/dev/null | grep -E "dram|gpu__time" | awk -F'","' -v vg=$vg '{print "vg" vg, $5, $(NF-2), $NF}'
done

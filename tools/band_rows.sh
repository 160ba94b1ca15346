#!/bin/bash
# band-height sweep (SGM_BAND_ROWS) on the bench configs (run under gpurun)
for spec in "batch 64 10" "driving 8 20" "wide 8 20" "highres 4 10"; do
  for br in 0 12 13 14 15 16 17; do
    set -- $spec
    SGM_BAND_ROWS=$br python tools/sweep_time.py $1 $2 $3 br$br 2>&1 | tail -1
  done
done

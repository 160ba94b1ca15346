#!/bin/bash
# Time the optical-flow call for every library variant (run under gpurun):
#   bash tools/var_flow_time.sh [reps]     (variants: VAR_SRC=flow.cu bash tools/build_vars.sh ...)
REPS=${1:-2}
L=paper_1801_04720_b200/lib
cp $L/libsgmsf.so /tmp/libsgmsf.keep
for rep in $(seq $REPS); do
for v in ${VAR_DIR:-$L/var}/*.so; do
    cp $v $L/libsgmsf.so
    echo "== $(basename $v .so)"
    timeout 600 python tools/flow_timing.py 8 3 2>&1 | grep -v Warn | tail -3
done
done
cp /tmp/libsgmsf.keep $L/libsgmsf.so

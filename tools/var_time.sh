#!/bin/bash
# Time library variants (run under gpurun): bash tools/var_time.sh "cfg n steps; cfg n steps" [reps]
# For each paper_1801_04720_b200/lib/var/*.so: output digests (tools/ab_dump.py) and
# tools/sweep_time.py per spec; the default library is restored at the end.
SPECS="$1"; REPS=${2:-2}
L=paper_1801_04720_b200/lib
mkdir -p gpurun_out
cp $L/libsgmsf.so /tmp/libsgmsf.keep
for rep in $(seq $REPS); do
for v in ${VAR_DIR:-$L/var}/*.so; do
    name=$(basename $v .so)
    cp $v $L/libsgmsf.so
    if [ $rep = 1 ]; then
        timeout 600 python tools/ab_dump.py gpurun_out/digest_$name.json > /dev/null 2>&1
        echo "$name digest $(cat gpurun_out/digest_$name.json | sha256sum | cut -c1-12)"
    fi
    IFS=';' read -ra specs <<< "$SPECS"
    for spec in "${specs[@]}"; do
        read -r cfg n steps <<< "$spec"
        timeout 600 python tools/sweep_time.py $cfg $n $steps $name 2>&1 | tail -1
    done
done
done
cp /tmp/libsgmsf.keep $L/libsgmsf.so

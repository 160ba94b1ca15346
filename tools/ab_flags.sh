#!/bin/bash
# tools/ab_flags.sh "tree:flags ..." "cfg n steps; ..."  (run under gpurun)
VARIANTS="$1"; SPECS="$2"
for rep in 1 2; do
for vf in $VARIANTS; do
    v=${vf%%:*}; f=${vf#*:}
    IFS=';' read -ra specs <<< "$SPECS"
    for spec in "${specs[@]}"; do
        read -r cfg n steps <<< "$spec"
        (cd ab/$v && SGM_DEBUG_FLAGS=$f python ../../tools/sweep_time.py $cfg $n $steps $vf)
    done
done
done

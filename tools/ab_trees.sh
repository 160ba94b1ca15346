#!/bin/bash
# A/B of whole source trees under ab/<name> (run under gpurun): tools/ab_trees.sh "name..." "cfg n steps; ..."
VARIANTS="$1"
SPECS="$2"
for rep in 1 2; do
for v in $VARIANTS; do
    IFS=';' read -ra specs <<< "$SPECS"
    for spec in "${specs[@]}"; do
        read -r cfg n steps <<< "$spec"
        (cd ab/$v && python ../../tools/sweep_time.py $cfg $n $steps $v)
    done
done
done

# A/B of the trees under ab/ (run under gpurun): bitwise output digests vs ab/base, then timings
set -u
V="${AB_VARIANTS:-base}"
SPECS="${AB_SPECS:-driving 8 20; batch 64 10; wide 8 20; highres 4 10}"
for v in $V; do (cd ab/$v && python ../../tools/ab_dump.py ../../gpurun_out/ab_$v.json > /dev/null); done
for v in $V; do [ "$v" = base ] || python tools/ab_cmp.py gpurun_out/ab_base.json gpurun_out/ab_$v.json; done
bash tools/ab_trees.sh "$V" "$SPECS"

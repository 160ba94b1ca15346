#!/bin/bash
# Build library variants for A/B timing (run here, on the CPU box):
#   bash tools/build_vars.sh name1:"-DSGM_X=1 -DSGM_Y=2" name2:"..."
# -> paper_1801_04720_b200/lib/var/<name>.so (plus base.so = the default build), timed on the
# GPU box by tools/var_time.sh.  The default library is rebuilt at the end.
set -e
V=paper_1801_04720_b200/lib/var
rm -rf $V; mkdir -p $V
python -m paper_1801_04720_b200.build --force > /dev/null
cp paper_1801_04720_b200/lib/libsgmsf.so $V/base.so
for spec in "$@"; do
    name=${spec%%:*}; flags=${spec#*:}
    SGM_NVCC_EXTRA="$flags" python -m paper_1801_04720_b200.build --force > /dev/null
    cp paper_1801_04720_b200/lib/libsgmsf.so $V/$name.so
    echo "built $name ($flags)"
done
cp $V/base.so paper_1801_04720_b200/lib/libsgmsf.so
touch paper_1801_04720_b200/lib/libsgmsf.so

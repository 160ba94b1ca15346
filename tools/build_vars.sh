#!/bin/bash
# Build library variants for A/B timing (run here, on the CPU box):
#   bash tools/build_vars.sh name1:"-DSGM_X=1 -DSGM_Y=2" name2:"..."
# -> paper_1801_04720_b200/lib/var/<name>.so (plus base.so = the default build), timed on the
# GPU box by tools/var_time.sh.  Only VAR_SRC (default sweep.cu) is recompiled per variant.
set -e
PKG=paper_1801_04720_b200
V=${VAR_OUT:-$PKG/lib/var}
SRC=${VAR_SRC:-sweep.cu}
O=/tmp/sgm_var_objs
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a"
FL="-O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I include"
rm -rf $V $O; mkdir -p $V $O
for f in $PKG/csrc/*.cu; do
    [ "$(basename $f)" = "$SRC" ] && continue
    $NV $FL -c $f -o $O/$(basename $f).o &
done
wait
one() {
    $NV $FL $2 -c $PKG/csrc/$SRC -o $O/var_$1.o
    $NV -shared -cudart static -o $V/$1.so $O/*.cu.o $O/var_$1.o
    echo "built $1 ($2)"
}
one base "" &
for spec in "$@"; do
    one "${spec%%:*}" "${spec#*:}" &
done
wait
rm -f $O/var_*.o
python -m paper_1801_04720_b200.build > /dev/null

#!/bin/bash
# Like tools/build_vars.sh, but every source file is compiled with the variant's flags (for
# macros of sgm_internal.cuh that several files see):  bash tools/build_vars_all.sh name:"flags" ...
set -e
PKG=paper_1801_04720_b200
V=${VAR_OUT:-$PKG/lib/var}
O=/tmp/sgm_var_objs_all
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a"
FL="-O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I include"
rm -rf $V $O; mkdir -p $V $O
one() {
    mkdir -p $O/$1
    for f in $PKG/csrc/*.cu; do $NV $FL $2 -c $f -o $O/$1/$(basename $f).o & done
    wait
    $NV -shared -cudart static -o $V/$1.so $O/$1/*.o
    echo "built $1 ($2)"
}
one base ""
for spec in "$@"; do one "${spec%%:*}" "${spec#*:}"; done
python -m paper_1801_04720_b200.build > /dev/null

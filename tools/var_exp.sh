# time library variants: bash tools/var_exp.sh  (paper_1801_04720_b200/lib/var/*.so)
for v in paper_1801_04720_b200/lib/var/*.so; do
  cp $v paper_1801_04720_b200/lib/libsgmsf.so
  echo "$v"; bash tools/bench_quick.sh 2>&1 | tail -1
done

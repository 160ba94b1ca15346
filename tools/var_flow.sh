# time library variants on the flow call: bash tools/var_flow.sh
for v in paper_1801_04720_b200/lib/var/*.so; do
  cp $v paper_1801_04720_b200/lib/libsgmsf.so
  echo "$v"; python tools/flow_timing.py 8 3 2>&1 | tail -2
done

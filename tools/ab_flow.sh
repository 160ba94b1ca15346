# A/B of the optical-flow call between source trees under ab/ (run under gpurun)
for rep in 1 2; do for v in ${AB_VARIANTS:-base ffast}; do
  echo "== $v"; (cd ab/$v && python ../../tools/flow_timing.py 8 3 2>&1 | grep -v Warn | tail -3)
done; done

# latency-mode check (run under gpurun): the GPU suite, then driving x1 / x2 / x4 with and without fine sync
python -m pytest tests -m gpu -q -x > gpurun_out/fc_tests.log 2>&1; tail -2 gpurun_out/fc_tests.log
for n in 1 2 4 8; do
  for f in 0 1; do SGM_FINE_SYNC=$f python tools/sweep_time.py driving $n 20 fine$f; done
done
for c in "highres 1" "highres 2" "wide 1" "wide 2" "tiny 1" "batch 64"; do python tools/sweep_time.py $c 10 default; done

bash tools/bench_configs.sh
A="--steps 10 --warmup 3 --no-cpu-baseline --no-stream --no-flow --no-eval --no-densify --no-e2e"
for c in "highres 2 16" "driving 4 16" "driving 2 16"; do set -- $c
  SGM_BAND_ROWS=$3 timeout 600 python bench.py $A --config $1 --quads-per-gpu $2 > gpurun_out/bc.log 2>&1
  echo "$c"; tail -1 gpurun_out/bc.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3))'
done
for c in "driving 4" "driving 2"; do set -- $c
  timeout 600 python bench.py $A --config $1 --quads-per-gpu $2 > gpurun_out/bc.log 2>&1
  echo "$c auto"; tail -1 gpurun_out/bc.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3))'
done

#!/bin/bash
# Turn the artefacts of tools/round_final.sh (gpurun_out/) into the tracked round-2 summaries
# under profiles/ (run here, after the gpurun call):  bash tools/profiles_r02.sh
set -e
cp gpurun_out/r02_bench.json profiles/r02_bench.json
cp gpurun_out/rf_tests.log profiles/r02_gpu_tests.log
python tools/launch_summary.py gpurun_out/r02_launches.csv 'Command: `ncu -f --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --minimal --no-e2e --no-graph --steps 2 --warmup 3` (the 64-quad configs[4] step, tools/profile_r02.sh; 3 warm-up + 2 timed steps + 6 setup launches). ncu serialises launches and runs them cold: compare shares, not absolute times. The torch kernels are the L2 flush between steps.' > profiles/r02_launches.md
{
  echo "# r02: ncu --set full of the sweep kernels, every single-GPU config and the 64-quad batch"
  echo
  echo "Command (tools/profile_r02.sh): \`ncu -f --set full --clock-control none --import-source on -k regex:sweep_kernel -c 2 python tools/sweep_time.py <config> <quads> 2\` (one forward + one backward launch each). Algorithmic bytes: view-pixels x (2D + 16) forward, x (2D + 6) backward (DESIGN.md section 7). Lane-instructions per view-cell = smsp__inst_executed x 32 / (4 quads W H D). These tables feed profiles/ncu_traffic.json (bench.py roofline.traffic)."
  echo
  python tools/ncu_traffic.py gpurun_out/r02_sweep_*.raw.csv
} > profiles/r02_sweep_ncu_table.md
{
  echo "# r02: executed-instruction mix and stall samples of the sweeps (8 Driving quads)"
  echo
  echo "From \`ncu --set full --import-source on\` of \`tools/sweep_time.py driving 8\` (tools/round_final.sh), source page, SASS level; per position = per warp and image-row position (128 view-cells), \`python tools/src_hot.py r02_d8_src.csv <kernel> 14902500\`."
  for k in "sweep_kernel<(int)4, (bool)1, (bool)0" "sweep_kernel<(int)4, (bool)1, (bool)1"; do
    case "$k" in *"(bool)0") echo; echo "## sweep_fwd";; *) echo; echo "## sweep_bwd_wta";; esac
    echo '```'
    python tools/src_hot.py gpurun_out/r02_d8_src.csv "$k" 14902500 | head -42
    echo '```'
  done
} > profiles/r02_sweep_opmix.md
git diff --stat profiles/

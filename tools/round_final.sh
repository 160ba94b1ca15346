#!/bin/bash
# Round-end verification and profile (run under gpurun from the repo root): the GPU suite,
# smoke(), then tools/profile_r02.sh (bench line, launch list, per-config sweep ncu) and the
# source-level instruction mix of the 8-quad Driving sweeps.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/rf_tests.log 2>&1; tail -2 gpurun_out/rf_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf_smoke.log 2>&1; tail -1 gpurun_out/rf_smoke.log
bash tools/profile_r02.sh
ncu -i gpurun_out/r02_sweep_drivingx8.ncu-rep --page source --csv --print-source sass \
    > gpurun_out/r02_d8_src.csv 2>/dev/null
rm -f gpurun_out/r02_sweep_drivingx8.ncu-rep
ls -la gpurun_out | tail -30

#!/bin/bash
# Round verification (run under gpurun from the repo root): the whole GPU suite, smoke(),
# the densification fidelity measurement, then the round profile (bench + ncu).
python -m pytest tests -m gpu -q > gpurun_out/rc_tests.log 2>&1; tail -3 gpurun_out/rc_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1; tail -1 gpurun_out/rc_smoke.log
timeout 900 python tools/densify_gap.py 8 24 > gpurun_out/rc_dgap.log 2>&1; cat gpurun_out/rc_dgap.log
bash tools/profile_r02.sh

#!/bin/bash
# ncu --set full of one C2 tally2_kernel launch (FULL), report kept in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tally2 -s 1 -c 1 \
  -f -o gpurun_out/t2_full python scripts/profile_step.py --workload c2 --reps 2 > gpurun_out/t2_full.log 2>&1
tail -2 gpurun_out/t2_full.log

#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-tally2} -s 1 -c 1 \
  -o gpurun_out/${OUT:-prof} -f python scripts/profile_step.py --workload ${WL:-c2} --n_v ${NV:-12000} --reps 2 --flags ${FLAGS:-3} > gpurun_out/prof.log 2>&1
tail -3 gpurun_out/prof.log

#!/bin/bash
# ncu --set full of one 3-way C4 stage launch (FULL and CHECKSUM), reports kept in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for f in ${FLAGSET:-3 8}; do
  STAGE=${STAGE:-15} FLAGS=$f timeout 900 ncu --set full --import-source on --clock-control none -k regex:tally3 -c 1 \
    -f -o gpurun_out/t3_f$f python scripts/time3.py > gpurun_out/t3_f$f.log 2>&1
  tail -2 gpurun_out/t3_f$f.log
done

#!/bin/bash
# ncu --set full of one C4 stage (0 and 15, FULL) with the aligned 3-way epilogue.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02w2
mkdir -p $O
for st in 15 0; do
  STAGE=$st FLAGS=3 timeout 900 ncu --set full --import-source on --clock-control none -k regex:tally3 -c 1 \
    -f -o $O/t3_s${st}_f3 python scripts/time3.py > $O/t3_s${st}.log 2>&1
  tail -2 $O/t3_s${st}.log
done

#!/bin/bash
# 3-way FULL limiter matrix on C4 stages 0 and 15 (diagnostic builds; values wrong, timing only).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02e
mkdir -p $O
for st in 0 15; do
  echo "== stage $st FULL"
  STAGE=$st FLAGS=3 LIBS="default d3notma d3nomma d3noxf d3epi d3noepi d3nostore" ROUNDS=2 bash scripts/ab3.sh 2>&1 | tee -a $O/ab3.txt
  echo "== stage $st CHECKSUM"
  STAGE=$st FLAGS=8 LIBS="default d3epi" ROUNDS=1 bash scripts/ab3.sh 2>&1 | tee -a $O/ab3.txt
done

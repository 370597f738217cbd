#!/bin/bash
# 3-way: do the per-row column-term reads of the aligned epilogue cost LSU time?  (timing only)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02y
mkdir -p $O
for st in 0 15; do
  echo "== stage $st FULL"
  STAGE=$st FLAGS=3 LIBS="default d3cccline" ROUNDS=3 bash scripts/ab3.sh 2>&1 | sed 's/paper_1705_08213_b200.//' | tee -a $O/ab3.txt
done

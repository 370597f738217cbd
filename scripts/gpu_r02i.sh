#!/bin/bash
# 3-way FULL: is the record-address scatter (DRAM locality) what holds the epilogue at 4.8 TB/s?
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02i
mkdir -p $O
for st in 0 15; do
  echo "== stage $st FULL"
  STAGE=$st FLAGS=3 LIBS="default d3compact d3epi d3epicompact" ROUNDS=2 bash scripts/ab3.sh 2>&1 | sed 's/paper_1705_08213_b200.//' | tee -a $O/ab3.txt
done

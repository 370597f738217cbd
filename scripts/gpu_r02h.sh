#!/bin/bash
# 3-way FULL: does less operand traffic help?  (no B loads; both CTAs loading the same A rows)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02h
mkdir -p $O
for st in 0 15; do
  echo "== stage $st FULL"
  STAGE=$st FLAGS=3 LIBS="default d3nob d3samea d3notma" ROUNDS=2 bash scripts/ab3.sh 2>&1 | sed 's/paper_1705_08213_b200.//' | tee -a $O/ab3.txt
done

#!/bin/bash
# 3-way FULL: does multicasting one A tile to both CTAs of the pair cut its L2 cost
# (unlike two unicast loads of the same rows, d3samea)?  Timing only.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02l
mkdir -p $O
for st in 0 15; do
  echo "== stage $st FULL"
  STAGE=$st FLAGS=3 LIBS="default d3mca d3samea d3nob" ROUNDS=3 bash scripts/ab3.sh 2>&1 | sed 's/paper_1705_08213_b200.//' | tee -a $O/ab3.txt
done

#!/bin/bash
# 3-way FULL: what about the record addresses costs the epilogue?  Units as contiguous blocks
# (compact), the same blocks 128/256 MB apart (spread: TLB reach), blocks whose rows are
# 4,096 records apart (stride: the real row stride of stage 0).  Timing only.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02n
mkdir -p $O
for st in 0; do
  echo "== stage $st FULL"
  STAGE=$st FLAGS=3 LIBS="default d3stride d3odd d3epi d3epistride d3epiodd" ROUNDS=2 bash scripts/ab3.sh 2>&1 | sed 's/paper_1705_08213_b200.//' | tee -a $O/ab3.txt
done

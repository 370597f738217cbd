#!/bin/bash
# 3-way aligned record groups: GPU parity of everything through tally3_kernel, then A/B
# against the previous epilogue (libccc_old3.so) on C4 stages 0, 8, 15.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02mc
mkdir -p $O
echo "== tests"; timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for st in 0 8 15; do
  echo "== stage $st FULL"
  STAGE=$st FLAGS=3 LIBS="pp2 default" ROUNDS=3 bash scripts/ab3.sh 2>&1 | sed 's/paper_1705_08213_b200.//' | tee -a $O/ab3.txt
done

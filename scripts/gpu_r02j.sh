#!/bin/bash
# 3-way: J-banded unit order (pivot groups of G x every column tile of a row band) vs the
# tile-outer / pivot-inner order; parity of the banded order through the 3-way GPU tests.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02j
mkdir -p $O
L=$(pwd)/paper_1705_08213_b200/libccc_diag.so
echo "== parity (banded G=4)"; CCC_LIB=$L CCC_PGROUP=4 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_compact.py -m gpu -q -x -k "3way or three or triple or c4 or C4 or stage" 2>&1 | tail -2
for st in 0 15 8; do
  for r in 1 2; do
    for g in 0 1 2 4 8 16; do
      echo -n "stage $st G=$g: "; CCC_LIB=$L CCC_PGROUP=$g STAGE=$st FLAGS=3 timeout 120 python scripts/time3.py 2>&1 | tail -1 | sed 's/.*flags/flags/'
    done
  done
done 2>&1 | tee $O/banded.txt

#!/bin/bash
# round 2: store-line-coalescing diagnostics (2-way, 3-way) + the new full-size phase tests
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fullsize.py -q -k "phases or pieces" 2>&1 | tail -2
P=paper_1705_08213_b200
for v in libccc libccc_lineccc libccc_lineccc8 libccc; do
  CCC_LIB=$PWD/$P/$v.so timeout 300 python scripts/time_variants.py | tail -1
done
for v in libccc libccc_line3 libccc; do
  for st in 0 15; do STAGE=$st CCC_LIB=$PWD/$P/$v.so timeout 300 python scripts/time3.py | tail -1; done
done

#!/bin/bash
# 2-way sector-aligned record pairs: the GPU suite, then A/B against the previous epilogue
# (libccc_old2.so) on the C2 launch, FULL.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02r
mkdir -p $O
echo "== tests"; timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
LIBS="old2 default" ROUNDS=4 FLAGSET="3" bash scripts/ab_libs.sh 2>&1 | tee $O/ab.txt

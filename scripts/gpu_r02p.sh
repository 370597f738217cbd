#!/bin/bash
# 2-way FULL: would line-aligned rows help (records at a multiple of 8; timing only)?
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02q
mkdir -p $O
LIBS="default d2align d2align2" ROUNDS=4 FLAGSET="3" bash scripts/ab_libs.sh 2>&1 | tee $O/ab.txt

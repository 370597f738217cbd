#!/bin/bash
# 2-way FULL: does the FP64 cell math (DFMA) slow the int8 MMA?  (no-TMA isolates it)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02g
mkdir -p $O
LIBS="default nofp64 notma nofp64_notma ccconst_notma" ROUNDS=3 FLAGSET="3" bash scripts/ab_libs.sh 2>&1 | tee $O/ab.txt

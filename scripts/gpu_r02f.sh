#!/bin/bash
# 2-way FULL: is the CCC half's cost its math or its stores?  (+ the 3-way store-pattern ceiling)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02f
mkdir -p $O
timeout 300 ./scripts/storebench > $O/storebench.txt 2>&1; cat $O/storebench.txt
LIBS="default nocccst ccconst notma nocccst_notma ccconst_notma" ROUNDS=3 FLAGSET="3" bash scripts/ab_libs.sh 2>&1 | tee $O/ab.txt

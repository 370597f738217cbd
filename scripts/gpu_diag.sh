#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
export SUPERS="2048,2048 3072,1536 4096,1024 6144,768 2048,2304"
for lib in libccc_e4.so libccc_e8.so; do
  CCC_LIB=paper_1705_08213_b200/$lib FLAGS=3 timeout 300 python scripts/time_variants.py 2>&1 | tail -1
done
CCC_LIB=paper_1705_08213_b200/libccc_e8.so FLAGS=0 SUPERS="2048,2048" timeout 300 python scripts/time_variants.py 2>&1 | tail -1

#!/bin/bash
# A/B of library variants on one sparse C4 stage (time3s.py), interleaved.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
P=paper_1705_08213_b200
for r in $(seq ${ROUNDS:-2}); do
  for v in ${LIBS:-default}; do
    if [ "$v" = default ]; then L=$P/libccc.so; else L=$P/libccc_$v.so; fi
    echo -n "$v: "; CCC_LIB=$(pwd)/$L timeout 120 python scripts/time3s.py 2>&1 | tail -1
  done
done

#!/bin/bash
# A/B timing of library variants on one box, interleaved: LIBS="default X Y", ROUNDS=n.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
P=paper_1705_08213_b200
for r in $(seq ${ROUNDS:-2}); do
  for v in ${LIBS:-default}; do
    if [ "$v" = default ]; then L=$P/libccc.so; else L=$P/libccc_$v.so; fi
    echo -n "$v: "; CCC_LIB=$(pwd)/$L PRE=${PRE:-expand} FLAGSET="${FLAGSET:-3 3}" timeout 120 python ${SCRIPT:-scripts/time2_flags.py} 2>&1 | tail -3
  done
done

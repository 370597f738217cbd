#!/bin/bash
# 3-way kernel diagnostics: one C4 stage under diagnostic library variants and output flags.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
P=paper_1705_08213_b200
for v in ${VARIANTS:-default NOXF NOMMA NOEPI NOXF_NOMMA}; do
  if [ "$v" = default ]; then L=$P/libccc.so; else L=$P/libccc_$v.so; fi
  for f in ${FLAGSET:-3 8}; do
    CCC_LIB=$(pwd)/$L FLAGS=$f timeout 120 python scripts/time3.py 2>&1 | tail -1 | sed "s|$(pwd)/||"
    CCC_LIB=$(pwd)/$L FLAGS=$f timeout 120 python scripts/trace3.py 2>&1 | tail -1 | sed "s|$(pwd)/||"
  done
done

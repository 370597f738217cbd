#!/bin/bash
# 3-way: FULL / CHECKSUM stage time with and without the smem Hadamard transform (NOXF build).
cd "${GRAFT_REPO_ROOT}"
mkdir -p gpurun_out
P=paper_1705_08213_b200
for st in 15 0; do
for v in default NOXF; do
  if [ "$v" = default ]; then L=$P/libccc.so; else L=$P/libccc_$v.so; fi
  for f in 3 8; do
    STAGE=$st CCC_LIB=$(pwd)/$L FLAGS=$f timeout 120 python scripts/time3.py 2>&1 | tail -1 | sed "s|$(pwd)/||" | sed "s/^/stage $st /"
  done
done
done

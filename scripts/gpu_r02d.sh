#!/bin/bash
# 2-way FULL limiter: default vs software-pipelined TMEM loads (PIPE) vs no TMA / no MMA
# diagnostics, interleaved on one box; PIPE parity.  Outputs in gpurun_out/r02d/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02d
mkdir -p $O
echo "== PIPE parity"; CCC_LIB=$(pwd)/paper_1705_08213_b200/libccc_PIPE.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "2way or two or pair or c2 or C2" 2>&1 | tail -3
LIBS="default PIPE notma nomma nommatma" ROUNDS=3 FLAGSET="3 8 1" bash scripts/ab_libs.sh 2>&1 | tee $O/ab.txt

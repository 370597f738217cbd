#!/bin/bash
# Whole C4 step (16 stages, FULL), interleaved A/B of library builds: LIBS, ROUNDS.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02ab4
mkdir -p $O
P=paper_1705_08213_b200
for r in $(seq ${ROUNDS:-3}); do
  for v in ${LIBS:-default}; do
    if [ "$v" = default ]; then L=$P/libccc.so; else L=$P/libccc_$v.so; fi
    CCC_LIB=$(pwd)/$L timeout 600 python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu > $O/c4_$v.json 2>/dev/null
    python -c "import json; d=json.loads(open('$O/c4_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],1), round(d['ms_per_step_best'],1), d['clocks']['sm_mhz'], d.get('parity', {}).get('mismatches'))"
  done
done | tee -a $O/ab.txt

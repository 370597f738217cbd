#!/bin/bash
# A/B of library variants on the whole C4 3-way bench step (16 stages, FULL), interleaved.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
P=paper_1705_08213_b200
for r in $(seq ${ROUNDS:-2}); do
  for v in ${LIBS:-default}; do
    if [ "$v" = default ]; then L=$P/libccc.so; else L=$P/libccc_$v.so; fi
    echo -n "$v: "; CCC_LIB=$(pwd)/$L timeout 300 python bench.py --workload ${WL:-c4} --steps ${STEPS:-10} --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; c=d['clocks']
print('%.4g ms/step %.1f median %.1f kernel %.2f frac %.3f mhz %s W %s' % (d['value'], d['ms_per_step'], d['ms_per_step_median'], r['kernel_ms'], r['frac'], c['sm_mhz'], c.get('power_w_median')))"
  done
done

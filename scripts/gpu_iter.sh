#!/bin/bash
# Fast iteration: smoke, selected GPU tests, short benches, dram metrics of the tally kernels.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
echo "== smoke"; timeout 180 python __graft_entry__.py smoke 2>&1 | tail -5
echo "== tests"; timeout 900 python -m pytest tests -m gpu -x -q ${TESTS:-} 2>&1 | tail -8
for mode in ${MODES:-2}; do
  echo "== bench c2 mode=$mode"; CCC_TALLY2_CTA=$mode timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    r=d['roofline']; print('value %.4g ms/step %.3f kernel_ms %.3f TOPS %.1f frac %.3f clocks %s'%(d['value'],d['ms_per_step'],r['kernel_ms'],r['achieved'],r['frac'],d['clocks']))"
done
if [ -n "$C4" ]; then
  echo "== bench c4"; timeout 600 python bench.py --workload c4 --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    r=d['roofline']; print('value %.4g ms/step %.3f kernel_ms %.3f GB/s %.1f frac %.3f TOPS %.1f'%(d['value'],d['ms_per_step'],r['kernel_ms'],r['achieved'],r['frac'],r['tensor_TOPS']))"
fi
if [ -n "$METRICS" ]; then
  echo "== metrics"
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:tally -s 1 -c 1 --csv python scripts/profile_step.py --workload ${METRICS} --reps 2 2>/dev/null | grep -E "dram__|gpu__time|imma|hit_rate" | awk -F'","' '{print $13, $15}'
fi

#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() {
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:tally -s 1 -c 1 --csv python scripts/profile_step.py --workload c2 --reps 2 --flags $1 2>/dev/null | grep -E "dram__|gpu__time|imma|hit_rate" | awk -F'","' '{printf "%s=%s  ", $13, $15} END {print ""}' | sed 's/sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed/tensor%/; s/lts__t_sector_hit_rate.pct/l2hit/; s/dram__bytes_//g; s/.sum//g; s/gpu__time_duration/ns/'
}
echo "== tests"; timeout 900 python -m pytest tests -m gpu -x -q -k "2way or pack" 2>&1 | tail -3
for flags in ${FLAGSET:-3 1 2 5 11}; do
  echo "== flags=$flags"; run $flags
done

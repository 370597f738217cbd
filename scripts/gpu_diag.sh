#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() {
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:tally -s 1 -c 1 --csv python scripts/profile_step.py --workload c2 --reps 2 --flags $1 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{printf "%s=%s  ", $13, $15} END {print ""}' | sed 's/dram__bytes_//g; s/.sum//g; s/gpu__time_duration/ns/'
}
for ka in 0 1 0 1; do echo "== kalt=$ka"; CCC_KALT=$ka run 3; CCC_KALT=$ka SUPERS="2048,2048 3072,1536" FLAGS=3 timeout 300 python scripts/time_variants.py | tail -1; done

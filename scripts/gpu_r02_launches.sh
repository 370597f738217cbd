#!/bin/bash
# Launch lists (our kernels only, ncu gpu__time_duration, cold/serialised) of the default 2-way
# bench command and of the 3-way (c4) and sparse 3-way (c4s) commands.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02c
mkdir -p $O
K="tally|expand|pack|fs_|popc"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" -c 100 --csv --log-file $O/launches_c2.csv \
  python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e --no-3way > $O/l_c2.out 2>&1; tail -c 200 $O/l_c2.out; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" -c 200 --csv --log-file $O/launches_c4.csv \
  python bench.py --workload c4 --steps 2 --warmup 1 --no-cpu --no-e2e > $O/l_c4.out 2>&1; tail -c 200 $O/l_c4.out; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" -c 200 --csv --log-file $O/launches_c4s.csv \
  python bench.py --workload c4s --steps 2 --warmup 1 --no-cpu --no-e2e > $O/l_c4s.out 2>&1; tail -c 200 $O/l_c4s.out; echo

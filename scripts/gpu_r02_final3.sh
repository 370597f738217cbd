#!/bin/bash
# Round-2 end-of-session evidence: smoke, the whole GPU suite, the launch list of the default
# bench command (our kernels only).  Outputs in gpurun_out/r02z/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02z
mkdir -p $O
echo "== smoke"; timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
echo "== tests"; timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
echo "== launch list"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'tally|expand|pack|fs_|popc' -c 300 --csv \
  --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/launches_default.out 2>&1
tail -c 200 $O/launches_default.out

#!/bin/bash
# exact23 vs general-gamma epilogue timing + GPU tests
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
echo "== tests"; timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
for g in 0.6666666666666666 0.6666; do
  GAMMA=$g FLAGS=3 timeout 300 python scripts/time_variants.py 2>&1 | tail -1
  GAMMA=$g FLAGS=2 timeout 300 python scripts/time_variants.py 2>&1 | tail -1
  GAMMA=$g FLAGS=3 timeout 300 python scripts/time3.py 2>&1 | tail -1
done
echo "== bench c2"; timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -1
echo "== bench c4"; timeout 600 python bench.py --workload c4 --steps 2 --warmup 1 --no-cpu 2>&1 | tail -1

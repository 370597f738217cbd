#!/bin/bash
# Round-2 iteration: selected GPU tests, then 3-way C4 stage timings (stage 15 and 0).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
echo "== tests ${TESTS:-}"; timeout ${TEST_TIMEOUT:-1200} python -m pytest ${TESTS:-tests} -m gpu -x -q 2>&1 | tail -15
for st in ${STAGES:-15 0}; do
  for f in ${FLAGSET:-3}; do
    STAGE=$st FLAGS=$f timeout 120 python scripts/time3.py 2>&1 | tail -1 | sed "s/^/stage $st /"
  done
done

#!/bin/bash
# One gpurun session: smoke, GPU tests, short bench. Each step under its own timeout.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
echo "== smoke"; timeout 180 python __graft_entry__.py smoke 2>&1 | tail -20
echo "== tests ${TESTS:-}"; timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${TESTS:-} 2>&1 | tail -30
if [ -z "$NOBENCH" ]; then
echo "== bench"; timeout 600 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS:---no-cpu --no-e2e} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
fi

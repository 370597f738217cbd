#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
echo "== tests"; timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
echo "== bench c2"; timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
echo "== bench c4"; timeout 900 python bench.py --workload c4 --steps 2 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -3 gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
bash scripts/gpu_profile.sh

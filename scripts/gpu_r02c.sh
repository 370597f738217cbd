#!/bin/bash
# Round-2 (session 3): validate HEAD on a B200 (smoke, GPU suite, default bench) and run the
# store-throughput microbenchmark.  Outputs in gpurun_out/r02c/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02c
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
echo "== storebench2"; timeout 300 ./scripts/storebench2 > $O/storebench2.txt 2>&1; cat $O/storebench2.txt
echo "== smoke"; timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
echo "== default"; timeout 900 python bench.py > $O/bench_c2_default.json 2> $O/bench_c2_default.err; tail -2 $O/bench_c2_default.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02c/bench_c2_default.json").read().strip().splitlines()[-1])
print("C2", d["value"], d["ms_per_step"], d["ms_per_step_best"], d["clocks"], d.get("parity"))
t = d.get("three_way", {})
print("C4", t.get("value"), t.get("ms_per_step"), t.get("clocks"))
PY
echo "== tests"; timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -5

#!/bin/bash
# Bench lines after the aligned 3-way epilogue: default (C2 + three_way C4), reference arm.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02s3
mkdir -p $O
echo "== default"; timeout 900 python bench.py > $O/bench_c2_default.json 2> $O/bench_c2_default.err; tail -1 $O/bench_c2_default.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02s3/bench_c2_default.json").read().strip().splitlines()[-1])
print("C2", d["value"], d["ms_per_step"], d["ms_per_step_best"], d["clocks"]["sm_mhz"], d["parity"]["mismatches"])
t = d["three_way"]
print("C4", t["value"], t["ms_per_step"], t["ms_per_step_best"], t["clocks"], t.get("parity"), t["roofline"]["frac"])
PY
echo "== reference"; timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; tail -c 300 $O/bench_reference.json

#!/bin/bash
# Secondary 3-way bench lines after the aligned record groups: c4f32, c4paper, c5.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02x2
mkdir -p $O
for wl in c4f32 c4paper; do
  timeout 900 python bench.py --workload $wl --steps 3 --warmup 3 --no-e2e > $O/bench_$wl.json 2> $O/bench_$wl.err
  python -c "import json; d=json.loads(open('$O/bench_$wl.json').read().strip().splitlines()[-1]); print('$wl', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d.get('parity', {}).get('mismatches'))"
done
timeout 1500 python bench.py --workload c5 --steps 1 --warmup 3 --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
python -c "import json; d=json.loads(open('$O/bench_c5.json').read().strip().splitlines()[-1]); print('c5', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['decomposition_check']['match'])"

#!/bin/bash
# c4ck (CHECKSUM mode) and c4s (sparse, unchanged kernel) with the final library.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02x3
mkdir -p $O
for wl in c4ck c4s; do
  timeout 900 python bench.py --workload $wl --steps 3 --warmup 3 --no-e2e > $O/bench_$wl.json 2> $O/bench_$wl.err
  python -c "import json; d=json.loads(open('$O/bench_$wl.json').read().strip().splitlines()[-1]); print('$wl', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d.get('parity', {}).get('mismatches'))"
done

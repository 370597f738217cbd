#!/bin/bash
# Functional run of bench.py's N > 1 path on a one-GPU box: torchrun ranks over gloo
# (CCC_DIST_BACKEND=gloo) sharing the GPU; every line must carry decomposition_check.match.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02k
mkdir -p $O
run() {  # name nproc args...
  local n=$1 np=$2; shift 2
  CCC_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np "$@" \
    > $O/$n.json 2> $O/$n.err
  echo "$n rc=$? $(python -c "import json,sys; d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1]); print(d['n_gpus'], d['config'].get('n_v'), d['ms_per_step'], d['decomposition_check']['match'], d.get('phases_per_rank'))" 2>&1 | tail -1)"
}

run c4_p2 2 --workload c4 --steps 1 --warmup 3 --no-e2e

run c4_p3 3 --workload c4 --steps 1 --warmup 3 --no-e2e





"""bench.py's N > 1 path (torchrun, one process per rank) run functionally on a one-GPU box.

The driver's scaling run launches `bench.py --gpus N` under torchrun with NCCL, one GPU per
rank.  A test box has one GPU and NCCL refuses two ranks on one device, so these runs use
the CCC_DIST_BACKEND=gloo hook: the ranks share the GPU and the ring moves packed blocks
through host memory -- every other line of the decomposed step (block-circulant units,
row-band phases, tetrahedral units and pieces, the process grid with its CUDA IPC field
groups, the max-over-ranks timing) is the one the multi-GPU run executes.  Each line must
carry `decomposition_check.match`: the ranks' summed 128-bit checksum equals a
single-GPU CHECKSUM-mode run of the whole problem.  Not a timing.
"""
import json
import os
import random
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(nproc, *args):
    env = dict(os.environ, CCC_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + random.randrange(400)),
           "bench.py", "--gpus", str(nproc), *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == nproc
    assert "gloo test hook" in line["transport"]
    assert line["decomposition_check"]["match"], line["decomposition_check"]
    return line


@pytest.mark.gpu
@pytest.mark.parametrize("nproc", [2, 3])
def test_bench_2way_ring_ranks(nproc):
    line = _run(nproc, "--workload", "c1", "--steps", "2", "--warmup", "3")
    assert line["config"]["n_v"] == 256 * nproc or line["config"]["n_v"] % (256 * nproc) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("grid", ["2,1,1", "1,2,1", "1,1,2"])
def test_bench_2way_process_grid_ranks(grid):
    _run(2, "--workload", "c1", "--grid", grid, "--steps", "2", "--warmup", "3", "--no-e2e")


@pytest.mark.gpu
def test_bench_3way_tetrahedral_ranks():
    line = _run(2, "--workload", "c4", "--steps", "1", "--warmup", "3", "--no-e2e")
    assert line["config"]["n_v"] == 5120

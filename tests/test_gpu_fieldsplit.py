"""field-axis split with the reduce-scatter fused onto the tally GEMM.

Single GPU: every field slice runs on cuda:0 with local slot buffers (run_simulated) --
the export kernel (tcgen05 GEMM whose epilogue stores partial tiles into the owners'
slots), the slot addressing of waves and owners, and the owners' reduce + Eq.2-3
epilogue -- against the CPU oracle and against ccc_2way.  Two or more GPUs: the
torchrun-style orchestration with CUDA IPC peer slots over NVLink (skipped otherwise).
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synthgen

pytestmark = pytest.mark.gpu

ccc = pytest.importorskip("paper_1705_08213_b200.ccc")
from paper_1705_08213_b200 import fieldsplit  # noqa: E402

F64, F32, TAL, CK = ccc.OUT_CCC_F64, ccc.OUT_CCC_F32, ccc.OUT_TALLY, ccc.OUT_CHECKSUM


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


def _t(t):
    return t.cpu().numpy().astype(np.int64) & 0xFFFFFFFF


def _ccc_close(got, want, rtol=1e-12):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert np.all((want == 0) == (got == 0))
    nz = want != 0
    rel = np.abs(got[nz] - want[nz]) / np.abs(want[nz])
    assert rel.size == 0 or rel.max() <= rtol, rel.max()


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n_v,n_f", [(2, 8), (300, 1000), (600, 4097)])
def test_field_split_matches_oracle(world, n_v, n_f):
    codes = synthgen.make_codes("random", n_v, n_f, n_v + n_f + world)
    T, C, ck = fieldsplit.run_simulated(codes.cuda(), world, TAL | F64 | CK)
    torch.cuda.synchronize()
    To, Co = oracle.all_pairs(codes, oracle.GAMMA)
    np.testing.assert_array_equal(_t(T), To)
    _ccc_close(C.cpu().numpy(), Co)
    assert ccc.checksum_int(ck) == oracle.checksum(2, oracle.pair_list(n_v), To)


@pytest.mark.parametrize("wave_tiles", [1, 2, 3, 7])
def test_field_split_waves_and_f32(wave_tiles):
    """Several waves (slot buffers reused), ragged slices, fp32 CCC, another gamma."""
    n_v, n_f = 700, 3001
    codes = synthgen.make_codes("hwe", n_v, n_f, None)
    T, C, _ = fieldsplit.run_simulated(codes.cuda(), 3, TAL | F32, wave_tiles=wave_tiles, gamma=0.5)
    To, Co = oracle.all_pairs(codes, 0.5)
    np.testing.assert_array_equal(_t(T), To)
    _ccc_close(C.cpu().numpy(), Co, rtol=1e-6)


def test_field_split_equals_single_gpu_path_mid_size():
    """4 slices of a 3,000 x 40,000 problem: tallies identical to ccc_2way's."""
    n_v, n_f = 3000, 40000
    codes = synthgen.random_codes(n_v, n_f, seed=7, device="cuda")
    T, _, ck = fieldsplit.run_simulated(codes, 4, TAL | CK, wave_tiles=5)
    T2, _, ck2 = ccc.two_way(codes, out_flags=TAL | CK)
    torch.cuda.synchronize()
    assert bool((T == T2).all())
    assert ccc.checksum_int(ck) == ccc.checksum_int(ck2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_v, n_f, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    codes = synthgen.random_codes(n_v, n_f, seed=9, device="cuda")
    fs = fieldsplit.FieldSplit2Way(rank, world, n_v, n_f, wave_tiles=3, out_flags=TAL | CK)
    T, _, ck = fs.run(codes[:, fs.f0:fs.f1].contiguous())
    torch.cuda.synchronize()
    q.put((rank, ccc.checksum_int(ck)))
    fs.close()
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (NVLink peer slots)")
def test_field_split_two_gpus_ipc():
    import torch.multiprocessing as mp
    n_v, n_f, world = 1500, 20000, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(world, _free_port(), n_v, n_f, q), nprocs=world)
    total = sum(q.get()[1] for _ in range(world)) % (1 << 128)
    codes = synthgen.random_codes(n_v, n_f, seed=9, device="cuda")
    _, _, ck = ccc.two_way(codes, out_flags=CK)
    assert total == ccc.checksum_int(ck)


def _worker_one_gpu(rank, world, port, n_v, n_f, q):
    """Two processes on cuda:0: the real FieldSplit2Way (CUDA IPC slot buffers opened in
    the other process, gloo for the collectives) -- the multi-process path without NVLink."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    codes = synthgen.random_codes(n_v, n_f, seed=9, device="cuda")
    fs = fieldsplit.FieldSplit2Way(rank, world, n_v, n_f, wave_tiles=2, out_flags=TAL | CK)
    T, _, ck = fs.run(codes[:, fs.f0:fs.f1].contiguous())
    torch.cuda.synchronize()
    rows = [ccc.ccc_pair_index(n_v, i, j) for i, j in ((0, 1), (5, n_v - 1), (n_v - 2, n_v - 1))]
    q.put((rank, ccc.checksum_int(ck), T[rows].cpu().numpy()))
    fs.close()
    dist.destroy_process_group()


def test_field_split_ipc_two_processes_one_gpu():
    import torch.multiprocessing as mp
    n_v, n_f, world = 700, 3000, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker_one_gpu, args=(world, _free_port(), n_v, n_f, q), nprocs=world)
    res = [q.get() for _ in range(world)]
    total = sum(r[1] for r in res) % (1 << 128)
    codes = synthgen.random_codes(n_v, n_f, seed=9)
    To, _ = oracle.all_pairs(codes)
    assert total == oracle.checksum(2, oracle.pair_list(n_v), To)

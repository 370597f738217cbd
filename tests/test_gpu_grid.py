"""The 2-way process grid n_pv x n_pr x n_pf on the B200 (§4; SURVEY
§8(f) f3): the field split composed with the block-circulant vector ring and the n_pr
split of every block row.

Single GPU: grid.run_grid_simulated runs every rank's work on cuda:0 -- the block
geometries of the vector decomposition, the export GEMM of every field slice into the
owners' slots (ccc_2way_fs_block_export: tcgen05 GEMM, partial tiles stored from the
epilogue), and every owner's reduce + Eq.2-3 finish (ccc_2way_fs_block_finish) -- and
the union of all parts is compared with the CPU oracle record by record.  Multi-process:
grid.Grid2Way in 4 processes sharing cuda:0 (gloo for the ring and the collectives, CUDA
IPC for the slots), checksums summed over ranks against the oracle's.
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
from paper_1705_08213_b200 import decomp, grid as gridmod  # noqa: E402

F64, F32, TAL, CK = ccc.OUT_CCC_F64, ccc.OUT_CCC_F32, ccc.OUT_TALLY, ccc.OUT_CHECKSUM


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


def _band_pairs(n_v, bounds, u, lo, hi):
    """Global pair indices (ccc_pair_index) of a band's records, in record order."""
    a0, b0 = bounds[u.a][0], bounds[u.b][0]
    n_b = bounds[u.b][1] - b0
    out = []
    for il in range(lo, hi):
        jl = np.arange(il + 1 if u.diag else 0, n_b, dtype=np.int64)
        i, j = a0 + il, b0 + jl
        out.append(i * (2 * n_v - i - 1) // 2 + (j - i - 1))
    return np.concatenate(out) if out else np.zeros(0, np.int64)


def _ccc_close(got, want, rtol):
    assert np.all((want == 0) == (got == 0))
    nz = want != 0
    rel = np.abs(got[nz] - want[nz]) / np.abs(want[nz])
    assert rel.size == 0 or rel.max() <= rtol, rel.max()


@pytest.mark.parametrize("shape", [(1, 1, 1), (2, 1, 2), (1, 2, 2), (2, 2, 1), (3, 1, 2), (2, 2, 2),
                                   (4, 1, 3), (3, 2, 3)])
def test_grid_simulated_matches_oracle(shape):
    """Every part of every rank on one GPU: all pairs exactly once, tallies bit-exact, CCC
    within 1e-12, checksum = the oracle's (ragged blocks, slices and a 2-tile wave size)."""
    n_v, n_f = 700, 3001
    g = decomp.Grid(*shape)
    codes = synthgen.random_codes(n_v, n_f, seed=17)
    res, ck = gridmod.run_grid_simulated(codes.cuda(), g, TAL | F64 | CK, wave_tiles=2)
    torch.cuda.synchronize()
    To, Co = oracle.all_pairs(codes)
    bounds = decomp.block_bounds(n_v, g.n_pv)
    seen = np.zeros(len(To), np.int64)
    for u, lo, hi, T, C in res:
        idx = _band_pairs(n_v, bounds, u, lo, hi)
        seen[idx] += 1
        np.testing.assert_array_equal(T.cpu().numpy().astype(np.int64) & 0xFFFFFFFF, To[idx])
        _ccc_close(C.cpu().numpy(), Co[idx], 1e-12)
    assert (seen == 1).all()
    assert ccc.checksum_int(ck) == oracle.checksum(2, oracle.pair_list(n_v), To)


def test_grid_simulated_f32_gamma_half():
    """fp32 CCC and another gamma through the grid's finish (general-gamma weights)."""
    n_v, n_f = 520, 2049
    g = decomp.Grid(2, 1, 3)
    codes = synthgen.make_codes("hwe", n_v, n_f, None)
    res, _ = gridmod.run_grid_simulated(codes.cuda(), g, TAL | F32, gamma=0.5)
    To, Co = oracle.all_pairs(codes, 0.5)
    bounds = decomp.block_bounds(n_v, g.n_pv)
    for u, lo, hi, T, C in res:
        idx = _band_pairs(n_v, bounds, u, lo, hi)
        np.testing.assert_array_equal(T.cpu().numpy().astype(np.int64) & 0xFFFFFFFF, To[idx])
        _ccc_close(C.cpu().numpy().astype(np.float64), Co[idx], 1e-6)


def test_grid_block_export_finish_equals_block_kernel():
    """One off-diagonal block and one diagonal row band at a mid size, 4 field slices:
    the reduced records equal ccc_2way_block's on the full fields (same layout)."""
    n_f = 20000
    codes = synthgen.random_codes(2600, n_f, seed=21, device="cuda")
    A, B = codes[:1200], codes[1200:]
    exA = ccc.ccc_expand(ccc.ccc_pack(A), n_f)
    exB = ccc.ccc_expand(ccc.ccc_pack(B), n_f)
    for diag, (X, Y, a0, b0, lo, hi) in ((False, (exA, exB, 0, 1200, 100, 1111)), (True, (exA, exA, 0, 0, 300, 900))):
        n_a, n_b = X[0].shape[0], Y[0].shape[0]
        n_rec = ccc.block_records(n_a, lo, hi, n_b, diag)
        T1, C1, k1 = ccc._outputs(n_rec, 4, TAL | F64 | CK, "cuda")
        ccc.ccc_2way_block(*X, a0, lo, hi, *Y, b0, diag, n_f, TAL | F64 | CK, T1, C1, k1)
        world = 4
        sl = [(r * n_f // world, (r + 1) * n_f // world) for r in range(world)]
        parts = []
        for f0, f1 in sl:
            xa = ccc.ccc_expand(ccc.ccc_pack(A[:, f0:f1].contiguous()), f1 - f0)
            xb = xa if diag else ccc.ccc_expand(ccc.ccc_pack(B[:, f0:f1].contiguous()), f1 - f0)
            parts.append((xa, xb))
        tiles = ccc.ccc_2way_fs_block_tiles(n_a, lo, hi, n_b, diag)
        nbytes = ccc.ccc_2way_fs_slot_bytes(world, 0, tiles)
        slots = [torch.empty(nbytes // 4, dtype=torch.int32, device="cuda") for _ in range(world)]
        ptrs = torch.tensor([s.data_ptr() for s in slots], dtype=torch.int64, device="cuda")
        for f, (xa, xb) in enumerate(parts):
            ccc.ccc_2way_fs_block_export(xa[0], xa[1], lo, hi, xb[0], xb[1], diag, sl[f][1] - sl[f][0], ptrs, f,
                                         world, 0, tiles)
        T2, C2, k2 = ccc._outputs(n_rec, 4, TAL | F64 | CK, "cuda")
        for f in range(world):
            ccc.ccc_2way_fs_block_finish(slots[f], X[1], a0, lo, hi, Y[1], b0, diag, n_f, f, world, 0, tiles,
                                         TAL | F64 | CK, T2, C2, k2)
        torch.cuda.synchronize()
        assert bool((T1 == T2).all())
        _ccc_close(C2.cpu().numpy(), C1.cpu().numpy(), 1e-13)
        assert ccc.checksum_int(k1) == ccc.checksum_int(k2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, shape, port, n_v, n_f, max_rec, q):
    """One grid rank on cuda:0: Grid2Way with the CUDA backend, gloo collectives, CUDA IPC
    slots opened in the field partners' processes."""
    import torch.distributed as dist
    from paper_1705_08213_b200.fieldsplit import field_slices
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    g = decomp.Grid(*shape)
    dist.init_process_group("gloo", rank=rank, world_size=g.world)
    v, r, f = g.coords(rank)
    bounds = decomp.block_bounds(n_v, g.n_pv, align=1)
    f0, f1 = field_slices(n_f, g.n_pf)[f]
    lo, hi = bounds[v]
    codes = synthgen.random_codes(n_v, n_f, seed=23, device="cuda")[lo:hi, f0:f1].contiguous()
    be = gridmod.CudaGridBackend(f1 - f0, n_f, ccc.GAMMA, TAL | CK)
    gr = gridmod.Grid2Way(be, g, rank, bounds, max_records=max_rec, wave_tiles=2)
    gr.run(be.pack(codes))
    torch.cuda.synchronize()
    q.put((rank, ccc.checksum_int(gr.ck)))
    gr.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("shape,max_rec", [((2, 1, 2), None), ((1, 2, 2), 30000)])
def test_grid_processes_one_gpu(shape, max_rec):
    """4 ranks of a grid as processes on one GPU: the real Grid2Way (ring shifts of packed
    blocks, allele-sum all-reduce, IPC slot exports, barrier, finish, phases); the ranks'
    checksums add up to the oracle's."""
    import torch.multiprocessing as mp
    n_v, n_f = 600, 2500
    world = decomp.Grid(*shape).world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(shape, _free_port(), n_v, n_f, max_rec, q), nprocs=world)
    total = sum(q.get()[1] for _ in range(world)) % (1 << 128)
    codes = synthgen.random_codes(n_v, n_f, seed=23)
    To, _ = oracle.all_pairs(codes)
    assert total == oracle.checksum(2, oracle.pair_list(n_v), To)


@pytest.mark.parametrize("shape", [(2, 1, 2), (2, 2, 2), (4, 1, 2)])
def test_grid_simulated_C2_size_checksum(shape):
    """configs[1] (20,000 x 50,000) on simulated grids: every rank's export/finish work on one
    GPU; the ranks' checksums (every record's tallies and global indices) sum to the
    checksum of the single-GPU path."""
    n_v, n_f = 20000, 50000
    codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
    _, _, k1 = ccc.ccc_2way_codes(codes, out_flags=CK)
    _, k2 = gridmod.run_grid_simulated(codes, decomp.Grid(*shape), CK, align=256)
    torch.cuda.synchronize()
    assert ccc.checksum_int(k1) == ccc.checksum_int(k2)

"""the paper's popcount tally (mGEMM2 idea) on CUDA cores,
through the C ABI, against the CPU oracle and against the tensor-core path.

Bars as for ccc_2way: tallies bit-exact, CCC within 1e-12 relative (1e-6 in
fp32), checksums equal.
"""
import numpy as np
import pytest
import torch

import oracle
import synthgen

pytestmark = pytest.mark.gpu

ccc = pytest.importorskip("paper_1705_08213_b200.ccc")

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


def _check(codes, flags=TAL | F64 | CK, gamma=oracle.GAMMA):
    n_v, n_f = codes.shape
    packed = ccc.ccc_pack(codes.cuda())
    T, C, ck = ccc.ccc_2way_popcount(packed, n_f, gamma, flags)
    torch.cuda.synchronize()
    To, Co = oracle.all_pairs(codes, gamma)
    if flags & TAL:
        np.testing.assert_array_equal(_t(T), To)
    if flags & F64:
        _ccc_close(C.cpu().numpy(), Co)
    if flags & F32:
        _ccc_close(C.cpu().numpy(), Co, rtol=1e-6)
    if flags & CK:
        assert ccc.checksum_int(ck) == oracle.checksum(2, oracle.pair_list(n_v), To)


@pytest.mark.parametrize("n_v", [2, 3, 127, 128, 129, 300])
@pytest.mark.parametrize("n_f", [1, 15, 16, 17, 255, 256, 257, 1000])
def test_popcount_ragged_shapes(n_v, n_f):
    """Tile edges (128 pairs) and word edges (16 genotypes per word, 256 per step)."""
    _check(synthgen.make_codes("random", n_v, n_f, n_v * 7 + n_f))


@pytest.mark.parametrize("kind", ["hwe", "planted"])
def test_popcount_other_inputs(kind):
    _check(synthgen.make_codes(kind, 200, 777, None))


def test_popcount_f32_gamma_and_degenerate():
    codes = synthgen.make_codes("random", 150, 300, 5)
    _check(codes, flags=TAL | F32)
    _check(codes, flags=F64, gamma=0.5)
    for c in (torch.zeros(70, 300, dtype=torch.uint8), torch.full((70, 300), 3, dtype=torch.uint8)):
        _check(c)
    packed = ccc.ccc_pack(torch.zeros(1, 5, dtype=torch.uint8).cuda())
    assert ccc.ccc_2way_popcount(packed, 5)[0].shape == (0, 4)


def test_popcount_equals_tensor_path_mid_size():
    """Bit-identical tallies to the tcgen05 path on a multi-tile problem (2,000 x 20,000)."""
    n_v, n_f = 2000, 20000
    codes = synthgen.random_codes(n_v, n_f, seed=11, device="cuda")
    packed = ccc.ccc_pack(codes)
    Tp, Cp, ckp = ccc.ccc_2way_popcount(packed, n_f, out_flags=TAL | F64 | CK)
    Tt, Ct, ckt = ccc.ccc_2way(packed, n_f, out_flags=TAL | F64 | CK)
    torch.cuda.synchronize()
    assert bool((Tp == Tt).all())
    assert ccc.checksum_int(ckp) == ccc.checksum_int(ckt)
    rel = ((Cp - Ct).abs() / Ct.abs().clamp_min(1e-300)).max().item()
    assert rel <= 1e-14
    rng = np.random.default_rng(3)
    pairs = sorted({(int(i), int(j)) for i, j in rng.integers(0, n_v, (400, 2)) if i < j})
    To, Co = oracle.pairs(codes.cpu(), np.array(pairs, dtype=np.int64))
    rows = torch.tensor([ccc.ccc_pair_index(n_v, i, j) for i, j in pairs], device="cuda")
    np.testing.assert_array_equal(_t(Tp[rows]), To)
    _ccc_close(Cp[rows].cpu().numpy(), Co)

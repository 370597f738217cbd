"""Sparse (missing-data) 2-way mode (reading A-17) through
the C ABI against the sparse oracle: tallies bit-exact, CCC within 1e-12 (fp64) / 1e-6
(fp32), checksums equal."""
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


def _close(got, want, rtol):
    got = np.asarray(got, np.float64)
    assert np.all((want == 0) == (got == 0))
    nz = want != 0
    assert not nz.any() or (np.abs(got[nz] - want[nz]) / np.abs(want[nz])).max() <= rtol


def _full(codes, flags=TAL | F64 | CK, gamma=oracle.GAMMA):
    n_v, n_f = codes.shape
    To, Co, _ = oracle.sparse_all_pairs(codes, gamma)
    T, C, ck = ccc.ccc_2way_sparse(ccc.ccc_pack(codes.cuda()), n_f, gamma, flags)
    if flags & TAL:
        np.testing.assert_array_equal(_t(T), To)
    if flags & F64:
        _close(C.cpu().numpy(), Co, 1e-12)
    if flags & F32:
        _close(C.cpu().numpy(), Co, 1e-6)
    if flags & CK:
        assert ccc.checksum_int(ck) == oracle.checksum(2, oracle.pair_list(n_v), To)


def test_expand_sparse_layout():
    n_v, n_f = 37, 333
    codes = synthgen.sparse_codes(n_v, n_f, seed=21)
    X, s, c, w = ccc.ccc_expand_sparse(ccc.ccc_pack(codes.cuda()), n_f)
    cn = codes.numpy()
    present = cn != oracle.MISSING
    n1 = np.where(present, ((cn >> 1) & 1) + (cn & 1), 0)
    Xn = X.cpu().numpy()
    assert Xn.shape == (2 * 48, ccc.ccc_k_pad(n_f))
    exp = np.zeros_like(Xn)
    for i in range(n_v):
        exp[32 * (i // 16) + i % 16, :n_f] = n1[i]
        exp[32 * (i // 16) + 16 + i % 16, :n_f] = present[i]
    np.testing.assert_array_equal(Xn, exp)
    S, cnt = oracle.sparse_sums(codes)
    np.testing.assert_array_equal(s.cpu().numpy(), S[:, 1])
    np.testing.assert_array_equal(c.cpu().numpy(), cnt)
    f = S / np.maximum(2 * cnt, 1)[:, None]
    np.testing.assert_allclose(w.cpu().numpy(), 1 - oracle.GAMMA * f, rtol=1e-15, atol=0)


@pytest.mark.parametrize("n_v,n_f", [(2, 1), (3, 65), (17, 128), (40, 333), (130, 65),
                                     (257, 1000), (300, 129)])
def test_sparse_full(n_v, n_f):
    _full(synthgen.sparse_codes(n_v, n_f, seed=n_v + n_f))


def test_sparse_variants():
    codes = synthgen.sparse_codes(150, 301, seed=22)
    _full(codes, flags=TAL | F32)
    _full(codes, flags=F64, gamma=0.0)
    _full(codes, flags=CK)


def test_sparse_degenerate():
    codes = synthgen.sparse_codes(50, 200, seed=23)
    codes[7] = oracle.MISSING                          # one vector entirely missing
    codes[20, :100] = oracle.MISSING
    codes[21, 100:] = oracle.MISSING                   # disjoint present sets: c_ij = 0
    _full(codes)
    dense = synthgen.random_codes(60, 250, seed=24)
    dense[dense == oracle.MISSING] = 1                 # no missing entry: equals dense mode
    T, C, _ = ccc.ccc_2way_sparse(ccc.ccc_pack(dense.cuda()), 250)
    Td, Cd, _ = ccc.two_way(dense.cuda())
    assert torch.equal(T, Td)
    _close(C.cpu().numpy(), Cd.cpu().numpy(), 1e-12)


def test_sparse_blocks_rect_and_row_ranges():
    """Off-diagonal blocks, diag blocks with a row range starting off a 16-vector group."""
    n_v, n_f = 300, 400
    codes = synthgen.sparse_codes(n_v, n_f, seed=25)
    To, Co, _ = oracle.sparse_all_pairs(codes)
    a0, a1 = 0, 150
    XA, _, _, wA = ccc.ccc_expand_sparse(ccc.ccc_pack(codes[a0:a1].contiguous().cuda()), n_f)
    XB, _, _, wB = ccc.ccc_expand_sparse(ccc.ccc_pack(codes[a1:].contiguous().cuda()), n_f)
    lo, hi = 37, 131
    nB = n_v - a1
    m = (hi - lo) * nB
    T = torch.empty((m, 4), dtype=torch.int32, device="cuda")
    C = torch.empty((m, 4), dtype=torch.float64, device="cuda")
    ck = torch.zeros(2, dtype=torch.int64, device="cuda")
    ccc.ccc_2way_sparse_block(XA, wA, a1 - a0, a0, lo, hi, XB, wB, nB, a1, False, n_f,
                              TAL | F64 | CK, T, C, ck)
    idx = np.array([(a0 + i, a1 + j) for i in range(lo, hi) for j in range(nB)])
    rows = [ccc.ccc_pair_index(n_v, i, j) for i, j in idx]
    np.testing.assert_array_equal(_t(T), To[rows])
    _close(C.cpu().numpy(), Co[rows], 1e-12)
    assert ccc.checksum_int(ck) == oracle.checksum(2, idx, To[rows])
    X, _, _, w = ccc.ccc_expand_sparse(ccc.ccc_pack(codes.cuda()), n_f)
    lo, hi = 45, 213
    m = sum(n_v - 1 - i for i in range(lo, hi))
    Td = torch.empty((m, 4), dtype=torch.int32, device="cuda")
    ccc.ccc_2way_sparse_block(X, w, n_v, 0, lo, hi, X, w, n_v, 0, True, n_f, TAL, Td)
    r0 = ccc.ccc_pair_index(n_v, lo, lo + 1)
    np.testing.assert_array_equal(_t(Td), To[r0:r0 + m])


def test_sparse_compact():
    n_v, n_f = 260, 500
    codes = synthgen.sparse_codes(n_v, n_f, seed=26)
    To, Co, _ = oracle.sparse_all_pairs(codes)
    m = np.unique(Co.max(1))
    thr = 0.5 * (m[-200] + m[-199])
    cm = ccc.Compact(thr, 1000, 4)
    ccc.ccc_2way_sparse(ccc.ccc_pack(codes.cuda()), n_f, compact=cm)
    n, keys, T, C = cm.result()
    exp = np.nonzero(Co.max(1) > thr)[0]
    assert n == len(exp)
    idx = ccc.decode_keys(keys, 2).cpu().numpy()
    rows = np.array([ccc.ccc_pair_index(n_v, int(i), int(j)) for i, j in idx])
    np.testing.assert_array_equal(np.sort(rows), exp)
    np.testing.assert_array_equal(_t(T), To[rows])
    _close(C.cpu().numpy(), Co[rows], 1e-12)


def test_sparse_large_sampled():
    """8,192 x 50,000 (C2's field count): stratified sampled pairs against the oracle and
    sum T = 4 c_ij (c_ij recomputed from the codes on the GPU) on every record."""
    n_v, n_f = 8192, 50000
    codes = synthgen.sparse_codes(n_v, n_f, seed=27, device="cuda")
    T, C, _ = ccc.ccc_2way_sparse(ccc.ccc_pack(codes), n_f, out_flags=TAL | F64)
    tot = T.to(torch.int64).sum(1)
    assert bool((tot % 4 == 0).all()) and bool((tot <= 4 * n_f).all())
    pres = (codes != oracle.MISSING).to(torch.float32)
    cij = pres @ pres.t()                                 # exact in fp32 (< 2^24)
    iu = torch.triu_indices(n_v, n_v, 1, device="cuda")
    assert torch.equal(tot, cij[iu[0], iu[1]].to(torch.int64) * 4)
    del cij, pres, iu
    rng = np.random.default_rng(7)
    pr = set()
    for _ in range(3000):
        i = int(rng.integers(0, n_v - 1))
        pr.add((i, int(rng.integers(i + 1, n_v))))
    for e in (0, 15, 16, 127, 128, 255, 256, 4095, 4096, n_v - 2):
        pr.add((e, e + 1))
        pr.add((e, n_v - 1))
    pr = np.array(sorted(pr), dtype=np.int64)
    To, Co, _ = oracle.sparse_pairs(codes.cpu(), pr)
    rows = torch.tensor([ccc.ccc_pair_index(n_v, int(i), int(j)) for i, j in pr], device="cuda")
    np.testing.assert_array_equal(_t(T[rows]), To)
    _close(C[rows].cpu().numpy(), Co, 1e-12)

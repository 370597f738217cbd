"""sparse (missing-data) mode through the C ABI against the oracle
(reading A-17 for triples).  Bars: tallies bit-exact, CCC 1e-12 relative (1e-6 fp32),
checksums equal."""
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


def _check(codes, n_stages=1, flags=TAL | F64 | CK, gamma=oracle.GAMMA):
    n_v, n_f = codes.shape
    T, C, cks = ccc.three_way_sparse(codes.cuda(), gamma, flags, n_stages)
    torch.cuda.synchronize()
    To, Co, _ = oracle.sparse_all_triples(codes, gamma)
    if flags & TAL:
        np.testing.assert_array_equal(_t(T), To)
    if flags & F64:
        _ccc_close(C.cpu().numpy(), Co)
    if flags & F32:
        _ccc_close(C.cpu().numpy(), Co, rtol=1e-6)
    if flags & CK:
        got = sum(ccc.checksum_int(c) for c in cks) % (1 << 128)
        assert got == oracle.checksum(3, oracle.triple_list(n_v), To)


@pytest.mark.parametrize("n_v,n_f", [(3, 1), (4, 65), (5, 127), (40, 200), (130, 65), (131, 300),
                                     (260, 129)])
def test_sparse3_full(n_v, n_f):
    _check(synthgen.sparse_codes(n_v, n_f, seed=n_v + n_f))


def test_sparse3_stages_f32_gamma():
    codes = synthgen.sparse_codes(150, 257, seed=31)
    _check(codes, n_stages=3)
    _check(codes, n_stages=7, flags=TAL | F32)
    _check(codes, n_stages=2, flags=F64 | CK, gamma=0.5)


def test_sparse3_degenerate():
    c = synthgen.sparse_codes(60, 200, seed=32)
    c[7, :] = oracle.MISSING              # an all-missing vector: its triples are all zero
    c[20, :100] = oracle.MISSING
    c[21, 100:] = oracle.MISSING          # disjoint present sets: c_ijk = 0 for (20, 21, k)
    _check(c)
    d = synthgen.random_codes(50, 150, seed=33)
    d[d == oracle.MISSING] = 1            # no missing entry: equals the dense mode
    T, C, _ = ccc.three_way_sparse(d.cuda(), out_flags=TAL | F64)
    Td, Cd, _ = ccc.three_way(d.cuda(), out_flags=TAL | F64)
    assert bool((T == Td).all())
    _ccc_close(C.cpu().numpy(), Cd.cpu().numpy(), rtol=1e-13)


def test_sparse3_large_stage_sampled():
    """A 1,024 x 8,192 problem in 4 stages: sampled triples of the first and last stage
    against the brute force, and sum T = 8 c_ijk on every record."""
    n_v, n_f, n_st = 1024, 8192, 4
    codes = synthgen.sparse_codes(n_v, n_f, seed=34, device="cuda")
    ws = ccc.ccc_3way_sparse_prepare(ccc.ccc_pack(codes), n_f)
    rng = np.random.default_rng(5)
    codes_h = codes.cpu()
    for st in (0, n_st - 1):
        T, C, _ = ccc.ccc_3way_sparse_stage(n_v, n_f, n_st, st, ws, TAL | F64)
        torch.cuda.synchronize()
        i0, i1, r0, rc = ccc.ccc_stage_range(n_v, n_st, st)
        tl = []
        for _ in range(600):
            i = int(rng.integers(i0, i1))
            if i > n_v - 3:
                continue
            j = int(rng.integers(i + 1, n_v - 1))
            k = int(rng.integers(j + 1, n_v))
            tl.append((i, j, k))
        tl = sorted(set(tl))
        rows = torch.tensor([ccc.ccc_triple_index(n_v, *t) - r0 for t in tl], device="cuda")
        To, Co, cc = oracle.sparse_triples(codes_h, np.array(tl))
        np.testing.assert_array_equal(_t(T[rows]), To)
        _ccc_close(C[rows].cpu().numpy(), Co)
        sums = T.to(torch.int64).sum(1)
        assert bool((sums % 8 == 0).all())


def test_sparse_hand_values_through_the_kernels():
    """The hand-worked sparse examples (tests/golden/sparse_hand_values.txt) through the
    CUDA path: tallies exact, CCC equal to the exact fractions within 1e-12."""
    from fractions import Fraction
    from conftest import read_golden
    for name, inputs, expected, _ in read_golden("sparse_hand_values.txt"):
        vs = [[int(c) for c in part.split("=")[1].split(",")] for part in inputs.split(";")]
        codes = torch.tensor(vs, dtype=torch.uint8)
        parts = dict(p.strip().split("=") for p in expected.split(";"))
        T_want = [int(x) for x in parts["T"].split(",")]
        C_want = [float(Fraction(x)) for x in parts["C"].split(",")]
        if name == "sparse_pair":
            T, C, _ = ccc.ccc_2way_sparse(ccc.ccc_pack(codes.cuda()), codes.shape[1], out_flags=TAL | F64)
        else:
            T, C, _ = ccc.three_way_sparse(codes.cuda(), out_flags=TAL | F64)
        torch.cuda.synchronize()
        assert list(_t(T)[0]) == T_want
        _ccc_close(C.cpu().numpy()[0], np.array(C_want))


def test_sparse3_bench_shape_sampled():
    """configs[3]'s shape in sparse mode (4,096 x 16,384, 16 stages, bench.py's c4s
    workload): first and last stage, sampled triples including the single-pass kernel's
    tile edges (m at multiples of 64 +- 1, n at multiples of 128 +- 1) against the brute
    force; sum T = 8 c_ijk on every record of both stages."""
    n_v, n_f, n_st = 4096, 16384, 16
    codes = synthgen.sparse_codes(n_v, n_f, seed=4, device="cuda")
    ws = ccc.ccc_3way_sparse_prepare(ccc.ccc_pack(codes), n_f)
    codes_h = codes.cpu()
    rng = np.random.default_rng(9)
    for st in (0, n_st - 1):
        T, C, _ = ccc.ccc_3way_sparse_stage(n_v, n_f, n_st, st, ws, TAL | F64)
        torch.cuda.synchronize()
        i0, i1, r0, rc = ccc.ccc_stage_range(n_v, n_st, st)
        tl = set()
        edges = [e + d for e in range(64, n_v, 64) for d in (-1, 0, 1)]
        while len(tl) < 1500:
            i = int(rng.integers(i0, min(i1, n_v - 2)))
            j = int(rng.choice(edges)) if rng.random() < 0.4 else int(rng.integers(i + 1, n_v - 1))
            if not i < j < n_v - 1:
                continue
            k = int(rng.choice(edges)) if rng.random() < 0.4 else int(rng.integers(j + 1, n_v))
            if j < k < n_v:
                tl.add((i, j, k))
        tl = sorted(tl)
        rows = torch.tensor([ccc.ccc_triple_index(n_v, *t) - r0 for t in tl], device="cuda")
        To, Co, _ = oracle.sparse_triples(codes_h, np.array(tl))
        np.testing.assert_array_equal(_t(T[rows]), To)
        _ccc_close(C[rows].cpu().numpy(), Co)
        assert bool((T.to(torch.int64).sum(1) % 8 == 0).all())

"""Threshold-compacted output ("only those above a certain
threshold") through the C ABI, against the oracle filtered by the same rule: keep a record
iff max over its cells of CCC > theta (reading A-13 / S:524).  Thresholds are placed
midway between two distinct oracle values, so no record sits within rounding of theta."""
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


def _threshold(C, keep_frac):
    """A theta keeping about keep_frac of the records, midway between two distinct maxima."""
    m = np.unique(C.max(1))
    k = min(len(m) - 2, max(0, int(len(m) * (1 - keep_frac))))
    return 0.5 * (m[k] + m[k + 1])


def _rows_of(keys, way, n_v):
    idx = ccc.decode_keys(keys, way).cpu().numpy()
    if way == 2:
        return np.array([ccc.ccc_pair_index(n_v, int(i), int(j)) for i, j in idx], dtype=np.int64)
    return np.array([ccc.ccc_triple_index(n_v, int(i), int(j), int(k)) for i, j, k in idx],
                    dtype=np.int64)


def _check(cm, way, n_v, To, Co, thr, flags, rtol):
    n, keys, T, C = cm.result()
    exp = np.nonzero(Co.max(1) > thr)[0]
    assert n == len(exp)
    rows = _rows_of(keys, way, n_v)
    assert len(np.unique(rows)) == len(rows)
    np.testing.assert_array_equal(np.sort(rows), exp)
    if flags & TAL:
        np.testing.assert_array_equal(_t(T), To[rows])
    if flags & (F64 | F32):
        got, want = C.cpu().numpy().astype(np.float64), Co[rows]
        assert np.all((got == 0) == (want == 0))
        nz = want != 0
        assert np.all(np.abs(got[nz] - want[nz]) <= rtol * np.abs(want[nz]))


@pytest.mark.parametrize("flags,rtol", [(TAL | F64, 1e-12), (TAL | F32, 1e-6), (F64 | CK, 1e-12)])
def test_2way_compact(flags, rtol):
    n_v, n_f = 300, 517
    codes = synthgen.make_codes("hwe", n_v, n_f, 41)
    To, Co = oracle.all_pairs(codes)
    thr = _threshold(Co, 0.03)
    cm = ccc.Compact(thr, len(To), 4, flags)
    _, _, ck = ccc.ccc_2way(ccc.ccc_pack(codes.cuda()), n_f, out_flags=flags, compact=cm)
    _check(cm, 2, n_v, To, Co, thr, flags, rtol)
    if flags & CK:   # the checksum still covers every record
        assert ccc.checksum_int(ck) == oracle.checksum(2, oracle.pair_list(n_v), To)


def test_2way_compact_keep_all_none_and_overflow():
    n_v, n_f = 200, 333
    codes = synthgen.make_codes("random", n_v, n_f, 42)
    To, Co = oracle.all_pairs(codes)
    packed = ccc.ccc_pack(codes.cuda())
    cm = ccc.Compact(-1.0, len(To), 4)                    # every record
    ccc.ccc_2way(packed, n_f, compact=cm)
    _check(cm, 2, n_v, To, Co, -1.0, TAL | F64, 1e-12)
    cm = ccc.Compact(float("inf"), 16, 4)                 # none
    ccc.ccc_2way(packed, n_f, compact=cm)
    assert cm.kept() == 0
    thr = _threshold(Co, 0.2)
    exp = set(np.nonzero(Co.max(1) > thr)[0].tolist())
    cm = ccc.Compact(thr, 50, 4)                          # capacity overflow
    ccc.ccc_2way(packed, n_f, compact=cm)
    n, keys, T, C = cm.result()
    assert n == len(exp) > 50 and len(keys) == 50
    rows = _rows_of(keys, 2, n_v)
    assert set(rows.tolist()) <= exp and len(set(rows.tolist())) == 50
    np.testing.assert_array_equal(_t(T), To[rows])


def test_2way_compact_general_gamma_blocks():
    """gamma != 2/3 and off-diagonal blocks (ccc_2way_block) accumulate into one buffer."""
    n_v, n_f, g = 260, 400, 0.5
    codes = synthgen.make_codes("hwe", n_v, n_f, 43)
    To, Co = oracle.all_pairs(codes, g)
    N, s, w = ccc.ccc_expand(ccc.ccc_pack(codes.cuda()), n_f, g)
    thr = _threshold(Co, 0.05)
    cm = ccc.Compact(thr, len(To), 4)
    h = 130
    ccc.ccc_2way_block(N[:h], s[:h], w[:h], 0, 0, h, N[:h], s[:h], w[:h], 0, True, n_f,
                       TAL | F64, gamma=g, compact=cm)
    ccc.ccc_2way_block(N[h:], s[h:], w[h:], h, 0, n_v - h, N[h:], s[h:], w[h:], h, True, n_f,
                       TAL | F64, gamma=g, compact=cm)
    ccc.ccc_2way_block(N[:h], s[:h], w[:h], 0, 0, h, N[h:], s[h:], w[h:], h, False, n_f,
                       TAL | F64, gamma=g, compact=cm)
    _check(cm, 2, n_v, To, Co, thr, TAL | F64, 1e-12)


@pytest.mark.parametrize("flags,rtol", [(TAL | F64, 1e-12), (TAL | F32, 1e-6)])
def test_3way_compact_stages(flags, rtol):
    n_v, n_f = 140, 301
    codes = synthgen.make_codes("hwe", n_v, n_f, 44)
    To, Co = oracle.all_triples(codes)
    thr = _threshold(Co, 0.02)
    ws = ccc.ccc_3way_prepare(ccc.ccc_pack(codes.cuda()), n_f)
    cm = ccc.Compact(thr, len(To), 8, flags)
    for st in range(3):
        ccc.ccc_3way_stage(n_v, n_f, 3, st, ws, flags, compact=cm)
    _check(cm, 3, n_v, To, Co, thr, flags, rtol)


def test_3way_compact_tetrahedral_units():
    from paper_1705_08213_b200 import decomp
    n_v, n_f, P = 120, 197, 3
    codes = synthgen.make_codes("random", n_v, n_f, 45)
    To, Co = oracle.all_triples(codes)
    thr = _threshold(Co, 0.05)
    N, s, w = ccc.ccc_expand(ccc.ccc_pack(codes.cuda()), n_f)
    G = torch.zeros((n_v, n_v), dtype=torch.int32, device="cuda")
    ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, 0, g=G, ldg=n_v)
    bounds = decomp.block_bounds(n_v, P)
    exp_ = [ccc.ccc_expand(ccc.ccc_pack(codes[lo:hi].contiguous().cuda()), n_f) for lo, hi in bounds]
    blks = [ccc.block(*exp_[b], bounds[b][0]) for b in range(P)]
    cm = ccc.Compact(thr, len(To), 8)
    for r in range(P):
        for u in decomp.plan_3way(P, r, bounds):
            ccc.ccc_3way_unit(blks[u.pb], u.p_lo, u.p_hi, blks[u.mb], u.m_lo, u.m_hi, blks[u.nb],
                              u.n_lo, u.n_hi, u.order, G, n_f, TAL | F64, compact=cm)
    _check(cm, 3, n_v, To, Co, thr, TAL | F64, 1e-12)


def test_3way_compact_C4_stage_full_size():
    """configs[3] size, last stage: the compacted records equal the dense records above
    theta (the dense path is oracle-verified in test_gpu_parity), and every kept record
    matches the brute-force oracle."""
    n_v, n_f, n_st = 4096, 16384, 16
    codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
    ws = ccc.ccc_3way_prepare(ccc.ccc_pack(codes), n_f)
    st = n_st - 1
    _, _, rb, rc = ccc.ccc_stage_range(n_v, n_st, st)
    T, C, _ = ccc.ccc_3way_stage(n_v, n_f, n_st, st, ws, TAL | F64)
    mx = C.max(1).values
    thr = float(torch.quantile(mx[:: max(1, rc // 1_000_000)].float(), 0.99999).item())
    dense = torch.nonzero(mx > thr).flatten()
    cm = ccc.Compact(thr, 1 << 20, 8)
    ccc.ccc_3way_stage(n_v, n_f, n_st, st, ws, TAL | F64, compact=cm)
    n, keys, Tc, Cc = cm.result()
    assert 0 < n == dense.numel() <= (1 << 20)
    idx = ccc.decode_keys(keys, 3)
    i, j, k = idx[:, 0], idx[:, 1], idx[:, 2]
    # lexicographic record index of (i,j,k), minus the stage's first record
    c3 = lambda x: x * (x - 1) * (x - 2) // 6
    c2 = lambda x: x * (x - 1) // 2
    rows = c3(torch.tensor(n_v)) - c3(n_v - i) + c2(n_v - i - 1) - c2(n_v - j) + (k - j - 1) - rb
    order = torch.argsort(rows)
    assert torch.equal(rows[order], dense)
    assert torch.equal(Tc[order], T[dense]) and torch.equal(Cc[order], C[dense])
    sample = idx[: 300].cpu().numpy()
    To, Co = oracle.triples(codes.cpu(), sample)
    np.testing.assert_array_equal(_t(Tc[:300]), To)
    np.testing.assert_allclose(Cc[:300].cpu().numpy(), Co, rtol=1e-12, atol=0)

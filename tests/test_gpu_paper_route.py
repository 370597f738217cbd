"""the paper's 3-way route (Table 1 class masks, three masked pivot
GEMMs, masked marginals, the eight reconstruction equations) on the tensor pipe, against
the oracle and against the product 3-way path.  Bars: tallies bit-exact, CCC 1e-12."""
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


def _run(codes, n_stages, flags, gamma=oracle.GAMMA):
    n_v, n_f = codes.shape
    ws = ccc.ccc_3way_paper_prepare(ccc.ccc_pack(codes.cuda()), n_f, gamma)
    outs = [ccc.ccc_3way_paper_stage(n_v, n_f, n_stages, st, ws, flags, gamma=gamma) for st in range(n_stages)]
    torch.cuda.synchronize()
    T = torch.cat([o[0] for o in outs]) if flags & TAL else None
    C = torch.cat([o[1] for o in outs]) if flags & (F64 | F32) else None
    ck = sum(ccc.checksum_int(o[2]) for o in outs) % (1 << 128) if flags & CK else None
    return T, C, ck


@pytest.mark.parametrize("n_v,n_f", [(3, 1), (4, 65), (5, 127), (40, 200), (130, 65), (131, 300),
                                     (260, 129)])
def test_paper_route_matches_oracle(n_v, n_f):
    codes = synthgen.make_codes("random", n_v, n_f, n_v * 3 + n_f)
    T, C, ck = _run(codes, 1, TAL | F64 | CK)
    To, Co = oracle.all_triples(codes)
    np.testing.assert_array_equal(_t(T), To)
    _ccc_close(C.cpu().numpy(), Co)
    assert ck == oracle.checksum(3, oracle.triple_list(n_v), To)


@pytest.mark.parametrize("kind", ["hwe", "planted"])
def test_paper_route_inputs_stages_gamma(kind):
    codes = synthgen.make_codes(kind, 150, 333, None)
    T, C, _ = _run(codes, 3, TAL | F64, gamma=0.5)
    To, Co = oracle.all_triples(codes, 0.5)
    np.testing.assert_array_equal(_t(T), To)
    _ccc_close(C.cpu().numpy(), Co)


def test_paper_route_equals_product_path():
    """1,024 x 8,192 in 4 stages: tallies identical to ccc_3way_stage's (the Hadamard route)."""
    n_v, n_f, n_st = 1024, 8192, 4
    codes = synthgen.random_codes(n_v, n_f, seed=41, device="cuda")
    packed = ccc.ccc_pack(codes)
    ws_p = ccc.ccc_3way_paper_prepare(packed, n_f)
    ws_h = ccc.ccc_3way_prepare(packed, n_f)
    for st in (0, n_st - 1):
        Tp, _, _ = ccc.ccc_3way_paper_stage(n_v, n_f, n_st, st, ws_p, TAL)
        Th, _, _ = ccc.ccc_3way_stage(n_v, n_f, n_st, st, ws_h, TAL)
        torch.cuda.synchronize()
        assert bool((Tp == Th).all())

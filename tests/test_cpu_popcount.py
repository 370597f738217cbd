"""the optimized bit-packed CPU baseline against the oracle (CPU)."""
import numpy as np
import pytest

import baselines
import oracle
import synthgen


@pytest.mark.parametrize("n_v,n_f", [(2, 1), (3, 31), (5, 32), (7, 33), (65, 63), (66, 64),
                                     (67, 65), (130, 1000), (70, 4111)])
def test_cpu_popcount_matches_oracle(n_v, n_f):
    c = synthgen.make_codes("random", n_v, n_f, n_v + n_f).numpy()
    T, C = baselines.popcount_2way(baselines.pack(c), n_f)
    To, Co = oracle.all_pairs(c, oracle.GAMMA)
    np.testing.assert_array_equal(T.astype(np.int64), To)
    nz = Co != 0
    assert np.all((C == 0) == ~nz)
    assert np.max(np.abs(C[nz] - Co[nz]) / np.abs(Co[nz])) <= 1e-12


@pytest.mark.parametrize("kind", ["hwe", "planted"])
def test_cpu_popcount_inputs_and_row_ranges(kind):
    c = synthgen.make_codes(kind, 150, 500, None).numpy()
    p = baselines.pack(c)
    To, _ = oracle.all_pairs(c, oracle.GAMMA)
    T, _ = baselines.popcount_2way(p, 500, want_ccc=False)
    np.testing.assert_array_equal(T.astype(np.int64), To)
    # a row range produces the contiguous slice of the global record array
    lo, hi = 40, 77
    first = lo * (2 * 150 - lo - 1) // 2
    Ts, _ = baselines.popcount_2way(p, 500, i_lo=lo, i_hi=hi, want_ccc=False)
    np.testing.assert_array_equal(Ts.astype(np.int64), To[first:first + len(Ts)])


def test_pack_layout():
    """The packing written out in baselines.pack is the C ABI layout (include/ccc.h)."""
    c = synthgen.make_codes("random", 3, 70, 1).numpy()
    p = baselines.pack(c)
    assert p.shape == (3, 32)
    for i in range(3):
        for q in range(70):
            assert (p[i, q // 4] >> (2 * (q % 4))) & 3 == c[i, q]
    assert np.all(p[:, 18:] == 0)

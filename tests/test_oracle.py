"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names what fixes the expected value: a value printed in SPEC.md / hand
enumeration of the paper's figure procedure (tests/golden/), a closed form, an
invariant the paper states, exact rational arithmetic, a textbook routine (numpy
integer matmul / einsum) or the paper's own Table-1 route.
"""
from fractions import Fraction
from itertools import combinations, permutations

import numpy as np
import pytest

import oracle
import synthgen
from conftest import read_golden


def _vec(spec):
    """'0*65' / '1,3' / '0*3,3*5' -> list of codes."""
    out = []
    for part in spec.split(","):
        if "*" in part:
            c, n = part.split("*")
            out += [int(c)] * int(n)
        else:
            out.append(int(part))
    return out


def _args(s):
    d = {}
    for kv in s.split(";"):
        k, v = kv.split("=")
        d[k.strip()] = v.strip()
    return d


# ------------------------------------------------------------------ golden values
@pytest.mark.parametrize("row", read_golden("spec_hand_values.txt"))
def test_spec_hand_values(row):
    name, inputs, expected, _cite = row
    if name in ("unique_pairs", "unique_triples"):
        n = int(inputs.split("=")[1])
        lst = oracle.pair_list(n) if name == "unique_pairs" else oracle.triple_list(n)
        assert len(lst) == int(expected)
        if name == "unique_pairs":
            T, _ = oracle.all_pairs(np.zeros((n, 3), np.uint8))
            assert T.size == 4 * int(expected)       # "6 tables, 24 values"
        return
    a = _args(inputs)
    exp = _args(expected) if "=" in expected and ";" in expected else None
    if name == "allele_freq":
        v = _vec(a["v"])
        f = oracle.frequencies(np.array([v], np.uint8))[0]
        assert oracle.freq_exact(v, 1) == Fraction(exp["f1"])
        assert oracle.freq_exact(v, 0) == Fraction(exp["f0"])
        assert f[1] == float(Fraction(exp["f1"])) and f[0] == float(Fraction(exp["f0"]))
        return
    vs = [_vec(a[k]) for k in ("vi", "vj", "vk") if k in a]
    codes = np.array(vs, np.uint8)
    key, val = expected.split("=")
    want = [Fraction(x) for x in val.split(",")]
    if name in ("pair_tally",):
        T, _ = oracle.pairs(codes, [[0, 1]])
        assert list(T[0]) == [int(x) for x in want]
        assert oracle.tally2_py(vs[0], vs[1]) == [int(x) for x in want]
    elif name == "reconstruct3":
        T, _ = oracle.triples(codes, [[0, 1, 2]])
        assert list(T[0]) == [int(x) for x in want]
        assert oracle.tally3_via_table1(*vs) == [int(x) for x in want]
    elif name == "ccc2":
        assert oracle.ccc2_exact(vs[0], vs[1]) == want
        _, C = oracle.pairs(codes, [[0, 1]])
        np.testing.assert_allclose(C[0], [float(x) for x in want], rtol=1e-15)
    elif name == "ccc3":
        assert oracle.ccc3_exact(*vs) == want
        _, C = oracle.triples(codes, [[0, 1, 2]])
        np.testing.assert_allclose(C[0], [float(x) for x in want], rtol=1e-15)
    else:
        raise AssertionError(name)


@pytest.mark.parametrize("row", read_golden("fig_examples_nf1.txt"))
def test_figure_style_examples_nf1(row):
    way, codes, expected, _ = row
    cs = [int(c) for c in codes.split()]
    want = [int(x) for x in expected.split(",")]
    arr = np.array([[c] for c in cs], np.uint8)
    if way == "2":
        assert oracle.tally2_py([cs[0]], [cs[1]]) == want
        assert list(oracle.pairs(arr, [[0, 1]])[0][0]) == want
    else:
        assert oracle.tally3_py([cs[0]], [cs[1]], [cs[2]]) == want
        assert list(oracle.triples(arr, [[0, 1, 2]])[0][0]) == want
        assert oracle.tally3_via_table1([cs[0]], [cs[1]], [cs[2]]) == want


def test_table1_reading_A3():
    """Table 1 as printed agrees with the text rule only with its first two
    columns swapped (reading A-3); the literal header reading contradicts the text."""
    rows = read_golden("table1.txt")
    tup = lambda s: tuple(int(x) for x in s.split(","))
    swapped_ok = literal_ok = True
    for c1, c2, x1, x2, x3 in rows:
        want = [tup(x1), tup(x2), tup(x3)]
        got_swapped = [oracle.x_entry(tup(c2), tup(c1), xi) for xi in (1, 2, 3)]
        got_literal = [oracle.x_entry(tup(c1), tup(c2), xi) for xi in (1, 2, 3)]
        swapped_ok &= got_swapped == want
        literal_ok &= got_literal == want
    assert swapped_ok
    assert not literal_ok


# ------------------------------------------------------------- C vs brute force py
@pytest.mark.parametrize("n_f", [1, 3, 17])
def test_c_oracle_equals_python_enumeration(n_f):
    rng = np.random.default_rng(n_f)
    codes = rng.integers(0, 4, size=(6, n_f), dtype=np.uint8)
    T2, C2 = oracle.all_pairs(codes)
    for r, (i, j) in enumerate(combinations(range(6), 2)):
        assert list(T2[r]) == oracle.tally2_py(codes[i], codes[j])
        ex = oracle.ccc2_exact(codes[i], codes[j])
        np.testing.assert_allclose(C2[r], [float(x) for x in ex], rtol=2e-15, atol=0)
    T3, C3 = oracle.all_triples(codes)
    for r, (i, j, k) in enumerate(combinations(range(6), 3)):
        assert list(T3[r]) == oracle.tally3_py(codes[i], codes[j], codes[k])
        ex = oracle.ccc3_exact(codes[i], codes[j], codes[k])
        np.testing.assert_allclose(C3[r], [float(x) for x in ex], rtol=2e-15, atol=0)
        assert list(T3[r]) == oracle.tally3_via_table1(codes[i], codes[j], codes[k])


def test_literal_req_order_fails():
    """Reading A-2: the printed R-eqs with the first slot as the i-allele (Eq.5 order)
    disagree with the brute force; with the first slot as the pivot allele they agree."""
    rng = np.random.default_rng(5)
    c = rng.integers(0, 4, size=(3, 40), dtype=np.uint8)
    B = [oracle.masked_tally(c[1], c[0], c[2], xi) for xi in (1, 2, 3)]
    literal = [0] * 8
    for x in (0, 1):
        for y in (0, 1):
            for z in (0, 1):
                Bx = B[0] if x == 0 else B[2]
                literal[4 * x + 2 * y + z] = 2 * Bx[2 * y + z] + B[1][2 * y + z]
    truth = oracle.tally3_py(c[0], c[1], c[2])
    assert oracle.reconstruct3(*B) == truth
    assert literal != truth


# ------------------------------------------------------- textbook-routine identities
def _counts(codes):
    """allele-1 count n_{iq} = rho_{i,q}(1) by direct decode (not via the oracle)."""
    return ((codes >> 1) & 1).astype(np.int64) + (codes & 1).astype(np.int64)


@pytest.mark.parametrize("shape", [(9, 130), (23, 257)])
def test_pairs_equal_integer_matmul(shape):
    """T(a,b) = R_a R_b^T with R_1 = N, R_0 = 2 - N (numpy integer matmul)."""
    codes = synthgen.random_codes(*shape, seed=11).numpy()
    N = _counts(codes)
    R = {1: N, 0: 2 - N}
    T, _ = oracle.all_pairs(codes)
    iu = np.triu_indices(shape[0], 1)
    for a in (0, 1):
        for b in (0, 1):
            G = R[a] @ R[b].T
            np.testing.assert_array_equal(T[:, 2 * a + b], G[iu])


def test_triples_equal_einsum():
    codes = synthgen.hwe_codes(8, 77, seed=4).numpy()
    N = _counts(codes)
    R = {1: N, 0: 2 - N}
    T, _ = oracle.all_triples(codes)
    tl = oracle.triple_list(8)
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                G3 = np.einsum("iq,jq,kq->ijk", R[a], R[b], R[c])
                np.testing.assert_array_equal(T[:, 4 * a + 2 * b + c],
                                              G3[tl[:, 0], tl[:, 1], tl[:, 2]])


# ---------------------------------------------------------------- invariants
def test_invariants_random():
    codes = synthgen.random_codes(10, 101, seed=7).numpy()
    n_f = codes.shape[1]
    S = oracle.allele_sums(codes)
    assert np.all(S.sum(1) == 2 * n_f)                       # f_i(0)+f_i(1) = 1
    T2, C2 = oracle.all_pairs(codes)
    assert np.all(T2.sum(1) == 4 * n_f)                      # sum f_ij = 1
    assert np.all(T2 >= 0) and np.all(C2 >= 0)
    T3, _ = oracle.all_triples(codes)
    assert np.all(T3.sum(1) == 8 * n_f)
    # marginalisation: sum_b T3(a,b,c) = 2 T2_ik(a,c)   (rho_j(0)+rho_j(1) = 2)
    pidx = {tuple(p): r for r, p in enumerate(oracle.pair_list(10))}
    for r, (i, j, k) in enumerate(oracle.triple_list(10)):
        t2 = T2[pidx[(i, k)]]
        for a in (0, 1):
            for c in (0, 1):
                assert T3[r, 4 * a + c] + T3[r, 4 * a + 2 + c] == 2 * t2[2 * a + c]


def test_permutation_symmetry():
    """f_ij symmetric; f_ijk symmetric in i,j,k."""
    codes = synthgen.random_codes(5, 64, seed=9).numpy()
    T, C = oracle.pairs(codes, [[1, 3], [3, 1]])
    assert [T[0][0], T[0][1], T[0][2], T[0][3]] == [T[1][0], T[1][2], T[1][1], T[1][3]]
    np.testing.assert_allclose(C[0][[0, 1, 2, 3]], C[1][[0, 2, 1, 3]], rtol=1e-15)
    base = (0, 2, 4)
    T0, C0 = oracle.triples(codes, [base])
    for p in permutations(range(3)):
        idx = [base[p[0]], base[p[1]], base[p[2]]]
        Tp, Cp = oracle.triples(codes, [idx])
        for a in (0, 1):
            for b in (0, 1):
                for c in (0, 1):
                    abc = (a, b, c)
                    q = [abc[p[0]], abc[p[1]], abc[p[2]]]
                    assert T0[0][4 * a + 2 * b + c] == Tp[0][4 * q[0] + 2 * q[1] + q[2]]


def test_closed_forms_ccc():
    n_f = 9
    het = np.ones((3, n_f), np.uint8)
    _, C = oracle.pairs(het, [[0, 1]])
    np.testing.assert_allclose(C[0], [1 / 9] * 4, rtol=1e-15)
    _, C = oracle.triples(het, [[0, 1, 2]])
    np.testing.assert_allclose(C[0], [1 / 27] * 8, rtol=1e-15)
    codes = synthgen.random_codes(4, 33, seed=3).numpy()
    _, C = oracle.all_pairs(codes, gamma=0.0)
    np.testing.assert_allclose(C.sum(1), 1.0, rtol=1e-15)    # gamma=0 -> sum CCC = 1
    _, C = oracle.all_triples(codes, gamma=0.0)
    np.testing.assert_allclose(C.sum(1), 1.0, rtol=1e-15)
    vi, vj = codes[0], codes[1]
    assert sum(oracle.ccc2_exact(vi, vj, gamma=Fraction(0))) == 1


def test_planted_closed_form():
    codes, L, H, _ = synthgen.planted_codes(12, 97, seed=3)
    codes = codes.numpy()
    T2, _ = oracle.all_pairs(codes)
    for r, (i, j) in enumerate(oracle.pair_list(12)):
        assert list(T2[r]) == oracle.planted_tally2(L, H, 97, i, j)
    T3, _ = oracle.all_triples(codes[:7])
    for r, (i, j, k) in enumerate(oracle.triple_list(7)):
        assert list(T3[r]) == oracle.planted_tally3(L, H, 97, i, j, k)


def _planted_by_hand(L, H, n_f, seed):
    """Planted codes built here from (L, H) without synthgen: (1,1) on [0, L), the two
    heterozygote codes alternating on [L, L+H), (0,0) after, then a shared column shuffle."""
    rng = np.random.default_rng(seed)
    codes = np.zeros((len(L), n_f), np.uint8)
    for i, (l, h) in enumerate(zip(L, H)):
        codes[i, :l] = 3
        codes[i, l:l + h] = rng.choice([1, 2], size=h)
    return codes[:, rng.permutation(n_f)]


@pytest.mark.parametrize("n_v,n_f,seed", [(40, 7, 1), (33, 64, 2), (25, 301, 3), (12, 1, 4)])
def test_planted_closed_form_c_vs_brute_force(n_v, n_f, seed):
    """The C closed form of the planted design (oracle_planted_*) equals the
    Fig.1 / Fig.2 brute force record for record -- tallies and fp64 CCC bit-identical --
    including the edge intervals L = 0, H = 0, L + H = n_f."""
    rng = np.random.default_rng(seed)
    L = rng.integers(0, n_f + 1, n_v)
    H = np.array([rng.integers(0, n_f - l + 1) for l in L])
    L[:4] = [0, n_f, 0, n_f // 2]
    H[:4] = [0, 0, n_f, n_f - n_f // 2]
    codes = _planted_by_hand(L, H, n_f, seed)
    T, C = oracle.all_pairs(codes)
    Tp, Cp = oracle.planted_pairs(L, H, n_f)
    np.testing.assert_array_equal(Tp, T)
    np.testing.assert_array_equal(Cp, C)
    T3, C3 = oracle.all_triples(codes[:20])
    Tp3, Cp3 = oracle.planted_triples(L[:20], H[:20], n_f)
    np.testing.assert_array_equal(Tp3, T3)
    np.testing.assert_array_equal(Cp3, C3)
    np.testing.assert_array_equal(oracle.planted_sums(L, H, n_f), oracle.allele_sums(codes))
    for g in (0.0, 0.5):
        np.testing.assert_array_equal(oracle.planted_pairs(L, H, n_f, gamma=g)[1],
                                      oracle.all_pairs(codes, g)[1])


def test_planted_closed_form_c_vs_python_intervals():
    """...and the Python interval form (planted_tally2/3) on synthgen's planted data."""
    n_v, n_f = 30, 1001
    L, H = synthgen.planted_lengths(n_v, n_f, 3)
    Tp, _ = oracle.planted_pairs(L, H, n_f)
    for r, (i, j) in enumerate(oracle.pair_list(n_v)):
        assert list(Tp[r]) == oracle.planted_tally2(L, H, n_f, i, j)
    Tp3, _ = oracle.planted_triples(L, H, n_f, 50, 400)
    for r, (i, j, k) in enumerate(oracle.triple_list(n_v)[50:450]):
        assert list(Tp3[r]) == oracle.planted_tally3(L, H, n_f, i, j, k)


@pytest.mark.parametrize("way", [2, 3])
def test_planted_checker_catches_errors(way):
    """The full-size checker (oracle_planted_check2/3) passes the closed-form records at
    rtol = 0 (the hoisted 3-way evaluation is bit-identical), on any sub-range, and flags a
    tally off by one, a CCC cell off by 1e-11 relative, a nonzero CCC where the tally is 0,
    a NaN, fp32 beyond 1e-6 and records shifted by one position."""
    n_v, n_f = 45, 333
    L, H = synthgen.planted_lengths(n_v, n_f, 3)
    T, C = (oracle.planted_pairs if way == 2 else oracle.planted_triples)(L, H, n_f)
    T = T.astype(np.uint32)
    m = len(T)
    chk = lambda rec0, t, c, **kw: oracle.planted_check(way, L, H, n_f, rec0, len(t if t is not None else c), t, c, **kw)  # noqa: E731
    assert chk(0, T, C, rtol=0) == {"bad_tallies": 0, "bad_ccc": 0, "first_bad": -1, "max_rel": 0.0}
    assert chk(m // 3, T[m // 3: m // 2], C[m // 3: m // 2], rtol=0)["first_bad"] == -1
    assert chk(0, T, C.astype(np.float32), rtol=1e-6)["bad_ccc"] == 0
    assert chk(0, T, C.astype(np.float32), rtol=1e-9)["bad_ccc"] > 0
    bad = T.copy()
    bad[m // 2, 1] += 1
    r = chk(0, bad, C)
    assert (r["bad_tallies"], r["bad_ccc"], r["first_bad"]) == (1, 0, m // 2)
    for r0, val in ((7, None), (m - 1, np.nan)):
        Cb = C.copy()
        nzc = np.flatnonzero(Cb[r0])[0]
        Cb[r0, nzc] = Cb[r0, nzc] * (1 + 1e-11) if val is None else val
        r = chk(0, T, Cb)
        assert (r["bad_tallies"], r["bad_ccc"], r["first_bad"]) == (0, 1, r0)
    zr, zc = np.argwhere(T == 0)[0]
    Cb = C.copy()
    Cb[zr, zc] = 1e-300
    assert chk(0, T, Cb)["bad_ccc"] == 1
    r = chk(1, T[:-1], C[:-1])
    assert r["bad_tallies"] > m // 2 and r["first_bad"] == 0
    assert chk(0, T, None)["bad_ccc"] == 0 and chk(0, None, C)["bad_tallies"] == 0


def test_padding_independence():
    """Results are over exactly n_f fields (A-9): appending fields changes sums by the
    appended contribution only; n_f=65 all-(0,0) gives 260 (not 4*128)."""
    z = np.zeros((2, 65), np.uint8)
    assert list(oracle.pairs(z, [[0, 1]])[0][0]) == [260, 0, 0, 0]


# ----------------------------------------------------------------- checksum
def test_checksum_properties():
    codes = synthgen.random_codes(9, 40, seed=2).numpy()
    T, _ = oracle.all_pairs(codes)
    idx = oracle.pair_list(9)
    full = oracle.checksum(2, idx, T)
    assert full == oracle.checksum_scalar(2, idx, T)
    T3, _ = oracle.all_triples(codes[:7])
    tl = oracle.triple_list(7)
    assert oracle.checksum(3, tl, T3) == oracle.checksum_scalar(3, tl, T3)
    assert oracle.checksum(2, idx[:0], T[:0]) == 0
    perm = np.random.default_rng(1).permutation(len(idx))
    assert oracle.checksum(2, idx[perm], T[perm]) == full
    part = (oracle.checksum(2, idx[:10], T[:10]) + oracle.checksum(2, idx[10:], T[10:])) % (1 << 128)
    assert part == full
    # a single flipped tally changes it
    T2 = T.copy()
    T2[5, 1] += 1
    assert oracle.checksum(2, idx, T2) != full
    # distinct single-record digests on a sample
    digs = {oracle.record_digest(2, idx[r], T[r]) for r in range(len(idx))}
    assert len(digs) == len(idx)
    assert oracle.fmix64(0) == 0 and oracle.fmix64(1) != 1


# ----------------------------------------------------------------- synthgen pins
def test_synthgen_scalar_vs_tensor_and_tiling():
    t = synthgen.random_codes(5, 70, seed=7)
    for i in range(5):
        for q in (0, 1, 57, 69):
            assert int(t[i, q]) == synthgen.code_scalar(7, i, q)
    tail = synthgen.random_codes(3, 70, seed=7, row0=2)
    assert np.array_equal(t[2:].numpy(), tail.numpy())
    assert not np.array_equal(t.numpy(), synthgen.random_codes(5, 70, seed=8).numpy())
    big = synthgen.random_codes(64, 4096, seed=1).numpy()
    freq = np.bincount(big.ravel(), minlength=4) / big.size
    assert np.all(np.abs(freq - 0.25) < 0.01)


# ------------------------------------------------------------ sparse mode (f1, A-17)
def test_sparse_no_missing_equals_dense():
    """with no missing entry the sparse tally equals the dense one, c_ij = n_f
    (and so does CCC: every divisor reduces to n_f)."""
    c = synthgen.random_codes(12, 77, seed=9).numpy()
    c[c == oracle.MISSING] = 1                      # (1,0) -> (0,1): same heterozygote
    Ts, Cs, cij = oracle.sparse_all_pairs(c)
    Td, Cd = oracle.all_pairs(c)
    np.testing.assert_array_equal(Ts, Td)
    np.testing.assert_allclose(Cs, Cd, rtol=1e-15, atol=0)
    assert np.all(cij == 77)


def test_sparse_all_missing_vector():
    """a vector with every entry missing has zero tallies, count 0, CCC 0."""
    c = synthgen.sparse_codes(6, 50, seed=10).numpy()
    c[2, :] = oracle.MISSING
    T, C, cij = oracle.sparse_all_pairs(c)
    for r, (i, j) in enumerate(oracle.pair_list(6)):
        if 2 in (i, j):
            assert cij[r] == 0 and not T[r].any() and not C[r].any()
    S, cnt = oracle.sparse_sums(c)
    assert cnt[2] == 0 and not S[2].any()


def test_sparse_equals_dense_on_present_columns():
    """Independent pin (column deletion): T_ij over the fields where both entries are
    present is the DENSE tally of the two vectors restricted to those fields; c_ij is
    that field count; the per-vector frequencies are the dense frequencies of the vector
    with its missing entries deleted."""
    c = synthgen.sparse_codes(9, 240, seed=11).numpy()
    T, C, cij = oracle.sparse_all_pairs(c)
    S, cnt = oracle.sparse_sums(c)
    for i in range(9):
        keep = c[i] != oracle.MISSING
        assert cnt[i] == keep.sum()
        if keep.any():
            np.testing.assert_array_equal(S[i], oracle.allele_sums(c[i:i + 1, keep])[0])
    for r, (i, j) in enumerate(oracle.pair_list(9)):
        keep = (c[i] != oracle.MISSING) & (c[j] != oracle.MISSING)
        assert cij[r] == keep.sum() and T[r].sum() == 4 * cij[r]
        Td, _ = oracle.pairs(c[[i, j]][:, keep], [[0, 1]])
        np.testing.assert_array_equal(T[r], Td[0])


def test_sparse_ccc_exact_rational():
    """CCC in fp64 against exact rationals built from the column-deleted dense pieces."""
    c = synthgen.sparse_codes(5, 31, seed=12).numpy()
    T, C, cij = oracle.sparse_all_pairs(c)
    g = Fraction(2, 3)
    for r, (i, j) in enumerate(oracle.pair_list(5)):
        fi = [Fraction(int(x), 2 * int((c[i] != 2).sum())) for x in oracle.sparse_sums(c)[0][i]]
        fj = [Fraction(int(x), 2 * int((c[j] != 2).sum())) for x in oracle.sparse_sums(c)[0][j]]
        for a in range(2):
            for b in range(2):
                exact = Fraction(int(T[r, 2 * a + b]), 4 * int(cij[r])) * (1 - g * fi[a]) * (1 - g * fj[b])
                assert abs(C[r, 2 * a + b] - float(exact)) <= 2e-15 * float(exact) + 1e-300


def test_sparse_codes_generator():
    c = synthgen.sparse_codes(64, 2000, seed=4).numpy()
    frac = (c == 2).mean(1)
    assert frac.max() < 0.35 and frac.min() >= 0.0 and frac.mean() > 0.05
    np.testing.assert_array_equal(synthgen.sparse_codes(8, 100, seed=4, row0=5).numpy(),
                                  synthgen.sparse_codes(13, 100, seed=4).numpy()[5:])


# ------------------------------------------------------------- sparse 3-way (A-17 for triples)
def test_sparse3_no_missing_equals_dense():
    """With no missing entry the sparse 3-way tally / CCC equal the dense ones, c_ijk = n_f."""
    c = synthgen.random_codes(9, 53, seed=21).numpy()
    c[c == oracle.MISSING] = 1
    Ts, Cs, cc = oracle.sparse_all_triples(c)
    Td, Cd = oracle.all_triples(c)
    np.testing.assert_array_equal(Ts, Td)
    np.testing.assert_allclose(Cs, Cd, rtol=1e-15, atol=0)
    assert np.all(cc == 53)


def test_sparse3_column_deletion_and_marginals():
    """Independent pins: T_ijk over the fields where all three are present is the DENSE
    3-way tally of the three vectors restricted to those fields; sum T = 8 c_ijk; summing
    out the k allele gives 2 x the sparse pair tally over the same fields; a vector with
    every entry missing zeroes all its triples."""
    c = synthgen.sparse_codes(8, 180, seed=22).numpy()
    c[5, :] = oracle.MISSING
    T, C, cc = oracle.sparse_all_triples(c)
    for r, (i, j, k) in enumerate(oracle.triple_list(8)):
        keep = (c[i] != oracle.MISSING) & (c[j] != oracle.MISSING) & (c[k] != oracle.MISSING)
        assert cc[r] == keep.sum() and T[r].sum() == 8 * cc[r]
        if 5 in (i, j, k):
            assert cc[r] == 0 and not T[r].any() and not C[r].any()
            continue
        Td, _ = oracle.triples(c[[i, j, k]][:, keep], [[0, 1, 2]])
        np.testing.assert_array_equal(T[r], Td[0])
        T2, _ = oracle.pairs(c[[i, j]][:, keep], [[0, 1]])
        np.testing.assert_array_equal(T[r].reshape(2, 2, 2).sum(2), 2 * T2[0].reshape(2, 2))


def test_sparse3_ccc_exact_rational():
    """3-way sparse CCC in fp64 against exact rationals (per-vector f over present entries,
    per-triple divisor 8 c_ijk)."""
    c = synthgen.sparse_codes(5, 37, seed=23).numpy()
    T, C, cc = oracle.sparse_all_triples(c)
    g = Fraction(2, 3)
    S, cnt = oracle.sparse_sums(c)
    for r, (i, j, k) in enumerate(oracle.triple_list(5)):
        fs = [[Fraction(int(S[x, a]), 2 * int(cnt[x])) for a in range(2)] for x in (i, j, k)]
        for a in range(2):
            for b in range(2):
                for d in range(2):
                    exact = (Fraction(int(T[r, 4 * a + 2 * b + d]), 8 * int(cc[r])) * (1 - g * fs[0][a]) *
                             (1 - g * fs[1][b]) * (1 - g * fs[2][d]))
                    assert abs(C[r, 4 * a + 2 * b + d] - float(exact)) <= 4e-15 * float(exact) + 1e-300


@pytest.mark.parametrize("row", read_golden("sparse_hand_values.txt"))
def test_sparse_hand_values(row):
    """Sparse mode worked by hand (tests/golden/sparse_hand_values.txt, reading A-17)."""
    name, inputs, expected, _ = row
    a = _args(inputs)
    vs = [_vec(a[k]) for k in ("vi", "vj", "vk") if k in a]
    codes = np.array(vs, np.uint8)
    parts = dict(p.split("=") for p in (x.strip() for x in expected.split(";")))
    T_want = [int(x) for x in parts["T"].split(",")]
    C_want = [Fraction(x) for x in parts["C"].split(",")]
    if name == "sparse_pair":
        T, C, c = oracle.sparse_pairs(codes, [[0, 1]])
    else:
        T, C, c = oracle.sparse_triples(codes, [[0, 1, 2]])
    assert list(T[0]) == T_want and int(c[0]) == int(parts["c"])
    for got, want in zip(C[0], C_want):
        assert abs(got - float(want)) <= 1e-15 * float(want) + (0.0 if want else 0.0)
        assert (got == 0) == (want == 0)

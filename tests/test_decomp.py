"""Exact-cover enumeration of the multi-GPU schedules (CPU only): every unique pair / triple
is produced by exactly one rank, per-rank loads are balanced, and record counts match
(SURVEY §4 "exact-cover enumeration")."""
from collections import Counter
from itertools import combinations

import pytest

from paper_1705_08213_b200 import decomp


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("n_v", [8, 37, 64])
def test_2way_exact_cover_and_balance(P, n_v):
    if n_v < P:
        pytest.skip("fewer vectors than ranks")
    bounds = decomp.block_bounds(n_v, P)
    seen = Counter()
    per_rank = []
    for r in range(P):
        cnt = 0
        for u in decomp.plan_2way(P, r, bounds):
            assert u.step <= decomp.ring_steps_2way(P)
            assert r in (u.a, u.b)                       # a rank only uses its own block + ring
            pairs = list(decomp.unit2_pairs(u, bounds))
            assert len(pairs) == decomp.unit2_records(u, bounds)
            for i, j in pairs:
                assert i < j
                seen[(i, j)] += 1
            cnt += len(pairs)
        per_rank.append(cnt)
    assert set(seen) == set(combinations(range(n_v), 2))
    assert max(seen.values()) == 1
    if n_v % P == 0 and (n_v // P) % 2 == 0:
        assert max(per_rank) == min(per_rank)           # equal loads with the antipodal split


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("n_v", [12, 24])
def test_3way_exact_cover_and_balance(P, n_v):
    bounds = decomp.block_bounds(n_v, P)
    if min(hi - lo for lo, hi in bounds) < 1:
        pytest.skip("empty block")
    seen = Counter()
    per_rank = []
    for r in range(P):
        cnt = 0
        for u in decomp.plan_3way(P, r, bounds):
            assert u.pb == r                            # pivot always from the own block
            tr = list(decomp.unit3_triples(u, bounds))
            assert len(tr) == decomp.unit3_count(u, bounds)
            for t in tr:
                seen[t] += 1
            cnt += len(tr)
        per_rank.append(cnt)
    assert set(seen) == set(combinations(range(n_v), 3))
    assert max(seen.values()) == 1
    assert decomp.total_triples(P, bounds) == len(seen)


def test_3way_balance_large_blocks():
    """Per-rank triple counts are within 1% of n_v^3/(6P) at realistic sizes (closed form)."""
    n_v = 16384
    for P in (2, 4, 8):
        bounds = decomp.block_bounds(n_v, P)
        loads = [sum(decomp.unit3_count(u, bounds) for u in decomp.plan_3way(P, r, bounds))
                 for r in range(P)]
        assert sum(loads) == n_v * (n_v - 1) * (n_v - 2) // 6
        assert max(loads) / min(loads) < 1.01


def test_block_bounds_alignment():
    b = decomp.block_bounds(56568, 8, align=256)
    assert b[0][0] == 0 and b[-1][1] == 56568
    assert all(lo % 256 == 0 for lo, _ in b)
    assert all(hi > lo for lo, hi in b)


def test_unit3_count_pivot_subranges():
    bounds = decomp.block_bounds(30, 3)
    for r in range(3):
        for u in decomp.plan_3way(3, r, bounds):
            for lo in range(u.p_lo, u.p_hi):
                for hi in range(lo, u.p_hi + 1):
                    sub = decomp.Unit3(u.pb, lo, hi, u.mb, u.m_lo, u.m_hi, u.nb, u.n_lo, u.n_hi, u.order)
                    assert decomp.unit3_count(sub, bounds) == len(list(decomp.unit3_triples(sub, bounds)))

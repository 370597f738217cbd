"""Multi-GPU decompositions of the unique-result space (§4).

Pure host logic (no torch, no CUDA): which rank computes which block of pairs / triples,
and which vector blocks it needs.  Vectors are split into P contiguous blocks; rank r owns
block r (the paper's n_pv axis).

2-way, block-circulant: rank r computes the diagonal block (r, r) and the
off-diagonal blocks (r, r+d mod P) for d = 1 .. ceil(P/2)-1.  For even P the antipodal
block pair {r, r+P/2} is split by rows of its lower-index block between its two owners, so
every rank has exactly the same number of pairs (the paper's rule, where ranks below P/2
own the whole antipodal block, leaves P=8 at 4.5 vs 3.5 block units; R-12).
The blocks a rank needs arrive by a ring shift (step d: block (r+d) mod P), so ceil(P/2)
... floor(P/2) ring steps are needed.

3-way, tetrahedral (the paper's exact slice rule is in an absent companion
paper, A-16): with the pivot always taken from the rank's own block,
  {A,A,A}                       -> owner of A
  {D,D,S}, D != S               -> owner of D
  {A<B<C} distinct blocks       -> split in three GEMM-shaped parts:
        owner(B): pivot y in B[0, 1/3),  x in A,        z in C
        owner(A): pivot x in A[0, 1/2),  y in B[1/3,1), z in C
        owner(C): pivot z in C,          x in A[1/2,1), y in B[1/3,1)
Exact cover and equal per-rank triple counts are checked by enumeration in
tests/test_decomp.py.  Each rank needs every block (a ring all-gather with retention).
"""
from __future__ import annotations

from dataclasses import dataclass
from math import comb


def block_bounds(n_v: int, P: int, align: int = 1):
    """Contiguous blocks [lo, hi) of the vector axis; block sizes differ by < align."""
    if P < 1:
        raise ValueError("P >= 1")
    units = -(-n_v // align)
    out = []
    for r in range(P):
        lo = (r * units // P) * align
        hi = ((r + 1) * units // P) * align
        out.append((min(lo, n_v), min(hi, n_v)))
    return out


# --------------------------------------------------------------------------- 2-way
@dataclass(frozen=True)
class Unit2:
    """One 2-way work unit: rows [a_lo, a_hi) (local to block a) x all rows of block b.
    diag: a == b and only local pairs i < j; else every (i, j), block a has the lower
    global indices.  step: ring step at which block `other` is resident on the rank."""
    a: int
    b: int
    a_lo: int
    a_hi: int
    diag: bool
    step: int


def plan_2way(P: int, rank: int, bounds) -> list[Unit2]:
    units = []
    n_r = bounds[rank][1] - bounds[rank][0]
    units.append(Unit2(rank, rank, 0, n_r, True, 0))
    for d in range(1, P // 2 + 1):
        other = (rank + d) % P
        lo_blk, hi_blk = (rank, other) if rank < other else (other, rank)
        n_lo = bounds[lo_blk][1] - bounds[lo_blk][0]
        if 2 * d < P:
            units.append(Unit2(lo_blk, hi_blk, 0, n_lo, False, d))
        elif 2 * d == P:                      # antipodal block, split by rows of lo_blk
            half = n_lo // 2
            if rank == lo_blk:
                units.append(Unit2(lo_blk, hi_blk, 0, half, False, d))
            else:
                units.append(Unit2(lo_blk, hi_blk, half, n_lo, False, d))
    return units


def ring_steps_2way(P: int) -> int:
    return P // 2


def unit2_records(u: Unit2, bounds) -> int:
    n_b = bounds[u.b][1] - bounds[u.b][0]
    if u.diag:
        return sum(n_b - 1 - i for i in range(u.a_lo, u.a_hi))
    return (u.a_hi - u.a_lo) * n_b


def unit2_pairs(u: Unit2, bounds):
    """Global (i, j) pairs of a unit in its record order (for tests)."""
    a0, b0 = bounds[u.a][0], bounds[u.b][0]
    n_b = bounds[u.b][1] - b0
    for il in range(u.a_lo, u.a_hi):
        for jl in range(il + 1 if u.diag else 0, n_b):
            yield (a0 + il, b0 + jl)


# ------------------------------------------------------- 2-way process grid (n_pv x n_pr x n_pf)
@dataclass(frozen=True)
class Grid:
    """The paper's process grid for the 2-way method: n_pv vector
    blocks (block-circulant ring), n_pr parts of every block row's result (the "n_pr axis
    ... parallelize the computation of the blocks of this block row"), n_pf field slices
    (a reduction of partial tallies follows the GEMM).  rank = (v n_pr + r) n_pf + f."""
    n_pv: int
    n_pr: int = 1
    n_pf: int = 1

    @property
    def world(self) -> int:
        return self.n_pv * self.n_pr * self.n_pf

    def coords(self, rank: int):
        if not 0 <= rank < self.world:
            raise ValueError("rank outside the grid")
        return rank // (self.n_pr * self.n_pf), (rank // self.n_pf) % self.n_pr, rank % self.n_pf

    def rank(self, v: int, r: int, f: int) -> int:
        return (v * self.n_pr + r) * self.n_pf + f

    def ring_ranks(self, r: int, f: int):
        """Global ranks of the vector-block ring that rank (., r, f) belongs to, by v."""
        return [self.rank(v, r, f) for v in range(self.n_pv)]

    def field_ranks(self, v: int, r: int):
        """Global ranks sharing block row v's part r over the n_pf field slices, by f."""
        return [self.rank(v, r, f) for f in range(self.n_pf)]


def split_rows(u: Unit2, bounds, parts: int):
    """The n_pr split of a unit: `parts` contiguous row ranges of [u.a_lo, u.a_hi) with
    record counts as equal as whole rows allow (some may be empty)."""
    n_b = bounds[u.b][1] - bounds[u.b][0]
    rows = list(range(u.a_lo, u.a_hi))
    cum = [0]
    for i in rows:
        cum.append(cum[-1] + ((n_b - 1 - i) if u.diag else n_b))
    tot = cum[-1]
    cuts = [u.a_lo]
    k = 0
    for p in range(1, parts):
        target = p * tot / parts
        while k < len(rows) and cum[k] < target:
            k += 1
        cuts.append(max(cuts[-1], u.a_lo + k))
    cuts.append(u.a_hi)
    return [(cuts[p], cuts[p + 1]) for p in range(parts)]


# --------------------------------------------------------------------------- 3-way
@dataclass(frozen=True)
class Unit3:
    """One 3-way work unit: pivot p over rows [p_lo, p_hi) of block pb (own block), m over
    rows [m_lo, m_hi) of block mb, n over rows [n_lo, n_hi) of block nb.  `order` maps the
    roles (p, m, n) to the canonical sorted slots: canonical triple = sorted indices and
    order[s] is the role in slot s.  Constraints: if two roles share a block the unit only
    contains index orders consistent with `order` (strict inequalities)."""
    pb: int
    p_lo: int
    p_hi: int
    mb: int
    m_lo: int
    m_hi: int
    nb: int
    n_lo: int
    n_hi: int
    order: tuple


def plan_3way(P: int, rank: int, bounds) -> list[Unit3]:
    def n(b):
        return bounds[b][1] - bounds[b][0]

    units = []
    r = rank
    # {A,A,A}
    units.append(Unit3(r, 0, n(r), r, 0, n(r), r, 0, n(r), ("p", "m", "n")))
    for s in range(P):
        if s == r:
            continue
        # {D,D,S} with D = r: pivot x < y both in D, z in S
        if s > r:   # canonical (x, y, z)
            units.append(Unit3(r, 0, n(r), r, 0, n(r), s, 0, n(s), ("p", "m", "n")))
        else:       # canonical (z, x, y)
            units.append(Unit3(r, 0, n(r), r, 0, n(r), s, 0, n(s), ("n", "p", "m")))
    for a in range(P):
        for b in range(a + 1, P):
            for c in range(b + 1, P):
                if r not in (a, b, c):
                    continue
                na, nbb, nc = n(a), n(b), n(c)
                b3 = nbb // 3
                a2 = na // 2
                if r == b:
                    units.append(Unit3(b, 0, b3, a, 0, na, c, 0, nc, ("m", "p", "n")))
                if r == a:
                    units.append(Unit3(a, 0, a2, b, b3, nbb, c, 0, nc, ("p", "m", "n")))
                if r == c:
                    units.append(Unit3(c, 0, nc, a, a2, na, b, b3, nbb, ("m", "n", "p")))
    return units


def unit3_triples(u: Unit3, bounds):
    """Canonical global (i<j<k) triples a unit produces (for tests / counting)."""
    p0, m0, n0 = bounds[u.pb][0], bounds[u.mb][0], bounds[u.nb][0]
    for p in range(p0 + u.p_lo, p0 + u.p_hi):
        for m in range(m0 + u.m_lo, m0 + u.m_hi):
            for nn in range(n0 + u.n_lo, n0 + u.n_hi):
                role = {"p": p, "m": m, "n": nn}
                t = tuple(role[x] for x in u.order)
                if t[0] < t[1] < t[2]:
                    yield t


def unit3_count(u: Unit3, bounds) -> int:
    """Number of canonical triples of a unit (closed form per case; the pivot range may be
    a sub-range -- a stage -- while same-block row / column ranges are whole blocks)."""
    np_, nm, nn = u.p_hi - u.p_lo, u.m_hi - u.m_lo, u.n_hi - u.n_lo
    nb = bounds[u.pb][1] - bounds[u.pb][0]
    if u.pb == u.mb and u.mb == u.nb:          # sum_p C(nb-1-p, 2)
        return comb(nb - u.p_lo, 3) - comb(nb - u.p_hi, 3)
    if u.pb == u.mb:                           # sum_p (nb-1-p) * |N|
        rs = lambda i: i * (2 * nb - i - 1) // 2
        return (rs(u.p_hi) - rs(u.p_lo)) * nn
    return np_ * nm * nn


def total_triples(P: int, bounds) -> int:
    return sum(unit3_count(u, bounds) for r in range(P) for u in plan_3way(P, r, bounds))

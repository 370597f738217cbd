"""Seeded synthetic genotype generators shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the CCC method (no allele counts, no tallies,
no frequencies). It only produces 2-bit genotype codes, deterministically, as a
pure function of (seed, vector index i, field index q) so that any tiling, rank
decomposition or device reproduces identical inputs (§5, P:653-656:
"exact same bit-for-bit result for all code versions and for all parallel
decompositions"; SPEC.md bitgrid.generate_random).

Code convention (reading R-1): an element v_{i,q} = (r1, r2) in S_2
(§2.1) is stored as one byte  code = 2*r1 + r2  in {0,1,2,3}.

Workload types (§5):
  * type 1  "random"  : code = splitmix64(splitmix64(seed ^ i*PHI) + q) >> 62,
                        uniform over the four codes (seed 1 is the timing input);
  * type 1b "hwe"     : Hardy-Weinberg SNP-like data, per-vector minor-allele
                        probability p_i ~ U(0.05, 0.5), each allele an
                        independent Bernoulli(p_i) draw from the same counter
                        stream (seed 2);
  * type 2  "planted" : analytically verifiable interval design (seed 3); the
                        interval lengths are returned with the codes so the
                        oracle can evaluate its closed form.

All generators are implemented with torch int64 tensors (two's-complement
wrap-around == arithmetic mod 2^64) so the same code runs on CPU or on a CUDA
device; `code_scalar` is an independent pure-Python big-int version used by
the tests to pin the tensor version.
"""
from __future__ import annotations

import torch

MASK64 = (1 << 64) - 1
PHI = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB


def _s64(x: int) -> int:
    """uint64 constant -> the int64 with the same bit pattern."""
    x &= MASK64
    return x - (1 << 64) if x >= (1 << 63) else x


_PHI_S, _M1_S, _M2_S = _s64(PHI), _s64(_M1), _s64(_M2)


def splitmix64_scalar(x: int) -> int:
    z = (x + PHI) & MASK64
    z = ((z ^ (z >> 30)) * _M1) & MASK64
    z = ((z ^ (z >> 27)) * _M2) & MASK64
    return z ^ (z >> 31)


def code_scalar(seed: int, i: int, q: int) -> int:
    """Type-1 code of element (i, q), pure Python (reference for the tensor path)."""
    h = splitmix64_scalar((seed ^ (i * PHI)) & MASK64)
    return splitmix64_scalar((h + q) & MASK64) >> 62


def _lsr(x: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (x >> s) & ((1 << (64 - s)) - 1)


def _splitmix64(x: torch.Tensor) -> torch.Tensor:
    z = x + _PHI_S
    z = (z ^ _lsr(z, 30)) * _M1_S
    z = (z ^ _lsr(z, 27)) * _M2_S
    return z ^ _lsr(z, 31)


def _row_hash(seed: int, rows: torch.Tensor) -> torch.Tensor:
    # seed ^ (i * PHI) in uint64 arithmetic, then one splitmix round.
    return _splitmix64(torch.bitwise_xor(rows * _PHI_S, _s64(seed)))


def random_codes(n_v: int, n_f: int, seed: int = 1, device="cpu",
                 row0: int = 0, chunk_rows: int = 256) -> torch.Tensor:
    """Type-1 uniform codes, uint8 [n_v][n_f] (rows are global indices row0..row0+n_v-1)."""
    out = torch.empty((n_v, n_f), dtype=torch.uint8, device=device)
    q = torch.arange(n_f, dtype=torch.int64, device=device)
    for r0 in range(0, n_v, chunk_rows):
        r1 = min(n_v, r0 + chunk_rows)
        rows = torch.arange(row0 + r0, row0 + r1, dtype=torch.int64, device=device)
        h = _row_hash(seed, rows)[:, None]
        z = _splitmix64(h + q[None, :])
        out[r0:r1] = _lsr(z, 62).to(torch.uint8)
    return out


def hwe_codes(n_v: int, n_f: int, seed: int = 2, device="cpu",
              row0: int = 0, chunk_rows: int = 256) -> torch.Tensor:
    """Type-1b Hardy-Weinberg codes: r1, r2 ~ Bernoulli(p_i), p_i ~ U(0.05, 0.5)."""
    out = torch.empty((n_v, n_f), dtype=torch.uint8, device=device)
    q = torch.arange(n_f, dtype=torch.int64, device=device)
    two53 = float(1 << 53)
    for r0 in range(0, n_v, chunk_rows):
        r1 = min(n_v, r0 + chunk_rows)
        rows = torch.arange(row0 + r0, row0 + r1, dtype=torch.int64, device=device)
        h = _row_hash(seed, rows)
        u_row = _lsr(_splitmix64(h ^ 0x5bd1e995), 11).to(torch.float64) / two53
        p = (0.05 + 0.45 * u_row)[:, None]
        z1 = _splitmix64(h[:, None] + 2 * q[None, :])
        z2 = _splitmix64(h[:, None] + 2 * q[None, :] + 1)
        u1 = _lsr(z1, 11).to(torch.float64) / two53
        u2 = _lsr(z2, 11).to(torch.float64) / two53
        out[r0:r1] = ((u1 < p).to(torch.uint8) << 1) | (u2 < p).to(torch.uint8)
    return out


def sparse_codes(n_v: int, n_f: int, seed: int = 4, device="cpu", row0: int = 0,
                 miss_max: float = 0.3, chunk_rows: int = 256) -> torch.Tensor:
    """Type-3 sparse-mode data (§7 item 1): Hardy-Weinberg
    genotypes as in hwe_codes with the heterozygote always stored as (0,1) = code 1, and
    each entry missing -- the marker (1,0) = code 2 -- with a per-vector probability
    m_i ~ U(0, miss_max)."""
    out = torch.empty((n_v, n_f), dtype=torch.uint8, device=device)
    q = torch.arange(n_f, dtype=torch.int64, device=device)
    two53 = float(1 << 53)
    for r0 in range(0, n_v, chunk_rows):
        r1 = min(n_v, r0 + chunk_rows)
        rows = torch.arange(row0 + r0, row0 + r1, dtype=torch.int64, device=device)
        h = _row_hash(seed, rows)
        u_row = _lsr(_splitmix64(h ^ 0x5bd1e995), 11).to(torch.float64) / two53
        u_mis = _lsr(_splitmix64(h ^ 0x27d4eb2f), 11).to(torch.float64) / two53
        p = (0.05 + 0.45 * u_row)[:, None]
        m = (miss_max * u_mis)[:, None]
        z1 = _splitmix64(h[:, None] + 3 * q[None, :])
        z2 = _splitmix64(h[:, None] + 3 * q[None, :] + 1)
        z3 = _splitmix64(h[:, None] + 3 * q[None, :] + 2)
        u1 = _lsr(z1, 11).to(torch.float64) / two53
        u2 = _lsr(z2, 11).to(torch.float64) / two53
        u3 = _lsr(z3, 11).to(torch.float64) / two53
        a1, a2 = (u1 < p), (u2 < p)
        code = torch.where(a1 & a2, 3, torch.where(a1 ^ a2, 1, 0))
        out[r0:r1] = torch.where(u3 < m, 2, code).to(torch.uint8)
    return out


def planted_lengths(n_v: int, n_f: int, seed: int = 3):
    """Interval lengths (L_i, H_i) of the planted type-2 design (L_i + H_i <= n_f)."""
    L, H = [], []
    for i in range(n_v):
        a = splitmix64_scalar((seed ^ (i * PHI)) & MASK64)
        b = splitmix64_scalar(a)
        li = a % (n_f + 1)
        hi = b % (n_f - li + 1)
        L.append(int(li))
        H.append(int(hi))
    return L, H


def planted_codes(n_v: int, n_f: int, seed: int = 3, device="cpu", permute: bool = True,
                  chunk_rows: int = 256):
    """Type-2 planted data (§5: "randomized placement of entries
    specifically chosen so that the correctness of every result value can be verified
    analytically").

    Before the column permutation, vector i holds code 3 = (1,1) on [0, L_i), the
    heterozygous codes 1 = (0,1) / 2 = (1,0) alternating (by field parity) on
    [L_i, L_i + H_i), and code 0 = (0,0) after. One seeded column permutation shared
    by all vectors is then applied. Generated chunk by chunk of rows on `device` (full
    sizes stay within memory). Returns (codes uint8 [n_v][n_f], L, H, perm).
    """
    L, H = planted_lengths(n_v, n_f, seed)
    perm = torch.arange(n_f)
    if permute:
        g = torch.Generator().manual_seed(seed)
        perm = torch.randperm(n_f, generator=g)
    out = torch.empty((n_v, n_f), dtype=torch.uint8, device=device)
    # column c of the output holds pre-permutation field perm[c]
    qp = perm.to(device=device, dtype=torch.int64)[None, :]
    het = torch.where((qp % 2) == 0, 1, 2).to(torch.uint8)
    Lt = torch.tensor(L, dtype=torch.int64, device=device)[:, None]
    Et = Lt + torch.tensor(H, dtype=torch.int64, device=device)[:, None]
    for r0 in range(0, n_v, chunk_rows):
        r1 = min(n_v, r0 + chunk_rows)
        lo, hi = Lt[r0:r1], Et[r0:r1]
        c = torch.where(qp < hi, het, torch.zeros((), dtype=torch.uint8, device=device))
        out[r0:r1] = torch.where(qp < lo, torch.full((), 3, dtype=torch.uint8, device=device), c)
    return out, L, H, perm


def make_codes(kind: str, n_v: int, n_f: int, seed: int | None = None, device="cpu",
               row0: int = 0) -> torch.Tensor:
    if kind == "random":
        return random_codes(n_v, n_f, 1 if seed is None else seed, device, row0)
    if kind == "hwe":
        return hwe_codes(n_v, n_f, 2 if seed is None else seed, device, row0)
    if kind == "sparse":
        return sparse_codes(n_v, n_f, 4 if seed is None else seed, device, row0)
    if kind == "planted":
        if row0:
            raise ValueError("planted data is generated whole")
        return planted_codes(n_v, n_f, 3 if seed is None else seed, device)[0]
    raise ValueError(f"unknown input kind {kind!r}")

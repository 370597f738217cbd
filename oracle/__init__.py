"""CPU oracle for the CCC method -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this package.  The product (paper_1705_08213_b200/) never imports,
links or executes anything under oracle/, and this package never imports the
product: the two share no code.

What lives here, each a literal transcription of PAPER.md (arXiv 1705.08213):

* ``ccc_oracle.c`` (built to ``liboracle.so``): brute-force per-field enumeration of
  Fig.1 / Fig.2 pairings (Eq.2, Eq.5), Eq.1 allele sums, Eq.3 / Eq.4 CCC in fp64.
* pure-Python versions of the same for tiny inputs (``tally2_py`` ...), exact
  rational CCC (``ccc2_exact`` / ``ccc3_exact``) with gamma = Fraction(2, 3),
* the paper's own 3-way route: Table 1 masking X_{j,xi} + the masked
  tally B_{j,xi} + the eight reconstruction equations, under
  the readings A-2 / A-3 of DESIGN.md,
* the closed form of the planted type-2 dataset,
* the order-independent 128-bit checksum (reading R-9).

Pins (tests/test_oracle.py): SPEC hand values and our own n_f = 1 worked examples
(tests/golden/), closed forms, invariants, exact rationals, the Table-1 route,
numpy integer matmul identities, brute force on tiny inputs.  Parity unpinned:
none of the functions above (see DESIGN.md §3 "pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction
from itertools import combinations

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ccc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
GAMMA = 2.0 / 3.0                       # P:284-285 "a fixed constant gamma = 2/3"
GAMMA_EXACT = Fraction(2, 3)

# ----------------------------------------------------------------------------------
# build / load the C brute force
# ----------------------------------------------------------------------------------


def build(force: bool = False) -> str:
    """Compile ccc_oracle.c with plain gcc -O2 -fopenmp (no tuning)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.oracle_allele_sums.argtypes = [p, i64, i64, p]
        for name in ("oracle_pairs", "oracle_triples"):
            getattr(L, name).argtypes = [p, i64, i64, p, ctypes.c_double, p, i64, p, p]
        for name in ("oracle_all_pairs", "oracle_all_triples"):
            getattr(L, name).argtypes = [p, i64, i64, p, ctypes.c_double, p, p]
        L.oracle_sparse_sums.argtypes = [p, i64, i64, p, p]
        L.oracle_sparse_pairs.argtypes = [p, i64, i64, p, p, ctypes.c_double, p, i64, p, p, p]
        L.oracle_sparse_triples.argtypes = [p, i64, i64, p, p, ctypes.c_double, p, i64, p, p, p]
        L.oracle_planted_sums.argtypes = [p, p, i64, i64, p]
        for name in ("oracle_planted_pairs", "oracle_planted_triples"):
            getattr(L, name).argtypes = [p, p, i64, i64, ctypes.c_double, i64, i64, p, p]
        for name in ("oracle_planted_check2", "oracle_planted_check3"):
            getattr(L, name).argtypes = [p, p, i64, i64, ctypes.c_double, i64, i64, p, p,
                                         ctypes.c_int, ctypes.c_double, p, p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _codes_np(codes) -> np.ndarray:
    if hasattr(codes, "numpy"):          # torch CPU tensor
        codes = codes.cpu().numpy()
    a = np.ascontiguousarray(codes, dtype=np.uint8)
    if a.ndim != 2:
        raise ValueError("codes must be [n_v][n_f]")
    return a


# ----------------------------------------------------------------------------------
# C-backed brute force (Eq.1-5 by enumeration)
# ----------------------------------------------------------------------------------


def allele_sums(codes) -> np.ndarray:
    """S[i][a] = sum_q rho_{i,q}(a)  (Eq.1 numerator); int64 [n_v][2]."""
    c = _codes_np(codes)
    S = np.zeros((c.shape[0], 2), dtype=np.int64)
    lib().oracle_allele_sums(_ptr(c), c.shape[0], c.shape[1], _ptr(S))
    return S


def frequencies(codes) -> np.ndarray:
    """f_i(a) = S_i(a) / (2 n_f)  (Eq.1)."""
    c = _codes_np(codes)
    return allele_sums(c) / (2.0 * c.shape[1])


def pairs(codes, idx, gamma: float = GAMMA, S=None):
    """Tallies int64 [m][4] and CCC fp64 [m][4] for the pairs idx [m][2] (Eq.2, Eq.3)."""
    c = _codes_np(codes)
    idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, 2)
    S = allele_sums(c) if S is None else np.ascontiguousarray(S, dtype=np.int64)
    T = np.zeros((len(idx), 4), dtype=np.int64)
    C = np.zeros((len(idx), 4), dtype=np.float64)
    lib().oracle_pairs(_ptr(c), c.shape[0], c.shape[1], _ptr(S), gamma, _ptr(idx), len(idx),
                       _ptr(T), _ptr(C))
    return T, C


def triples(codes, idx, gamma: float = GAMMA, S=None):
    """Tallies int64 [m][8] and CCC fp64 [m][8] for triples idx [m][3] (Eq.4, Eq.5)."""
    c = _codes_np(codes)
    idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, 3)
    S = allele_sums(c) if S is None else np.ascontiguousarray(S, dtype=np.int64)
    T = np.zeros((len(idx), 8), dtype=np.int64)
    C = np.zeros((len(idx), 8), dtype=np.float64)
    lib().oracle_triples(_ptr(c), c.shape[0], c.shape[1], _ptr(S), gamma, _ptr(idx), len(idx),
                         _ptr(T), _ptr(C))
    return T, C


def all_pairs(codes, gamma: float = GAMMA):
    """Every unique pair i<j, lexicographic: (T [C(n,2)][4], CCC [..][4])."""
    c = _codes_np(codes)
    n = c.shape[0]
    m = n * (n - 1) // 2
    S = allele_sums(c)
    T = np.zeros((m, 4), dtype=np.int64)
    C = np.zeros((m, 4), dtype=np.float64)
    if m:
        lib().oracle_all_pairs(_ptr(c), n, c.shape[1], _ptr(S), gamma, _ptr(T), _ptr(C))
    return T, C


def all_triples(codes, gamma: float = GAMMA):
    """Every unique triple i<j<k, lexicographic: (T [C(n,3)][8], CCC)."""
    c = _codes_np(codes)
    n = c.shape[0]
    m = n * (n - 1) * (n - 2) // 6
    S = allele_sums(c)
    T = np.zeros((m, 8), dtype=np.int64)
    C = np.zeros((m, 8), dtype=np.float64)
    if m:
        lib().oracle_all_triples(_ptr(c), n, c.shape[1], _ptr(S), gamma, _ptr(T), _ptr(C))
    return T, C


# ----------------------------------------------------------------------------------
# Sparse (missing-data) mode, P:1028-1043 under reading A-17 (see ccc_oracle.c)
# ----------------------------------------------------------------------------------
MISSING = 2   # code of the element (1,0), the missing-entry marker


def sparse_sums(codes):
    """(S int64 [n_v][2] over present entries, c int64 [n_v] = #present entries)."""
    c = _codes_np(codes)
    S = np.zeros((c.shape[0], 2), dtype=np.int64)
    cnt = np.zeros(c.shape[0], dtype=np.int64)
    lib().oracle_sparse_sums(_ptr(c), c.shape[0], c.shape[1], _ptr(S), _ptr(cnt))
    return S, cnt


def sparse_pairs(codes, idx, gamma: float = GAMMA):
    """Sparse-mode tallies [m][4], CCC [m][4] and c_ij [m] for the pairs idx [m][2]."""
    c = _codes_np(codes)
    idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, 2)
    S, cnt = sparse_sums(c)
    T = np.zeros((len(idx), 4), dtype=np.int64)
    C = np.zeros((len(idx), 4), dtype=np.float64)
    cij = np.zeros(len(idx), dtype=np.int64)
    if len(idx):
        lib().oracle_sparse_pairs(_ptr(c), c.shape[0], c.shape[1], _ptr(S), _ptr(cnt), gamma,
                                  _ptr(idx), len(idx), _ptr(T), _ptr(C), _ptr(cij))
    return T, C, cij


def sparse_triples(codes, idx, gamma: float = GAMMA):
    """Sparse mode (reading A-17) for an explicit triple list: (T [m][8], CCC, c_ijk)."""
    c = _codes_np(codes)
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64).reshape(-1, 3))
    S, cnt = sparse_sums(c)
    m = idx.shape[0]
    T = np.zeros((m, 8), np.int64)
    C = np.zeros((m, 8), np.float64)
    cc = np.zeros(m, np.int64)
    if m:
        lib().oracle_sparse_triples(_ptr(c), c.shape[0], c.shape[1], _ptr(S), _ptr(cnt), gamma,
                                    _ptr(idx), m, _ptr(T), _ptr(C), _ptr(cc))
    return T, C, cc


def sparse_all_triples(codes, gamma: float = GAMMA):
    """Every unique triple i<j<k, lexicographic: sparse (T, CCC, c_ijk)."""
    return sparse_triples(codes, triple_list(_codes_np(codes).shape[0]), gamma)


def sparse_all_pairs(codes, gamma: float = GAMMA):
    """Every unique pair i<j, lexicographic: sparse (T, CCC, c_ij)."""
    return sparse_pairs(codes, pair_list(_codes_np(codes).shape[0]), gamma)


def pair_list(n_v: int) -> np.ndarray:
    """The unique pairs in the order the paper's results are enumerated (i<j, lexicographic)."""
    return np.array(list(combinations(range(n_v), 2)), dtype=np.int64).reshape(-1, 2)


def triple_list(n_v: int) -> np.ndarray:
    return np.array(list(combinations(range(n_v), 3)), dtype=np.int64).reshape(-1, 3)


# ----------------------------------------------------------------------------------
# pure-Python versions (tiny inputs) and exact rationals
# ----------------------------------------------------------------------------------


def decode(code: int):
    """code -> v_{i,q} = (r1, r2)   (R-1)."""
    return ((code >> 1) & 1, code & 1)


def rho(code: int, a: int) -> int:
    """rho_{i,q}(a) = sum_r chi_a((v_{i,q})_r)."""
    return sum(1 for r in decode(code) if r == a)


def tally2_py(vi, vj):
    """Fig.1: enumerate the 4 pairings of each field and tally them."""
    T = [0, 0, 0, 0]
    for ci, cj in zip(vi, vj):
        for r in decode(int(ci)):
            for rp in decode(int(cj)):
                T[2 * r + rp] += 1
    return T


def tally3_py(vi, vj, vk):
    """Fig.2: enumerate the 8 combinations of each field and tally them."""
    T = [0] * 8
    for ci, cj, ck in zip(vi, vj, vk):
        for r in decode(int(ci)):
            for rp in decode(int(cj)):
                for rpp in decode(int(ck)):
                    T[4 * r + 2 * rp + rpp] += 1
    return T


def freq_exact(v, a: int) -> Fraction:
    """Eq.1 in rationals."""
    return Fraction(sum(rho(int(c), a) for c in v), 2 * len(v))


def ccc2_exact(vi, vj, gamma=GAMMA_EXACT):
    """Eq.2 + Eq.3 in exact rationals, cells a-major."""
    n_f = len(vi)
    T = tally2_py(vi, vj)
    out = []
    for a in (0, 1):
        for b in (0, 1):
            f_ij = Fraction(T[2 * a + b], 4 * n_f)
            out.append(f_ij * (1 - gamma * freq_exact(vi, a)) * (1 - gamma * freq_exact(vj, b)))
    return out


def ccc3_exact(vi, vj, vk, gamma=GAMMA_EXACT):
    """Eq.4 + Eq.5 in exact rationals, cells a-major (a for i, b for j, c for k)."""
    n_f = len(vi)
    T = tally3_py(vi, vj, vk)
    out = []
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                f = Fraction(T[4 * a + 2 * b + c], 8 * n_f)
                out.append(f * (1 - gamma * freq_exact(vi, a)) * (1 - gamma * freq_exact(vj, b))
                           * (1 - gamma * freq_exact(vk, c)))
    return out


# ----------------------------------------------------------------------------------
# the paper's 3-way route: Table 1 masks + masked 2-way tallies + R-eqs (§3.2)
# ----------------------------------------------------------------------------------

NULL = (1, 0)                                     # the "null" indicator
CLASSES = {1: ((0, 0),), 2: ((0, 1), (1, 0)), 3: ((1, 1),)}   # xi -> classes of v_j


def x_entry(v_entry, vj_entry, xi: int):
    """(X_{j,xi})_{q,p} by the TEXT rule (reading A-3 of DESIGN.md):
    the entry of V, with (1,0) mapped to (0,1), if v_j equals class xi, else null."""
    if tuple(vj_entry) in CLASSES[xi]:
        return (0, 1) if tuple(v_entry) == (1, 0) else tuple(v_entry)
    return NULL


def masked_tally(vj, vi, vk, xi: int):
    """(B_{j,xi})_{(i,k)} = X_{j,xi}^T o_3 V at (i,k): the 2-way tally of column i of
    X_{j,xi} against v_k with null entries discarded."""
    T = [0, 0, 0, 0]
    for cj, ci, ck in zip(vj, vi, vk):
        x = x_entry(decode(int(ci)), decode(int(cj)), xi)
        if x == NULL:
            continue
        for r in x:
            for rp in decode(int(ck)):
                T[2 * r + rp] += 1
    return T


def reconstruct3(B1, B2, B3):
    """The eight equations of P:537-560 under reading A-2 of DESIGN.md: the first
    argument slot of the printed f_{i,j,k}(x,y,z) is the pivot (j) allele, (y,z) are
    the (i,k) alleles.  Returns tallies in the Eq.5 order, index 4a+2b+c."""
    T = [0] * 8
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                Bx = B1 if b == 0 else B3
                T[4 * a + 2 * b + c] = 2 * Bx[2 * a + c] + B2[2 * a + c]
    return T


def tally3_via_table1(vi, vj, vk):
    return reconstruct3(masked_tally(vj, vi, vk, 1), masked_tally(vj, vi, vk, 2),
                        masked_tally(vj, vi, vk, 3))


# ----------------------------------------------------------------------------------
# planted type-2 closed form
# ----------------------------------------------------------------------------------


def _overlap(a0, a1, b0, b1):
    return max(0, min(a1, b1) - max(a0, b0))


def planted_count_intervals(L, H, i):
    """Per vector: [(start, end, allele-1 count)] intervals before the column permutation."""
    return [(0, L[i], 2), (L[i], L[i] + H[i], 1)]


def planted_tally2(L, H, n_f, i, j):
    """Closed-form 2x2 tally of the planted design: with n = allele-1 count,
    T(1,1) = sum n_i n_j, T(1,0) = sum n_i (2-n_j), T(0,1) = sum (2-n_i) n_j,
    T(0,0) = sum (2-n_i)(2-n_j) evaluated per interval intersection (rho(1)=n, rho(0)=2-n)."""
    T = [0, 0, 0, 0]
    bi = [(0, L[i], 2), (L[i], L[i] + H[i], 1), (L[i] + H[i], n_f, 0)]
    bj = [(0, L[j], 2), (L[j], L[j] + H[j], 1), (L[j] + H[j], n_f, 0)]
    for (s0, e0, ni) in bi:
        for (s1, e1, nj) in bj:
            w = _overlap(s0, e0, s1, e1)
            if not w:
                continue
            for a in (0, 1):
                for b in (0, 1):
                    ra = ni if a == 1 else 2 - ni
                    rb = nj if b == 1 else 2 - nj
                    T[2 * a + b] += w * ra * rb
    return T


def _lh(L, H):
    return (np.ascontiguousarray(L, dtype=np.int64), np.ascontiguousarray(H, dtype=np.int64))


def planted_sums(L, H, n_f):
    """Eq.1 numerators S [n_v][2] of the planted vectors, by the piecewise closed form of
    ccc_oracle.c (rho constant between the breakpoints 0, L_i, L_i + H_i, n_f)."""
    L, H = _lh(L, H)
    S = np.zeros((len(L), 2), dtype=np.int64)
    lib().oracle_planted_sums(_ptr(L), _ptr(H), len(L), n_f, _ptr(S))
    return S


def planted_pairs(L, H, n_f, rec0=0, nrec=None, gamma: float = GAMMA):
    """Closed-form records [rec0, rec0+nrec) of the lexicographic pair order:
    (T int64 [nrec][4], CCC fp64 [nrec][4])."""
    L, H = _lh(L, H)
    n_v = len(L)
    if nrec is None:
        nrec = n_v * (n_v - 1) // 2 - rec0
    T = np.zeros((nrec, 4), np.int64)
    C = np.zeros((nrec, 4), np.float64)
    if nrec:
        lib().oracle_planted_pairs(_ptr(L), _ptr(H), n_v, n_f, gamma, rec0, nrec, _ptr(T), _ptr(C))
    return T, C


def planted_triples(L, H, n_f, rec0=0, nrec=None, gamma: float = GAMMA):
    """Closed-form records [rec0, rec0+nrec) of the lexicographic triple order."""
    L, H = _lh(L, H)
    n_v = len(L)
    if nrec is None:
        nrec = n_v * (n_v - 1) * (n_v - 2) // 6 - rec0
    T = np.zeros((nrec, 8), np.int64)
    C = np.zeros((nrec, 8), np.float64)
    if nrec:
        lib().oracle_planted_triples(_ptr(L), _ptr(H), n_v, n_f, gamma, rec0, nrec, _ptr(T), _ptr(C))
    return T, C


def _host_ptr(a):
    """(pointer, element size) of a contiguous host array (numpy or torch CPU tensor)."""
    if a is None:
        return None, 0
    if hasattr(a, "data_ptr"):
        if a.is_cuda or not a.is_contiguous():
            raise ValueError("records must be contiguous host memory")
        return ctypes.c_void_p(a.data_ptr()), a.element_size()
    a = np.ascontiguousarray(a)
    return _ptr(a), a.itemsize


def planted_check(way: int, L, H, n_f, rec0, nrec, T=None, C=None, rtol=1e-12,
                  gamma: float = GAMMA):
    """Compare caller-held records [rec0, rec0+nrec) (tallies uint32/int32 [nrec][cells],
    CCC fp64 or fp32 [nrec][cells], host memory) with the planted closed form, record by
    record in C.  Returns dict(bad_tallies, bad_ccc, first_bad, max_rel)."""
    L, H = _lh(L, H)
    cells = 4 if way == 2 else 8
    for a in (T, C):
        if a is not None and tuple(a.shape) != (nrec, cells):
            raise ValueError(f"records must be [{nrec}][{cells}]")
    pt, st = _host_ptr(T)
    if T is not None and st != 4:
        raise ValueError("tallies must be 32-bit")
    pc, sc = _host_ptr(C)
    res = np.zeros(3, np.int64)
    mrel = ctypes.c_double(0.0)
    fn = lib().oracle_planted_check2 if way == 2 else lib().oracle_planted_check3
    fn(_ptr(L), _ptr(H), len(L), n_f, gamma, rec0, nrec, pt, pc, sc, rtol, _ptr(res),
       ctypes.byref(mrel))
    keep = (T, C)   # noqa: F841 -- alive across the call
    return {"bad_tallies": int(res[0]), "bad_ccc": int(res[1]), "first_bad": int(res[2]),
            "max_rel": mrel.value}


def planted_tally3(L, H, n_f, i, j, k):
    T = [0] * 8
    segs = lambda v: [(0, L[v], 2), (L[v], L[v] + H[v], 1), (L[v] + H[v], n_f, 0)]
    for (s0, e0, ni) in segs(i):
        for (s1, e1, nj) in segs(j):
            for (s2, e2, nk) in segs(k):
                w = max(0, min(e0, e1, e2) - max(s0, s1, s2))
                if not w:
                    continue
                for a in (0, 1):
                    for b in (0, 1):
                        for c in (0, 1):
                            ra = ni if a else 2 - ni
                            rb = nj if b else 2 - nj
                            rc = nk if c else 2 - nk
                            T[4 * a + 2 * b + c] += w * ra * rb * rc
    return T


# ----------------------------------------------------------------------------------
# checksum ("extended precision integer arithmetic"; reading R-9)
# ----------------------------------------------------------------------------------

M64 = (1 << 64) - 1
CK_SEED = 0x243F6A8885A308D3
CK_HI = 0x13198A2E03707344


def fmix64(k: int) -> int:
    k &= M64
    k ^= k >> 33
    k = (k * 0xFF51AFD7ED558CCD) & M64
    k ^= k >> 33
    k = (k * 0xC4CEB9FE1A85EC53) & M64
    k ^= k >> 33
    return k


def record_digest(way: int, idx, tallies) -> int:
    """128-bit digest of one record (way, i, j[, k], tallies) per DESIGN.md R-9."""
    i, j = int(idx[0]), int(idx[1])
    k = int(idx[2]) if way == 3 else 0
    lanes = [(way << 60) | (i << 40) | (j << 20) | k]
    t = [int(x) for x in tallies]
    for p in range(0, len(t), 2):
        lanes.append((t[p] & 0xFFFFFFFF) | ((t[p + 1] & 0xFFFFFFFF) << 32))
    h = CK_SEED
    for lane in lanes:
        h = fmix64(h ^ lane)
    return (fmix64(h ^ CK_HI) << 64) | h


def checksum_scalar(way: int, idx, T) -> int:
    """Sum of record digests mod 2^128 (record by record, Python integers)."""
    acc = 0
    for r in range(len(idx)):
        acc = (acc + record_digest(way, idx[r], T[r])) & ((1 << 128) - 1)
    return acc


def _fmix64_np(k):
    k = k ^ (k >> np.uint64(33))
    k = k * np.uint64(0xFF51AFD7ED558CCD)
    k = k ^ (k >> np.uint64(33))
    k = k * np.uint64(0xC4CEB9FE1A85EC53)
    return k ^ (k >> np.uint64(33))


def checksum(way: int, idx, T) -> int:
    """Same value as checksum_scalar, evaluated with numpy uint64 (wrap-around) arrays."""
    if len(T) == 0:
        return 0
    idx = np.asarray(idx, dtype=np.int64).reshape(len(T), -1).astype(np.uint64)
    T = np.asarray(T, dtype=np.int64).astype(np.uint64) & np.uint64(0xFFFFFFFF)
    k = idx[:, 2] if way == 3 else np.zeros(len(T), np.uint64)
    lane0 = ((np.uint64(way) << np.uint64(60)) | (idx[:, 0] << np.uint64(40))
             | (idx[:, 1] << np.uint64(20)) | k)
    with np.errstate(over="ignore"):
        h = _fmix64_np(np.uint64(CK_SEED) ^ lane0)
        for p in range(0, T.shape[1], 2):
            h = _fmix64_np(h ^ (T[:, p] | (T[:, p + 1] << np.uint64(32))))
        hi = _fmix64_np(h ^ np.uint64(CK_HI))
    m32 = np.uint64(0xFFFFFFFF)
    total = 0
    for part, shift in ((h, 0), (hi, 64)):
        lo32 = int((part & m32).sum(dtype=np.uint64))
        hi32 = int((part >> np.uint64(32)).sum(dtype=np.uint64))
        total += (lo32 + (hi32 << 32)) << shift
    return total & ((1 << 128) - 1)

"""Comparison baselines -- REPORTED LINES ONLY.

``cpu_popcount.c`` is the paper's "optimized CPU version": a bit-packed,
OpenMP, popcount 2-way tally on the host cores.  bench.py reports it next to the oracle;
the product path (paper_1705_08213_b200/) never imports or calls anything here, and this
package imports neither the product nor the oracle (tests compare it with the oracle).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cpu_popcount.c")
_LIB = os.path.join(_HERE, "libcpu_popcount.so")
_lib = None


def build(force: bool = False) -> str:
    """gcc -O3 -fopenmp with the x86-64 popcnt instruction (portable to any box CPU)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-mpopcnt", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        f = L.cpu_popcount_2way
        f.restype = None
        f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                      ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        _lib = L
    return _lib


def pack(codes: np.ndarray) -> np.ndarray:
    """2-bit packing of the C ABI's ccc_pack layout (4 codes per byte, LSB first, rows of
    ceil(n_f/64)*16 bytes), written out here so the baseline has no GPU dependency."""
    codes = np.asarray(codes, np.uint8)
    n_v, n_f = codes.shape
    stride = (n_f + 63) // 64 * 16
    c = np.zeros((n_v, stride * 4), np.uint8)
    c[:, :n_f] = codes & 3
    c = c.reshape(n_v, stride, 4)
    return (c[..., 0] | (c[..., 1] << 2) | (c[..., 2] << 4) | (c[..., 3] << 6)).astype(np.uint8)


def popcount_2way(packed: np.ndarray, n_f: int, gamma: float = 2.0 / 3.0, i_lo: int = 0,
                  i_hi: int | None = None, want_ccc: bool = True):
    """Tallies [m][4] (uint32) and CCC [m][4] for the pairs of rows [i_lo, i_hi)."""
    packed = np.ascontiguousarray(packed, np.uint8)
    n_v = packed.shape[0]
    i_hi = n_v if i_hi is None else i_hi
    m = sum(max(0, n_v - i - 1) for i in range(i_lo, i_hi))
    T = np.zeros((m, 4), np.uint32)
    C = np.zeros((m, 4), np.float64) if want_ccc else None
    lib().cpu_popcount_2way(packed.ctypes.data, n_v, n_f, gamma, i_lo, i_hi, T.ctypes.data,
                            C.ctypes.data if want_ccc else None)
    return T, C

"""paper_1705_08213_b200 -- B200-native (sm_100a) CCC tally engine.

The hot path of arXiv 1705.08213 (CoMet CCC): 2-way / 3-way allele co-occurrence
tallies and CCC values for every unique pair / triple of 2-bit genotype vectors,
computed by hand-written tcgen05 kind::i8 kernels in libccc.so behind the C ABI of
include/ccc.h.  `ccc` is the ctypes binding; `decomp` / `dist` hold the multi-GPU
block-circulant (2-way) and tetrahedral (3-way) schedules.
"""
from . import ccc  # noqa: F401
from .ccc import (OUT_CCC_F32, OUT_CCC_F64, OUT_CHECKSUM, OUT_TALLY, GAMMA, CCCError,  # noqa
                  two_way, three_way)

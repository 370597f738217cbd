"""Diagnostic check: C2 records of a library variant (CCC_LIB) -- checksum and a sample vs the oracle."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import oracle
import synthgen
from paper_1705_08213_b200 import ccc
n_v, n_f = 20000, 50000
codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
T, C, ck = ccc.ccc_2way_codes(codes, out_flags=11)
rng = np.random.default_rng(2)
i = rng.integers(0, n_v - 1, 300)
j = np.array([rng.integers(a + 1, n_v) for a in i])
rows = torch.tensor([ccc.ccc_pair_index(n_v, int(a), int(b)) for a, b in zip(i, j)], device="cuda")
To, Co = oracle.pairs(codes.cpu(), np.stack([i, j], 1))
print("sample ok", np.array_equal(T[rows].cpu().numpy().astype(np.int64) & 0xFFFFFFFF, To),
      "checksum", f"{ccc.checksum_int(ck):032x}")

"""Diagnostic check: C4 stage records of a library variant equal the default library's
(run twice with CCC_LIB; compares via a checksum and sampled records against the oracle)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import oracle
import synthgen
from paper_1705_08213_b200 import ccc
n_v, n_f, n_st = 4096, 16384, 16
codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
ws = ccc.ccc_3way_prepare(ccc.ccc_pack(codes), n_f)
rng = np.random.default_rng(2)
for st in (0, 15):
    T, C, ck = ccc.ccc_3way_stage(n_v, n_f, n_st, st, ws, 11)
    i0, i1, r0, rc = ccc.ccc_stage_range(n_v, n_st, st)
    tl = set()
    while len(tl) < 400:
        i = int(rng.integers(i0, min(i1, n_v - 2)))
        j = int(rng.integers(i + 1, n_v - 1))
        k = int(rng.integers(j + 1, n_v))
        tl.add((i, j, k))
    tl = sorted(tl)
    rows = torch.tensor([ccc.ccc_triple_index(n_v, *t) - r0 for t in tl], device="cuda")
    To, Co = oracle.triples(codes.cpu(), np.array(tl))
    ok = np.array_equal(T[rows].cpu().numpy().astype(np.int64) & 0xFFFFFFFF, To)
    print("stage", st, "sample ok", ok, "checksum", f"{ccc.checksum_int(ck):032x}")

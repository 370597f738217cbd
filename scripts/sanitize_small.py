"""Small end-to-end run of every kernel for compute-sanitizer (memcheck/racecheck/synccheck)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import oracle
import synthgen
from paper_1705_08213_b200 import ccc, decomp

F = ccc.OUT_TALLY | ccc.OUT_CCC_F64 | ccc.OUT_CHECKSUM
codes = synthgen.random_codes(300, 333, seed=3)
T, C, ck = ccc.two_way(codes.cuda(), out_flags=F)
To, _ = oracle.all_pairs(codes)
assert np.array_equal(T.cpu().numpy().astype(np.int64) & 0xFFFFFFFF, To)
codes = synthgen.random_codes(150, 200, seed=4)
T, C, ck = ccc.three_way(codes.cuda(), out_flags=F, n_stages=2, stage=1)
n_v, n_f = 150, 200
N, s, w = ccc.ccc_expand(ccc.ccc_pack(codes.cuda()), n_f)
G = torch.zeros((n_v, n_v), dtype=torch.int32, device="cuda")
ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, 0, g=G, ldg=n_v)
bounds = decomp.block_bounds(n_v, 3)
ex = [ccc.ccc_expand(ccc.ccc_pack(codes[lo:hi].contiguous().cuda()), n_f) for lo, hi in bounds]
b = [ccc.block(*ex[i], bounds[i][0]) for i in range(3)]
u = decomp.plan_3way(3, 1, bounds)[-1]
ccc.ccc_3way_unit(b[u.pb], u.p_lo, u.p_hi, b[u.mb], u.m_lo, u.m_hi, b[u.nb], u.n_lo, u.n_hi, u.order, G, n_f, F)
torch.cuda.synchronize()
print("sanitize run ok")

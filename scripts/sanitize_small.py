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
# the flag-free FULL epilogue (aligned record groups, extra chunk) over two column tiles
T, C, _ = ccc.three_way(synthgen.random_codes(300, 130, seed=6).cuda(),
                        out_flags=ccc.OUT_TALLY | ccc.OUT_CCC_F64, n_stages=3, stage=2)
n_v, n_f = 150, 200
N, s, w = ccc.ccc_expand(ccc.ccc_pack(codes.cuda()), n_f)
G = torch.zeros((n_v, n_v), dtype=torch.int32, device="cuda")
ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, 0, g=G, ldg=n_v)
bounds = decomp.block_bounds(n_v, 3)
ex = [ccc.ccc_expand(ccc.ccc_pack(codes[lo:hi].contiguous().cuda()), n_f) for lo, hi in bounds]
b = [ccc.block(*ex[i], bounds[i][0]) for i in range(3)]
u = decomp.plan_3way(3, 1, bounds)[-1]
ccc.ccc_3way_unit(b[u.pb], u.p_lo, u.p_hi, b[u.mb], u.m_lo, u.m_hi, b[u.nb], u.n_lo, u.n_hi, u.order, G, n_f, F)
# sparse 2-way / 3-way, popcount baseline, field split (f1, f4, f3)
sc = synthgen.sparse_codes(140, 210, seed=5)
ccc.ccc_2way_sparse(ccc.ccc_pack(sc.cuda()), 210, out_flags=F)
T3, C3, _ = ccc.three_way_sparse(sc[:90].contiguous().cuda(), out_flags=F, n_stages=2)
To3, _, _ = oracle.sparse_all_triples(sc[:90])
assert np.array_equal(T3.cpu().numpy().astype(np.int64) & 0xFFFFFFFF, To3)
pc = ccc.ccc_pack(codes.cuda())
Tp, _, _ = ccc.ccc_2way_popcount(pc, n_f, out_flags=F)
from paper_1705_08213_b200 import fieldsplit
Tf, _, _ = fieldsplit.run_simulated(codes.cuda(), 3, F, wave_tiles=1)
Td, _, _ = ccc.two_way(codes.cuda(), out_flags=F)
assert bool((Tp == Td).all()) and bool((Tf == Td).all())
Tf5, _, _ = fieldsplit.run_simulated(codes.cuda(), 5, F)          # generic-world finish
assert bool((Tf5 == Td).all())
c16 = synthgen.random_codes(130, 4096 + 256, seed=6)              # vector pack path
T16, _, _ = ccc.two_way(c16.cuda(), out_flags=ccc.OUT_TALLY)
To16, _ = oracle.all_pairs(c16)
assert np.array_equal(T16.cpu().numpy().astype(np.int64) & 0xFFFFFFFF, To16)
# round 2: expand_codes / ccc_2way_codes, the grid's block export/finish, the 3-way sparse
# single pass (tally3s) at a shape spanning several of its 64 x 128 tiles
Tc, _, _ = ccc.ccc_2way_codes(codes.cuda(), out_flags=F)
assert bool((Tc == Td).all())
from paper_1705_08213_b200 import grid as gridmod
res, _ = gridmod.run_grid_simulated(codes.cuda(), decomp.Grid(2, 1, 2), F, wave_tiles=1)
sc3 = synthgen.sparse_codes(200, 300, seed=7)
T3b, _, _ = ccc.three_way_sparse(sc3.cuda(), out_flags=F, n_stages=3)
To3b, _, _ = oracle.sparse_all_triples(sc3)
assert np.array_equal(T3b.cpu().numpy().astype(np.int64) & 0xFFFFFFFF, To3b)
torch.cuda.synchronize()
print("sanitize run ok")

"""Time one sparse C4 3-way stage (tally3s_kernel) with CUDA events."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synthgen
from paper_1705_08213_b200 import ccc
n_v, n_f, n_st = 4096, 16384, 16
codes = synthgen.sparse_codes(n_v, n_f, seed=4, device="cuda")
ws = ccc.ccc_3way_sparse_prepare(ccc.ccc_pack(codes), n_f)
st = int(os.environ.get("STAGE", 15))
rc = ccc.ccc_stage_range(n_v, n_st, st)[3]
T = torch.empty((rc, 8), dtype=torch.int32, device="cuda")
C = torch.empty((rc, 8), dtype=torch.float64, device="cuda")
for _ in range(2):
    ccc.ccc_3way_sparse_stage(n_v, n_f, n_st, st, ws, 3, T, C)
torch.cuda.synchronize()
ts = []
for _ in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); ccc.ccc_3way_sparse_stage(n_v, n_f, n_st, st, ws, 3, T, C); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print("sparse stage", st, "ms", sorted(ts))

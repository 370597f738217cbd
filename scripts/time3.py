"""Time one C4 3-way stage (last of 16) with CUDA events."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synthgen
from paper_1705_08213_b200 import ccc
n_v, n_f, n_st = 4096, 16384, 16
codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
gamma = float(os.environ.get("GAMMA", 2.0 / 3.0))
ws = ccc.ccc_3way_prepare(ccc.ccc_pack(codes), n_f, gamma)
st = int(os.environ.get("STAGE", 15))
_, _, _, rc = ccc.ccc_stage_range(n_v, n_st, st)
T = torch.empty((rc, 8), dtype=torch.int32, device="cuda")
C = torch.empty((rc, 8), dtype=torch.float64, device="cuda")
flags = int(os.environ.get("FLAGS", 3))
for _ in range(2):
    ccc.ccc_3way_stage(n_v, n_f, n_st, st, ws, flags, T, C, gamma=gamma)
torch.cuda.synchronize()
ts = []
for _ in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); ccc.ccc_3way_stage(n_v, n_f, n_st, st, ws, flags, T, C, gamma=gamma); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(os.environ.get("CCC_LIB", "default"), "gamma", gamma, "flags", flags, "ms", sorted(ts), "GB/s", rc * 96 / min(ts) / 1e6)

"""Per-unit %globaltimer trace of the 3-way kernel (last C4 stage) -- diagnostics."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import synthgen
from paper_1705_08213_b200 import ccc
n_v, n_f, n_st, st = 4096, 16384, 16, 15
codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
ws = ccc.ccc_3way_prepare(ccc.ccc_pack(codes), n_f)
_, _, _, rc = ccc.ccc_stage_range(n_v, n_st, st)
T = torch.empty((rc, 8), dtype=torch.int32, device="cuda")
C = torch.empty((rc, 8), dtype=torch.float64, device="cuda")
flags = int(os.environ.get("FLAGS", 3))
tr = torch.zeros((200000, 8), dtype=torch.int64, device="cuda")
os.environ["CCC_TRACE_PTR"] = str(tr.data_ptr())
ccc.ccc_3way_stage(n_v, n_f, n_st, st, ws, flags, T, C)
torch.cuda.synchronize(); tr.zero_()
ccc.ccc_3way_stage(n_v, n_f, n_st, st, ws, flags, T, C)
torch.cuda.synchronize()
a = tr.cpu().numpy()
n = int((a[:, 0] > 0).sum()); a = a[:n].astype(np.float64); a = (a - a[:, 0].min()) / 1e3
print(os.environ.get("CCC_LIB", "default"), "flags", flags, json.dumps({
    "units": n, "end_us": a[:, 2].max(), "mma_us": np.percentile(a[:, 2] - a[:, 1], [10, 50, 90]).tolist(),
    "mma_wait_tmem_us": float((a[:, 1] - a[:, 0]).mean()),
    "epi_us": np.percentile(a[:, 5] - a[:, 4], [10, 50, 90]).tolist(),
    "epi_wait_us": float((a[:, 4] - a[:, 3]).mean())}))

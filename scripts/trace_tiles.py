"""Per-tile %globaltimer trace of the 2-way tally kernel (diagnostics)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import numpy as np
import synthgen
from paper_1705_08213_b200 import ccc

n_v, n_f = int(os.environ.get("NV", 20000)), 50000
flags = int(os.environ.get("FLAGS", 3))
codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
packed = ccc.ccc_pack(codes)
N, s, w = ccc.ccc_expand(packed, n_f)
m = ccc.ccc_num_unique(2, n_v)
T = torch.empty((m, 4), dtype=torch.int32, device="cuda")
C = torch.empty((m, 4), dtype=torch.float64, device="cuda")
tr = torch.zeros((20000, 8), dtype=torch.int64, device="cuda")
os.environ["CCC_TRACE_PTR"] = str(tr.data_ptr())
ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, flags, T, C)  # warm (env read once? no: per launch)
torch.cuda.synchronize()
tr.zero_()
ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, flags, T, C)
torch.cuda.synchronize()
a = tr.cpu().numpy()
nt = int((a[:, 0] > 0).sum())
a = a[:nt].astype(np.float64)
t0 = a[:, 0].min()
a = (a - t0) / 1e3  # us
mma_wait_tmem = a[:, 1] - a[:, 0]
mma_time = a[:, 2] - a[:, 1]
epi_wait = a[:, 4] - a[:, 3]
epi_time = a[:, 5] - a[:, 4]
end = a[:, 2].max()
print(json.dumps({"tiles": nt, "kernel_us_mma_end": end,
                  "mma_wait_tmem_us_mean": mma_wait_tmem.mean(), "mma_time_us_mean": mma_time.mean(),
                  "mma_time_us_p10_p50_p90": list(np.percentile(mma_time, [10, 50, 90])),
                  "epi_time_us_mean": epi_time.mean(), "epi_time_p50_p90": list(np.percentile(epi_time, [50, 90])),
                  "epi_wait_us_mean": epi_wait.mean()}))
# per-wave view: tiles grouped by launch index
np.save(os.path.join(ROOT, "gpurun_out", f"trace_f{flags}.npy"), a)

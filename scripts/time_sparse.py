"""Time sparse-mode 2-way at C2 size (CUDA events, no profiler)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synthgen
from paper_1705_08213_b200 import ccc
n_v, n_f = int(os.environ.get("NV", 20000)), int(os.environ.get("NF", 50000))
flags = int(os.environ.get("FLAGS", 3))
codes = synthgen.sparse_codes(n_v, n_f, seed=4, device="cuda")
packed = ccc.ccc_pack(codes)
X, s, c, w = ccc.ccc_expand_sparse(packed, n_f)
m = ccc.ccc_num_unique(2, n_v)
T = torch.empty((m, 4), dtype=torch.int32, device="cuda")
C = torch.empty((m, 4), dtype=torch.float64, device="cuda")
for _ in range(2):
    ccc.ccc_2way_sparse_block(X, w, n_v, 0, 0, n_v, X, w, n_v, 0, True, n_f, flags, T, C)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ccc.ccc_2way_sparse_block(X, w, n_v, 0, 0, n_v, X, w, n_v, 0, True, n_f, flags, T, C)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
best = min(ts)
macs = 4 * m * n_f
print("sparse", n_v, n_f, "flags", flags, "ms", [round(x, 3) for x in sorted(ts)],
      "comparisons/s %.3e" % (m * n_f / best * 1e3), "int8 TOPS %.0f" % (2 * macs / best / 1e9))

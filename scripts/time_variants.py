"""Time the C2 2-way block kernel under env-selected variants (CUDA events, no profiler)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synthgen
from paper_1705_08213_b200 import ccc
n_v, n_f = 20000, 50000
flags = int(os.environ.get("FLAGS", 3))
gamma = float(os.environ.get("GAMMA", 2.0 / 3.0))
codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
packed = ccc.ccc_pack(codes)
N, s, w = ccc.ccc_expand(packed, n_f, gamma)
m = ccc.ccc_num_unique(2, n_v)
T = torch.empty((m, 4), dtype=torch.int32, device="cuda")
C = torch.empty((m, 4), dtype=torch.float64, device="cuda")
res = {}
for sup in os.environ.get("SUPERS", "2048,2048").split():
    os.environ["CCC_SUPER"] = sup
    for _ in range(2):
        ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, flags, T, C, gamma=gamma)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, flags, T, C, gamma=gamma)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res[sup] = [round(x, 3) for x in sorted(ts)]
print(os.environ.get("CCC_LIB", "default"), "gamma", gamma, json.dumps(res))

"""2-way kernel with a short K: how fast can the fused epilogue write while the MMA runs?"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synthgen
from paper_1705_08213_b200 import ccc
n_v = 20000
for n_f in [int(x) for x in os.environ.get("NFS", "128 1024 4096").split()]:
    codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
    N, s, w = ccc.ccc_expand(ccc.ccc_pack(codes), n_f)
    m = ccc.ccc_num_unique(2, n_v)
    T = torch.empty((m, 4), dtype=torch.int32, device="cuda")
    C = torch.empty((m, 4), dtype=torch.float64, device="cuda")
    ck = torch.zeros(2, dtype=torch.int64, device="cuda")
    for flags in (3, 8):
        for _ in range(2):
            ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, flags, T, C, ck)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, flags, T, C, ck); b.record()
            torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        t = min(ts)
        print(f"cta={os.environ.get('CCC_TALLY2_CTA', '2')} n_f={n_f} flags={flags} ms={t:.3f} "
              f"write GB/s={m * 48 / t / 1e6 if flags == 3 else 0:.0f} MMA TOPS={2 * m * n_f / t / 1e9:.0f}")

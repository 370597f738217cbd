"""C2 2-way block kernel time vs output flags (what the stored bytes cost), CUDA events."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import pynvml
import synthgen
pynvml.nvmlInit()
_h = pynvml.nvmlDeviceGetHandleByIndex(0)
from paper_1705_08213_b200 import ccc
n_v, n_f = int(os.environ.get("NV", 20000)), int(os.environ.get("NF", 50000))
codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
N, s, w = ccc.ccc_expand_codes(codes)
m = ccc.ccc_num_unique(2, n_v)
T = torch.empty((m, 4), dtype=torch.int32, device="cuda")
C = torch.empty((m, 4), dtype=torch.float64, device="cuda")
ck = torch.zeros(2, dtype=torch.int64, device="cuda")
_flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for flags in [int(x) for x in os.environ.get("FLAGSET", "8 1 2 5 3").split()]:
    Cx = C if flags & 2 else C.view(torch.float32)[:, :4].contiguous() if flags & 4 else None
    if flags & 4:
        Cx = torch.empty((m, 4), dtype=torch.float32, device="cuda")
    for _ in range(2):
        ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, flags, T if flags & 1 else None, Cx, ck)
    torch.cuda.synchronize()
    ts = []
    pre = os.environ.get("PRE", "")
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if pre == "expand":          # the bench step's first kernel right before
            ccc.ccc_expand_codes(codes, ccc.GAMMA, N, s, w)
        elif pre == "flush":         # a 256 MB write: evicts L2 (clean)
            torch.cuda.synchronize()
            _flush.zero_()
        a.record()
        ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, flags, T if flags & 1 else None, Cx, ck)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    byt = m * ((16 if flags & 1 else 0) + (32 if flags & 2 else 16 if flags & 4 else 0))
    mhz = pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM)
    print(f"flags={flags} bytes/pair={byt // m} ms={[round(x, 3) for x in sorted(ts)]} sm_mhz_after={mhz}")

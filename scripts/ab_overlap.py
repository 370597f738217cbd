"""A/B on one box: C2 step as expand_codes -> tally (serial) vs ccc_2way_codes (overlapped)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synthgen
from paper_1705_08213_b200 import ccc
n_v, n_f = 20000, 50000
codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
N, s, w = ccc.ccc_expand_codes(codes)
m = ccc.ccc_num_unique(2, n_v)
T = torch.empty((m, 4), dtype=torch.int32, device="cuda")
C = torch.empty((m, 4), dtype=torch.float64, device="cuda")
ws = ccc.workspace(2, n_v, n_f)


def serial():
    ccc.ccc_expand_codes(codes, ccc.GAMMA, N, s, w)
    ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, 3, T, C)


def overlapped():
    ccc.ccc_2way_codes(codes, ccc.GAMMA, 3, T, C, None, ws)


for rnd in range(3):
    for name, fn in (("serial", serial), ("overlapped", overlapped)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
        ev[0].record()
        for k in range(10):
            fn()
            ev[k + 1].record()
        torch.cuda.synchronize()
        per = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(10))
        print(f"{name:10s} mean {ev[0].elapsed_time(ev[10]) / 10:.3f} median {per[5]:.3f} best {per[0]:.3f} ms")

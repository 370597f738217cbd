"""Run the bench step (pack -> expand -> fused tally kernel) a few times for ncu.

python scripts/profile_step.py [--workload c2|c4] [--n_v N] [--n_f F] [--reps R]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synthgen  # noqa: E402
from paper_1705_08213_b200 import ccc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--n_v", type=int, default=0)
    ap.add_argument("--n_f", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--flags", type=int, default=ccc.OUT_TALLY | ccc.OUT_CCC_F64)
    a = ap.parse_args()
    if a.workload == "c2":
        n_v, n_f = a.n_v or 20000, a.n_f or 50000
        codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
        packed = ccc.ccc_pack(codes)
        N, s, w = ccc.ccc_expand(packed, n_f)
        m = ccc.ccc_num_unique(2, n_v)
        T = torch.empty((m, 4), dtype=torch.int32, device="cuda")
        C = torch.empty((m, 4), dtype=torch.float64, device="cuda")
        ck = torch.zeros(2, dtype=torch.int64, device="cuda")
        for _ in range(a.reps):
            ccc.ccc_pack(codes, packed)
            ccc.ccc_expand(packed, n_f, ccc.GAMMA, N, s, w)
            ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, a.flags, T, C, ck)
    else:
        n_v, n_f, n_st = a.n_v or 4096, a.n_f or 16384, 16
        codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
        packed = ccc.ccc_pack(codes)
        ws = ccc.ccc_3way_prepare(packed, n_f)
        for _ in range(a.reps):
            ccc.ccc_3way_stage(n_v, n_f, n_st, n_st - 1, ws, a.flags)
    torch.cuda.synchronize()
    print("done", n_v, n_f)


if __name__ == "__main__":
    main()

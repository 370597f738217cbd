"""Per-rank compute of the tetrahedral 3-way decomposition, measured on one B200.

For configs[4] (C5: 16,384 x 32,768) at P = 8 (and 1): the full expanded N and pairwise G
are built once; then every rank's units (decomp.plan_3way) run on this GPU exactly as that
rank would run them (ccc_3way_unit, FULL output into one reused piece buffer), timed with
CUDA events; no communication.  Balance of the exact cover (reading A-16) on hardware.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synthgen  # noqa: E402
from paper_1705_08213_b200 import ccc, decomp  # noqa: E402

n_v, n_f = int(os.environ.get("NV", 16384)), int(os.environ.get("NF", 32768))
flags = ccc.OUT_TALLY | ccc.OUT_CCC_F64
max_rec = int(os.environ.get("MAXREC", 600_000_000))     # 57.6 GB piece buffer
T = torch.empty((max_rec, 8), dtype=torch.int32, device="cuda")
C = torch.empty((max_rec, 8), dtype=torch.float64, device="cuda")
codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
N, s, w = ccc.ccc_expand_codes(codes)
del codes
G = torch.zeros((n_v, n_v), dtype=torch.int32, device="cuda")
ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, 0, g=G, ldg=n_v)
torch.cuda.synchronize()
out = {"n_v": n_v, "n_f": n_f, "P": {}}
for P in [int(x) for x in os.environ.get("PS", "8").split()]:
    bounds = decomp.block_bounds(n_v, P, align=256)
    blks = [ccc.block(N[lo:hi], s[lo:hi], w[lo:hi], lo) for lo, hi in bounds]
    per_rank = []
    for r in range(P):
        units = decomp.plan_3way(P, r, bounds)
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        trip = 0
        a_ev.record()
        for u in units:
            lo = u.p_lo
            while lo < u.p_hi:            # pivot pieces of <= max_rec records
                hi = lo + 1
                while hi < u.p_hi and decomp.unit3_count(decomp.Unit3(u.pb, lo, hi + 1, u.mb, u.m_lo, u.m_hi, u.nb,
                                                                      u.n_lo, u.n_hi, u.order), bounds) <= max_rec:
                    hi += 1
                n = decomp.unit3_count(decomp.Unit3(u.pb, lo, hi, u.mb, u.m_lo, u.m_hi, u.nb, u.n_lo, u.n_hi,
                                                    u.order), bounds)
                ccc.ccc_3way_unit(blks[u.pb], lo, hi, blks[u.mb], u.m_lo, u.m_hi, blks[u.nb], u.n_lo, u.n_hi,
                                  u.order, G, n_f, flags, T[:n], C[:n])
                trip += n
                lo = hi
        b_ev.record()
        torch.cuda.synchronize()
        ms = a_ev.elapsed_time(b_ev)
        per_rank.append({"rank": r, "ms": ms, "triples": trip, "units": len(units)})
        print(P, r, round(ms, 1), trip, flush=True)
    out["P"][P] = per_rank
print(json.dumps(out))

"""Per-rank compute of the block-circulant 2-way decomposition, measured on one B200.

For configs[2] (C3: 160,000 x 100,000) at P = 2, 4, 8: every rank's units (its diagonal
block, its off-diagonal blocks, the antipodal row half) run on this GPU exactly as that rank
would run them (ccc_2way_block, FULL output into one reused band buffer), timed with CUDA
events; no communication.  max over ranks / (the whole problem's time on one GPU / P) is
the efficiency the decomposition itself allows (tile quantisation of smaller blocks, the
half-empty diagonal tiles, the antipodal split), before any NVLink cost.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synthgen  # noqa: E402
from paper_1705_08213_b200 import ccc, decomp  # noqa: E402
from paper_1705_08213_b200.dist import band_records, row_bands  # noqa: E402

n_v, n_f = int(os.environ.get("NV", 160000)), int(os.environ.get("NF", 100000))
flags = ccc.OUT_TALLY | ccc.OUT_CCC_F64
max_rec = int(os.environ.get("MAXREC", 1_000_000_000))    # 48 GB band buffer
buf = ccc._outputs(max_rec, 4, flags, "cuda")[:2]
out = {"n_v": n_v, "n_f": n_f, "P": {}}
for P in [int(x) for x in os.environ.get("PS", "1 2 4 8").split()]:
    bounds = decomp.block_bounds(n_v, P, align=256)
    per_rank = []
    for r in range(P):
        units = decomp.plan_2way(P, r, bounds)
        need = sorted({b for u in units for b in (u.a, u.b)})
        ex = {}
        for b in need:
            lo, hi = bounds[b]
            ex[b] = ccc.ccc_expand_codes(synthgen.random_codes(hi - lo, n_f, seed=1, device="cuda", row0=lo))
        torch.cuda.synchronize()
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        comps = 0
        a_ev.record()
        for u in units:
            for lo, hi in row_bands(u, bounds, max_rec):
                n = band_records(u, bounds, lo, hi)
                T, C = (x[:n] for x in buf)
                ccc.ccc_2way_block(*ex[u.a], bounds[u.a][0], lo, hi, *ex[u.b], bounds[u.b][0], u.diag, n_f, flags,
                                   T, C)
                comps += n * n_f
        b_ev.record()
        torch.cuda.synchronize()
        ms = a_ev.elapsed_time(b_ev)
        per_rank.append({"rank": r, "ms": ms, "comparisons": comps})
        del ex
        torch.cuda.empty_cache()
        print(P, r, round(ms, 2), comps, flush=True)
    out["P"][P] = per_rank
if 1 in out["P"]:
    t1 = out["P"][1][0]["ms"]
    for P, pr in out["P"].items():
        worst = max(x["ms"] for x in pr)
        out.setdefault("efficiency_bound", {})[P] = t1 / P / worst
print(json.dumps(out))

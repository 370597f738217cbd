"""bench.py -- CCC comparisons/s of the B200 hot path.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                [--workload c2|c2hwe|c4|c1|c2s|c4s|c4f32|c4ck|c2pop|c2fs|c4paper] [--no-e2e] [--no-cpu]

One step = one pass of the whole hot path over one synthetic batch resident in HBM:
  2-way (default, BASELINE configs[1] = C2: 20,000 vectors x 50,000 individuals):
      ccc_pack -> ccc_expand -> ccc_2way_block (fused tally GEMM + CCC epilogue,
      every unique pair's uint32 tallies + fp64 CCC written to HBM)
  3-way (--workload c4: 4,096 x 16,384, 16 stages, FULL output, buffer reused)
  sparse 2-way (--workload c2s: C2's shape, ~15% missing entries):
      ccc_pack -> ccc_expand_sparse -> ccc_2way_sparse_block
  popcount baseline (--workload c2pop: C2 through ccc_2way_popcount, the paper's
      AND + popcount tally on CUDA cores): ccc_pack -> ccc_2way_popcount
  field split (--workload c2fs: C2 split into 4 field slices, all slices
      on one GPU): per slice ccc_pack -> ccc_expand -> ccc_2way_fs_export (tally GEMM whose
      epilogue stores partial tiles into the owners' slots), then per owner ccc_2way_fs_finish
At N > 1 (torchrun), the 2-way path runs the block-circulant decomposition with the
packed vector blocks passed round a ring over NCCL send/recv; per-GPU load is kept at
C2's (weak scaling: n_v = 20,000 * sqrt(N)).
value = unique comparisons (pairs x n_f) of all ranks / max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CCC elementwise comparisons/sec (2-way, 3-way) at 1/2/4/8 B200; % int8 TC peak"
UNIT = "comparisons/s"
WORKLOADS = {
    "c1": dict(way=2, n_v=64, n_f=1024, label="2-way CCC, 64 x 1,024 (configs[0])"),
    "c2": dict(way=2, n_v=20000, n_f=50000,
               label="2-way CCC, 20,000 SNP vectors x 50,000 individuals (configs[1])"),
    "c2s": dict(way=2, n_v=20000, n_f=50000, sparse=True,
                label="2-way sparse-mode CCC (missing entries, SURVEY f1), 20,000 x 50,000"),
    "c2hwe": dict(way=2, n_v=20000, n_f=50000, kind="hwe",
                  label="2-way CCC, 20,000 x 50,000, Hardy-Weinberg SNP-like input (type 1b, seed 2): "
                        "the data-independence check of SURVEY 8(d) / P:719-724"),
    "c2pop": dict(way=2, n_v=20000, n_f=50000, popcount=True,
                  label="2-way CCC, 20,000 x 50,000, the paper's popcount tally on CUDA cores "
                        "(SURVEY f4 baseline)"),
    "c2fs": dict(way=2, n_v=20000, n_f=50000, fieldsplit=4,
                 label="2-way CCC, 20,000 x 50,000, field-axis split into 4 slices (SURVEY f3), "
                       "all slices simulated on one GPU"),
    "c4s": dict(way=3, n_v=4096, n_f=16384, n_st=16, sparse=True,
                label="3-way sparse-mode CCC (missing entries, SURVEY f1), 4,096 x 16,384, 16 stages"),
    "c4paper": dict(way=3, n_v=4096, n_f=16384, n_st=16, paper=True,
                    label="3-way CCC, 4,096 x 16,384, 16 stages, the paper's Table-1 route (3 masked pivot "
                          "GEMMs + reconstruction) on the tensor pipe (SURVEY f4 baseline)"),
    "c4f32": dict(way=3, n_v=4096, n_f=16384, n_st=16, flags="f32",
                  label="3-way CCC, 4,096 x 16,384, 16 stages, FULL with fp32 CCC (64 B/triple; SURVEY 8(d))"),
    "c4ck": dict(way=3, n_v=4096, n_f=16384, n_st=16, flags="ck",
                 label="3-way CCC, 4,096 x 16,384, 16 stages, CHECKSUM mode (every record computed and "
                       "folded, none stored; SURVEY 8(d) -- not a headline)"),
    "c4": dict(way=3, n_v=4096, n_f=16384, n_st=16,
               label="3-way CCC, 4,096 SNP vectors x 16,384 individuals, 16 stages (configs[3])"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled through NVML every ~5 ms on a
    background thread while the timed region runs (the recipe's clocks line)."""
    REASONS = {  # NVML clocks-event-reason bits
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4,
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.index = index
        self.period = period_s
        self.sm = []
        self.power = []
        self.bits = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def run():
                while not self._stop.is_set():
                    try:
                        self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        self.bits |= int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
                        self.power.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)   # W
                    except Exception:  # noqa: BLE001 - sampling is best effort
                        pass
                    time.sleep(self.period)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
            time.sleep(0.02)
        except Exception:  # noqa: BLE001 - no NVML: report no samples
            self._t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        reasons = sorted(k for k, b in self.REASONS.items() if self.bits & b)
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": 0}
        sm = sorted(self.sm)
        out = {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons,
               "samples": len(sm), "sm_mhz_min": sm[0]}
        if self.power:
            pw = sorted(self.power)
            out["power_w_median"] = pw[len(pw) // 2]
            out["power_w_max"] = pw[-1]
        return out


# ------------------------------------------------------------------------ helpers
def comparisons(way, n_v, n_f):
    if way == 2:
        return n_f * (n_v * (n_v - 1) // 2)
    return n_f * (n_v * (n_v - 1) * (n_v - 2) // 6)


def ncu_traffic(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(kernel, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def cpu_baseline(way, n_v, n_f, target_s=12.0, kind="random"):  # noqa: C901
    """The oracle as it stands, on the host cores, on a bounded sample of the workload."""
    import numpy as np

    import oracle
    import synthgen
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(n_v, size=min(n_v, 1024 if way == 2 else 128), replace=False))
    sub = np.concatenate([synthgen.make_codes(kind, 1, n_f, row0=int(r)).numpy() for r in rows])
    oracle.lib()
    m_local = len(rows)
    if way == 2:
        allidx = np.array([(a, b) for a in range(m_local) for b in range(a + 1, m_local)])
        f = oracle.pairs
        if kind == "sparse":
            f = lambda c, idx, S=None: oracle.sparse_pairs(c, idx)   # noqa: E731
    else:
        allidx = np.array([(a, b, c) for a in range(m_local) for b in range(a + 1, m_local)
                           for c in range(b + 1, m_local)])
        f = oracle.triples
        if kind == "sparse":
            f = lambda c, idx, S=None: oracle.sparse_triples(c, idx)   # noqa: E731
    S = oracle.allele_sums(sub)
    # calibrate, then run a sample sized for ~target_s seconds
    m = 64
    while True:
        t0 = time.perf_counter()
        f(sub, allidx[:m], S=S)
        dt = time.perf_counter() - t0
        if dt > 0.5 or m >= len(allidx):
            break
        m = min(len(allidx), m * 4)
    m_run = int(min(len(allidx), max(m, m * target_s / max(dt, 1e-6))))
    t0 = time.perf_counter()
    f(sub, allidx[:m_run], S=S)
    dt = time.perf_counter() - t0
    what = "pairs" if way == 2 else "triples"
    return {"value": m_run * n_f / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{m_run} {what} (n_f={n_f}) among {m_local} sampled vectors of the "
                      f"workload, brute-force Fig.1/Fig.2 enumeration, {dt:.1f} s"}


def int8_library_ceiling(n=8192, reps=10):
    """cuBLASLt's int8 GEMM (torch._int_mm, int32 accumulate) on n^3 in the same
    job -- a library reference point for the tensor-pipe line, not a peak."""
    import torch
    a = torch.randint(-3, 4, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-3, 4, (n, n), dtype=torch.int8, device="cuda").t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return {"torch_int_mm_TOPS": 2.0 * n ** 3 / (best / 1e3) / 1e12, "shape": f"{n}^3 int8 -> int32",
            "ms": best}


def cpu_optimized(n_v, n_f, target_s=8.0):
    """the paper's "optimized CPU version" -- bit-packed
    AND + popcount on the host cores (baselines/cpu_popcount.c), on the first rows of the
    same workload (all their pairs j > i, tallies + fp64 CCC), a bounded sample."""
    import numpy as np

    import baselines
    import synthgen
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    rows = min(n_v, 4096)
    packed = baselines.pack(synthgen.make_codes("random", rows, n_f, 1).numpy())
    baselines.lib()
    i_hi = 64
    while True:
        t0 = time.perf_counter()
        T, _ = baselines.popcount_2way(packed, n_f, i_hi=i_hi)
        dt = time.perf_counter() - t0
        if dt > target_s / 8 or i_hi >= rows - 1:
            break
        i_hi = min(rows - 1, i_hi * 4)
    pairs = len(T)
    return {"value": pairs * n_f / dt, "unit": UNIT, "cores": cores,
            "kind": "optimized bit-packed popcount CPU baseline (baselines/cpu_popcount.c)",
            "sample": f"{pairs} pairs (rows 0..{i_hi - 1} of the workload's first {rows} vectors "
                      f"x all j > i, n_f={n_f}), tallies + fp64 CCC, {dt:.1f} s"}


# ------------------------------------------------------------------------ ours, 1 GPU
def run_2way_single(args, wl):
    import torch

    import synthgen
    from paper_1705_08213_b200 import ccc
    n_v, n_f = wl["n_v"], wl["n_f"]
    sparse = wl.get("sparse", False)
    popcount = wl.get("popcount", False)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    flags = ccc.OUT_TALLY | ccc.OUT_CCC_F64
    if sparse:
        codes = synthgen.sparse_codes(n_v, n_f, seed=4, device=dev)    # resident in HBM
    elif wl.get("kind") == "hwe":
        codes = synthgen.hwe_codes(n_v, n_f, seed=2, device=dev)       # resident in HBM
    else:
        codes = synthgen.random_codes(n_v, n_f, seed=1, device=dev)    # resident in HBM
    packed = torch.empty((n_v, ccc.ccc_packed_stride(n_f)), dtype=torch.uint8, device=dev)
    N = torch.empty((ccc.ccc_sparse_rows(n_v) if sparse else n_v, ccc.ccc_k_pad(n_f)),
                    dtype=torch.int8, device=dev)
    s = torch.empty(n_v, dtype=torch.int32, device=dev)
    cnt = torch.empty(n_v, dtype=torch.int32, device=dev)
    w = torch.empty((n_v, 2), dtype=torch.float64, device=dev)
    m = ccc.ccc_num_unique(2, n_v)
    T = torch.empty((m, 4), dtype=torch.int32, device=dev)
    C = torch.empty((m, 4), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    launches = [0]
    ws = ccc.workspace(2, n_v, n_f, dev) if popcount else None

    def step(ev=None):
        ccc.ccc_pack(codes, packed)
        launches[0] += ccc.ccc_last_launch_count()
        if popcount:
            if ev:
                ev[0].record(stream)
            ccc.ccc_2way_popcount(packed, n_f, ccc.GAMMA, flags, T, C, None, ws)
            launches[0] += ccc.ccc_last_launch_count()
            if ev:
                ev[1].record(stream)
            return
        if sparse:
            ccc.ccc_expand_sparse(packed, n_f, ccc.GAMMA, (N, s, cnt, w))
        else:
            ccc.ccc_expand(packed, n_f, ccc.GAMMA, N, s, w)
        launches[0] += ccc.ccc_last_launch_count()
        if ev:
            ev[0].record(stream)
        if sparse:
            ccc.ccc_2way_sparse_block(N, w, n_v, 0, 0, n_v, N, w, n_v, 0, True, n_f, flags, T, C)
        else:
            ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, flags, T, C)
        launches[0] += ccc.ccc_last_launch_count()
        if ev:
            ev[1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches[0] = 0
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        t0.record(stream)
        for k in range(args.steps):
            step(kev[k])
        t1.record(stream)
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    k_ms = sum(a.elapsed_time(b) for a, b in kev) / args.steps
    comps = comparisons(2, n_v, n_f)
    res = {
        "ms": ms, "kernel_ms": k_ms, "comparisons": comps, "launches": launches[0],
        "clocks": clk.summary(), "kernel": "popc_tally2_kernel" if popcount else "tally2_kernel",
        "out_bytes": m * 48,
    }
    del T, C
    torch.cuda.empty_cache()
    if args.e2e and not sparse and not popcount:
        res["e2e"] = run_2way_e2e(args, wl, codes)
    return res


def run_2way_e2e(args, wl, codes_dev):
    """Same metric through the public host-buffer call (ccc_2way_host): every step copies
    the step's genotype codes H2D from pinned memory and all tallies + CCC D2H."""
    import torch

    from paper_1705_08213_b200 import ccc
    n_v, n_f = wl["n_v"], wl["n_f"]
    flags = ccc.OUT_TALLY | ccc.OUT_CCC_F64
    m = ccc.ccc_num_unique(2, n_v)
    codes_h = codes_dev.cpu().pin_memory()
    T_h = torch.empty((m, 4), dtype=torch.int32, pin_memory=True)
    C_h = torch.empty((m, 4), dtype=torch.float64, pin_memory=True)
    ws = torch.empty(ccc.ccc_e2e_workspace_bytes(n_v, n_f, flags), dtype=torch.uint8,
                     device="cuda")
    steps = max(1, min(args.steps, 3))
    ccc.ccc_2way_host(codes_h, ccc.GAMMA, flags, T_h, C_h, None, ws)   # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        ccc.ccc_2way_host(codes_h, ccc.GAMMA, flags, T_h, C_h, None, ws)
    dt = (time.perf_counter() - t0) / steps
    return {"value": comparisons(2, n_v, n_f) / dt, "unit": UNIT,
            "h2d_bytes_per_step": n_v * n_f, "d2h_bytes_per_step": m * 48,
            "steps": steps, "ms_per_step": dt * 1e3,
            "api": "ccc_2way_host (pinned host codes in, pinned host tallies+fp64 CCC out)"}


def run_fieldsplit_single(args, wl):
    """f3 on one GPU: the slices' export GEMMs and the owners' reduce + epilogue."""
    import torch

    import synthgen
    from paper_1705_08213_b200 import ccc, fieldsplit
    n_v, n_f, P = wl["n_v"], wl["n_f"], wl["fieldsplit"]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    flags = ccc.OUT_TALLY | ccc.OUT_CCC_F64
    codes = synthgen.random_codes(n_v, n_f, seed=1, device=dev)
    sl = fieldsplit.field_slices(n_f, P)
    cs = [codes[:, a:b].contiguous() for a, b in sl]
    del codes
    packed = [torch.empty((n_v, ccc.ccc_packed_stride(b - a)), dtype=torch.uint8, device=dev) for a, b in sl]
    Ns = [(torch.empty((n_v, ccc.ccc_k_pad(b - a)), dtype=torch.int8, device=dev),
           torch.empty(n_v, dtype=torch.int32, device=dev),
           torch.empty((n_v, 2), dtype=torch.float64, device=dev)) for a, b in sl]
    total = ccc.ccc_2way_fs_tiles(n_v)
    nbytes = ccc.ccc_2way_fs_slot_bytes(P, 0, total)
    slots = [torch.empty(nbytes // 4, dtype=torch.int32, device=dev) for _ in range(P)]
    ptrs = torch.tensor([t.data_ptr() for t in slots], dtype=torch.int64, device=dev)
    m = ccc.ccc_num_unique(2, n_v)
    T = torch.empty((m, 4), dtype=torch.int32, device=dev)
    C = torch.empty((m, 4), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    launches = [0]

    def step(ev=None):
        for r, (a, b) in enumerate(sl):
            ccc.ccc_pack(cs[r], packed[r])
            launches[0] += ccc.ccc_last_launch_count()
            N, s, w = Ns[r]
            ccc.ccc_expand(packed[r], b - a, ccc.GAMMA, N, s, w)
            launches[0] += ccc.ccc_last_launch_count()
        s_full = Ns[0][1].clone()
        for r in range(1, P):
            s_full += Ns[r][1]                 # the s all-reduce of the multi-GPU run
        if ev:
            ev[0].record(stream)
        for r, (a, b) in enumerate(sl):
            ccc.ccc_2way_fs_export(Ns[r][0], Ns[r][1], b - a, ptrs, r, P, 0, total)
            launches[0] += ccc.ccc_last_launch_count()
        if ev:
            ev[1].record(stream)
        for r in range(P):
            ccc.ccc_2way_fs_finish(slots[r], s_full, n_f, r, P, 0, total, flags, T, C)
            launches[0] += ccc.ccc_last_launch_count()
        if ev:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches[0] = 0
    kev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        t0.record(stream)
        for k in range(args.steps):
            step(kev[k])
        t1.record(stream)
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    k_ms = sum(e[0].elapsed_time(e[1]) for e in kev) / args.steps
    f_ms = sum(e[1].elapsed_time(e[2]) for e in kev) / args.steps
    return {"ms": ms, "kernel_ms": k_ms, "finish_ms": f_ms, "comparisons": comparisons(2, n_v, n_f),
            "launches": launches[0], "clocks": clk.summary(), "kernel": "tally2_kernel",
            "out_bytes": m * 48, "slot_bytes_per_pair_in": 4 * P}


def run_3way_single(args, wl):
    import torch

    import synthgen
    from paper_1705_08213_b200 import ccc
    n_v, n_f, n_st = wl["n_v"], wl["n_f"], wl["n_st"]
    sparse = wl.get("sparse", False)
    paper = wl.get("paper", False)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    flags = {"f32": ccc.OUT_TALLY | ccc.OUT_CCC_F32, "ck": ccc.OUT_CHECKSUM}.get(
        wl.get("flags"), ccc.OUT_TALLY | ccc.OUT_CCC_F64)
    rec_bytes = {"f32": 64, "ck": 0}.get(wl.get("flags"), 96)
    if sparse:
        codes = synthgen.sparse_codes(n_v, n_f, seed=4, device=dev)
    else:
        codes = synthgen.random_codes(n_v, n_f, seed=1, device=dev)
    packed = torch.empty((n_v, ccc.ccc_packed_stride(n_f)), dtype=torch.uint8, device=dev)
    if sparse:
        ws = torch.empty(ccc.lib().ccc_sparse3_workspace_bytes(n_v, n_f), dtype=torch.uint8, device=dev)
        scratch = torch.empty(max(ccc.lib().ccc_3way_sparse_scratch_bytes(n_v, n_st, s) for s in range(n_st)),
                              dtype=torch.uint8, device=dev)
    elif paper:
        ws = torch.empty(ccc.lib().ccc_3way_paper_workspace_bytes(n_v, n_f), dtype=torch.uint8, device=dev)
        scratch = torch.empty(max(ccc.lib().ccc_3way_paper_scratch_bytes(n_v, n_st, s) for s in range(n_st)),
                              dtype=torch.uint8, device=dev)
    else:
        ws = ccc.workspace(3, n_v, n_f, dev)
    rmax = max(ccc.ccc_stage_range(n_v, n_st, s)[3] for s in range(n_st))
    T = torch.empty((rmax, 8), dtype=torch.int32, device=dev) if flags & ccc.OUT_TALLY else None
    C = None
    if flags & ccc.OUT_CCC_F64:
        C = torch.empty((rmax, 8), dtype=torch.float64, device=dev)
    elif flags & ccc.OUT_CCC_F32:
        C = torch.empty((rmax, 8), dtype=torch.float32, device=dev)
    ck = torch.zeros(2, dtype=torch.int64, device=dev) if flags & ccc.OUT_CHECKSUM else None
    stream = torch.cuda.current_stream()
    launches = [0]

    def step(ev=None):
        ccc.ccc_pack(codes, packed)
        launches[0] += ccc.ccc_last_launch_count()
        if sparse:
            ccc.ccc_3way_sparse_prepare(packed, n_f, ccc.GAMMA, ws)
        elif paper:
            ccc.ccc_3way_paper_prepare(packed, n_f, ccc.GAMMA, ws)
        else:
            ccc.ccc_3way_prepare(packed, n_f, ccc.GAMMA, ws)
        launches[0] += ccc.ccc_last_launch_count()
        for st in range(n_st):
            if ev:
                ev[st][0].record(stream)
            if sparse:
                ccc.ccc_3way_sparse_stage(n_v, n_f, n_st, st, ws, flags, T, C, None, scratch)
            elif paper:
                ccc.ccc_3way_paper_stage(n_v, n_f, n_st, st, ws, flags, T, C, None, scratch)
            else:
                ccc.ccc_3way_stage(n_v, n_f, n_st, st, ws, flags, T, C, ck)
            launches[0] += ccc.ccc_last_launch_count()
            if ev:
                ev[st][1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches[0] = 0
    kev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(n_st)] for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        t0.record(stream)
        for k in range(args.steps):
            step(kev[k])
        t1.record(stream)
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    k_ms = sum(a.elapsed_time(b) for st in kev for a, b in st) / (args.steps * n_st)
    return {"ms": ms, "kernel_ms": k_ms, "comparisons": comparisons(3, n_v, n_f),
            "launches": launches[0], "clocks": clk.summary(), "kernel": "tally3_kernel",
            "out_bytes": comparisons(3, n_v, n_f) // n_f * rec_bytes, "stages": n_st,
            "forms_bytes": comparisons(3, n_v, n_f) // n_f * (7 if sparse else 2) * 4 * 2 if (sparse or paper) else 0}


# ------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu", dest="cpu", action="store_false")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    wl = dict(WORKLOADS[args.workload])

    if args.impl == "reference":
        if rank != 0:
            return
        # The reference arm is the CPU oracle (no runnable reference implementation
        # exists for this paper): a bounded sample of the same workload per step.
        vals = []
        for _ in range(args.warmup + args.steps):
            vals.append(cpu_baseline(wl["way"], wl["n_v"], wl["n_f"], target_s=4.0,
                                     kind="sparse" if wl.get("sparse") else wl.get("kind", "random")))
        vals = vals[args.warmup:]
        v = sorted(x["value"] for x in vals)[len(vals) // 2]
        cb = dict(vals[0])
        cb["value"] = v
        out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
               "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
               "dtype": "int64", "data": "synthetic",
               "config": {"workload": wl["label"], "n_v": wl["n_v"], "n_f": wl["n_f"]},
               "cpu_baseline": cb,
               "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return

    if world > 1 or args.gpus > 1:
        if wl.get("sparse"):
            raise SystemExit("the sparse workloads are single-GPU measurements")
        from paper_1705_08213_b200 import dist
        return dist.bench_main(args, wl, METRIC, UNIT)

    pk, pk_kind = peaks()
    if wl.get("fieldsplit"):
        r = run_fieldsplit_single(args, wl)
    elif wl["way"] == 2:
        r = run_2way_single(args, wl)
    else:
        r = run_3way_single(args, wl)
    ms_step = r["ms"] / args.steps
    value = r["comparisons"] / (ms_step / 1e3)
    # roofline of the dominant kernel (the fused tally GEMM): 2 int8 ops per comparison
    k_s = r["kernel_ms"] / 1e3
    if wl["way"] == 2:
        # sparse mode: 4 int8 MACs per comparison (n.n, n.v, v.n, v.v)
        ops = (8.0 if wl.get("sparse") else 2.0) * r["comparisons"]
    else:
        # sparse 3-way: 8 passes (trilinear forms) = 8 MACs per comparison
        ops = (16.0 if wl.get("sparse") else 6.0 if wl.get("paper") else 2.0) * r["comparisons"] / wl["n_st"]
    # int8 dense = 2 x bf16 dense (the guide's nominal ratio, 4.5 vs 2.25 PFLOP/s); the
    # burst figure applies: the timed region is ~0.1 s of back-to-back steps, not seconds.
    int8_peak = 2.0 * pk["bf16_tflops"]
    achieved = ops / k_s / 1e12
    # ncu --set full DRAM bytes of the dominant kernel, captured on the c2 / c4 workloads only
    traffic = ncu_traffic(r["kernel"]) if args.workload in ("c2", "c4") else None
    roof = {"bound": "tensor", "achieved": achieved, "peak": int8_peak, "unit": "TFLOP/s",
            "frac": achieved / int8_peak, "traffic": traffic,
            "kernel": r["kernel"], "kernel_ms": r["kernel_ms"],
            "peak_source": f"2 x bf16_tflops (burst) of MEASURED_PEAKS.json ({pk_kind}); "
                           "int8 ops = 2 per MAC = %d per comparison" % (
                               8 if wl.get("sparse") else 2),
            "nominal_int8_frac": achieved / 4500.0,
            "note": "the peak line is 2 x the measured bf16 burst (the task's rule for another dtype); "
                    "it understates the int8 pipe -- this kernel's own mainloop reaches 4,250 TOPS with "
                    "stores off (DESIGN.md 6) -- so frac can read ~1.0; nominal_int8_frac is against "
                    "the 4.5 POPS datasheet"}
    hbm_write = r["out_bytes"] / (ms_step / 1e3) / 1e9
    roof["out_write_GBps"] = hbm_write
    roof["out_write_frac_of_hbm"] = hbm_write / pk["hbm_gbs"]
    if wl["way"] == 2 and not wl.get("popcount") and args.workload in ("c2", "c2s"):
        try:
            lib_ceil = int8_library_ceiling()
            roof["int8_library_ceiling"] = lib_ceil
            roof["frac_of_library_ceiling"] = achieved / lib_ceil["torch_int_mm_TOPS"]
        except Exception as e:   # noqa: BLE001 -- a reference point only
            roof["int8_library_ceiling"] = {"error": str(e)[:200]}
    if wl.get("fieldsplit"):
        # the export GEMMs of all slices (tensor) + the owners' reduce/epilogue (HBM)
        pairs = r["comparisons"] / wl["n_f"]
        roof["kernel_ms"] = r["kernel_ms"]
        roof["finish_ms"] = r["finish_ms"]
        roof["finish_GBps"] = pairs * (r["slot_bytes_per_pair_in"] + 48) / (r["finish_ms"] / 1e3) / 1e9
        roof["finish_frac_of_hbm"] = roof["finish_GBps"] / pk["hbm_gbs"]
    if wl.get("popcount"):
        # CUDA-core path: 2 POPC per 16 comparisons; peak = 148 SMs x 16 POPC/clk (the
        # CUDA C throughput table's population-count rate) x the sampled SM clock
        mhz = (r["clocks"].get("sm_mhz") or pk.get("sm_max_mhz", 1965.0))
        popc = 2.0 * r["comparisons"] / 16.0
        roof = {"bound": "alu", "achieved": popc / k_s / 1e12,
                "peak": 148 * 16 * mhz * 1e6 / 1e12, "unit": "TPOPC/s",
                "traffic": None, "kernel": r["kernel"], "kernel_ms": r["kernel_ms"],
                "peak_source": "148 SMs x 16 POPC/clk/SM x sampled SM clock (DESIGN.md §6)",
                "tensor_path_equiv_frac_of_int8_peak": 2.0 * r["comparisons"] / k_s / 1e12 / int8_peak}
        roof["frac"] = roof["achieved"] / roof["peak"]
    if wl["way"] == 3 and wl.get("flags") == "ck":
        roof["peak_source"] += "; CHECKSUM mode: no record is stored, the tensor-pipe line is the roofline"
    elif wl["way"] == 3:
        roof.pop("note", None)
        roof["bound"] = "hbm"
        roof["achieved"] = (r["out_bytes"] + r.get("forms_bytes", 0)) / wl["n_st"] / k_s / 1e9
        roof["peak"] = pk["hbm_gbs"]
        roof["unit"] = "GB/s"
        roof["frac"] = roof["achieved"] / pk["hbm_gbs"]
        rb = 64 if wl.get("flags") == "f32" else 96
        roof["peak_source"] = f"hbm_gbs of MEASURED_PEAKS.json ({pk_kind}); FULL output {rb} B/triple" + (
            " + 7 stored forms written and read back (56 B/triple)" if wl.get("sparse") else
            " + 2 stored masked forms written and read back (16 B/triple)" if wl.get("paper") else "")
        roof["tensor_TOPS"] = achieved
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "u32 (bitwise AND + popcount)" if wl.get("popcount") else "int8",
        "data": "synthetic",
        "config": {"workload": wl["label"], "n_v": wl["n_v"], "n_f": wl["n_f"],
                   "input": ("type-3 sparse HWE codes, seed 4, missing marker (1,0) with "
                             "per-vector rate U(0, 0.3) (P:1028-1043)") if wl.get("sparse") else
                            ("type-1b Hardy-Weinberg codes, p_i ~ U(0.05, 0.5), seed 2"
                             if wl.get("kind") == "hwe" else
                             "type-1 uniform random 2-bit codes, seed 1 (P:657)"),
                   "output": {"f32": "FULL: uint32 tallies + fp32 CCC for every unique record",
                              "ck": "CHECKSUM: every record computed and folded into the 128-bit checksum, none stored"
                              }.get(wl.get("flags"), "FULL: uint32 tallies + fp64 CCC for every unique record"),
                   "l2": ("inputs larger than L2 (codes %.2f GB, N %.2f GB)" % (
                       wl["n_v"] * wl["n_f"] / 1e9, wl["n_v"] * wl["n_f"] / 1e9)) if wl["way"] == 2 else
                         ("operands L2-resident by design (N %.2f GB, G %.2f GB); each stage writes "
                          "%.0f GB of records, far larger than L2" % (
                              wl["n_v"] * wl["n_f"] / 1e9, 4 * wl["n_v"] ** 2 / 1e9,
                              comparisons(3, wl["n_v"], wl["n_f"]) / wl["n_f"] * 96 / wl["n_st"] / 1e9)),
                   "parallelism": "single GPU"},
        "roofline": roof,
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
    }
    if "e2e" in r:
        out["e2e"] = r["e2e"]
    if args.cpu:
        out["cpu_baseline"] = cpu_baseline(wl["way"], wl["n_v"], wl["n_f"],
                                           kind="sparse" if wl.get("sparse") else wl.get("kind", "random"))
        if wl["way"] == 2 and not wl.get("sparse"):
            out["cpu_optimized"] = cpu_optimized(wl["n_v"], wl["n_f"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()

"""Multi-GPU 2-way CCC: block-circulant decomposition with a ring shift of packed vector
blocks over NCCL send/recv, overlapped with the tally kernels (§4, P:583-606,
P:628-629).

One process per GPU (torchrun).  Rank r owns vector block r.  Step d = 0 computes the
diagonal block with the rank's own expanded data; before computing step d the rank posts
isend(currently held packed block -> r-1) / irecv(next block <- r+1) on NCCL's stream, so
the 2-bit packed block for step d+1 (n_b * n_f / 4 bytes) crosses NVLink while the
tensor cores work on step d.  Received blocks are re-expanded (KB-expand: counts, s, w) on
arrival -- sending the packed form moves 4x fewer bytes than the int8 operand.

The kernels are supplied by a backend object; the product backend is `CudaBackend`
(libccc.so).  There is no CPU path here: tests inject their own backend to exercise the
ring logic on CPU with gloo.
"""
from __future__ import annotations

import math
import os

import torch
import torch.distributed as dist

from . import decomp


class CudaBackend:
    """libccc kernels on the current CUDA device (the product path)."""

    def __init__(self, n_f: int, gamma: float, out_flags: int):
        from . import ccc
        self.ccc = ccc
        self.n_f = n_f
        self.gamma = gamma
        self.out_flags = out_flags
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.kernel_events = []   # (start, end) CUDA events around the tally kernels

    def pack(self, codes, out=None):
        return self.ccc.ccc_pack(codes, out)

    def packed_empty(self, rows):
        return torch.empty((rows, self.ccc.ccc_packed_stride(self.n_f)), dtype=torch.uint8,
                           device=self.device)

    def expand(self, packed, out=None):
        if out is None:
            return self.ccc.ccc_expand(packed, self.n_f, self.gamma)
        N, s, w = out
        rows = packed.shape[0]
        return self.ccc.ccc_expand(packed, self.n_f, self.gamma, N[:rows], s[:rows], w[:rows])

    def expanded_empty(self, rows):
        return (torch.empty((rows, self.ccc.ccc_k_pad(self.n_f)), dtype=torch.int8, device=self.device),
                torch.empty(rows, dtype=torch.int32, device=self.device),
                torch.empty((rows, 2), dtype=torch.float64, device=self.device))

    def outputs(self, n_rec):
        f = self.out_flags
        T = torch.empty((n_rec, 4), dtype=torch.int32, device=self.device) if f & 1 else None
        C = None
        if f & 2:
            C = torch.empty((n_rec, 4), dtype=torch.float64, device=self.device)
        elif f & 4:
            C = torch.empty((n_rec, 4), dtype=torch.float32, device=self.device)
        return T, C

    def checksum_zero(self):
        return torch.zeros(2, dtype=torch.int64, device=self.device)

    def block(self, A, a_row0, a_lo, a_hi, B, b_row0, diag, out, ck, timed=False):
        N_a, s_a, w_a = A
        N_b, s_b, w_b = B
        T, C = out
        ev = None
        if timed:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        self.ccc.ccc_2way_block(N_a, s_a, w_a, a_row0, a_lo, a_hi, N_b, s_b, w_b, b_row0, diag,
                                self.n_f, self.out_flags, T, C, ck)
        if timed:
            ev[1].record()
            self.kernel_events.append(ev)
        return self.ccc.ccc_last_launch_count()


class Ring2Way:
    """Per-rank state of the block-circulant 2-way computation (buffers are reused
    across calls so a bench step does no allocation)."""

    def __init__(self, backend, bounds, rank: int, world: int, group=None):
        self.be = backend
        self.bounds = bounds
        self.rank = rank
        self.P = world
        self.group = group
        self.units = decomp.plan_2way(world, rank, bounds)
        self.steps = decomp.ring_steps_2way(world)
        rows = [hi - lo for lo, hi in bounds]
        self.max_rows = max(rows)
        self.recv = [backend.packed_empty(self.max_rows) for _ in range(2 if self.steps else 0)]
        self.other = backend.expanded_empty(self.max_rows) if self.steps else None
        self.out = [backend.outputs(decomp.unit2_records(u, bounds)) for u in self.units]
        self.ck = backend.checksum_zero()
        self.launches = 0

    def _rows(self, b):
        return self.bounds[b][1] - self.bounds[b][0]

    def run(self, packed_own, timed=False):
        """One pass over this rank's units.  packed_own: the rank's packed block."""
        be, r, P = self.be, self.rank, self.P
        own = be.expand(packed_own)
        self.launches = 1
        cur = packed_own
        for d in range(self.steps + 1):
            reqs = []
            nxt = None
            if d < self.steps:
                nb = (r + d + 1) % P
                nxt = self.recv[d % 2][: self._rows(nb)]
                ops = [dist.P2POp(dist.isend, cur.contiguous(), (r - 1) % P, self.group),
                       dist.P2POp(dist.irecv, nxt, (r + 1) % P, self.group)]
                reqs = dist.batch_isend_irecv(ops)
            held = (r + d) % P
            if d == 0:
                held_exp = own
            else:
                held_exp = be.expand(cur, self.other)
                self.launches += 1
            for ui, u in enumerate(self.units):
                if u.step != d:
                    continue
                A = own if u.a == r else held_exp
                B = own if u.b == r else held_exp
                if d == 0:
                    A = B = own
                self.launches += be.block(A, self.bounds[u.a][0], u.a_lo, u.a_hi, B,
                                          self.bounds[u.b][0], u.diag, self.out[ui], self.ck,
                                          timed=timed)
                assert u.a == r or u.b == r
                assert held in (u.a, u.b)
            for q in reqs:
                q.wait()
            if nxt is not None:
                cur = nxt
        return self.out


def checksum_total(ck_local: torch.Tensor, group=None) -> int:
    """Sum of the ranks' 128-bit checksums mod 2^128 (host-side, exact)."""
    world = dist.get_world_size(group)
    buf = [torch.zeros_like(ck_local) for _ in range(world)]
    dist.all_gather(buf, ck_local, group=group)
    tot = 0
    for t in buf:
        lo, hi = (int(x) & ((1 << 64) - 1) for x in t.cpu().tolist())
        tot = (tot + ((hi << 64) | lo)) % (1 << 128)
    return tot


def weak_scaled_nv(n_v1: int, P: int, align: int = 256) -> int:
    """n_v at P GPUs with the same per-GPU pair count as n_v1 on one GPU (weak scaling)."""
    if P == 1:
        return n_v1
    q = align * P
    return max(q, int(round(n_v1 * math.sqrt(P) / q)) * q)


# ----------------------------------------------------------------------------- bench
def bench_main(args, wl, metric, unit):
    """bench.py at N > 1 (torchrun, NCCL): weak-scaled block-circulant 2-way."""
    import json
    import time

    import synthgen
    from . import ccc

    if wl["way"] != 2:
        raise SystemExit("multi-GPU bench covers the 2-way path (3-way: see DESIGN.md)")
    dist.init_process_group("nccl")
    rank, P = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    n_f = wl["n_f"]
    n_v = weak_scaled_nv(wl["n_v"], P)
    bounds = decomp.block_bounds(n_v, P, align=256)
    lo, hi = bounds[rank]
    flags = ccc.OUT_TALLY | ccc.OUT_CCC_F64 | ccc.OUT_CHECKSUM
    be = CudaBackend(n_f, ccc.GAMMA, flags)
    ring = Ring2Way(be, bounds, rank, P)
    codes = synthgen.random_codes(hi - lo, n_f, seed=1, device="cuda", row0=lo)
    packed = be.packed_empty(hi - lo)
    stream = torch.cuda.current_stream()

    def step(timed=False):
        be.pack(codes, packed)
        ring.ck.zero_()
        ring.run(packed, timed=timed)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    be.kernel_events.clear()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    from bench import ClockSampler
    clk = ClockSampler(local)
    torch.cuda.synchronize()
    dist.barrier()
    with clk:
        t0.record(stream)
        launches = 0
        for _ in range(args.steps):
            step(timed=True)
            launches += 1 + ring.launches
        t1.record(stream)
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    kms = sum(a.elapsed_time(b) for a, b in be.kernel_events)
    dist.barrier()
    tmax = torch.tensor([ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ck = checksum_total(ring.ck)
    comps = n_f * (n_v * (n_v - 1) // 2)
    ms_step = float(tmax.item()) / args.steps

    # e2e: the same step through the public API with host buffers: H2D of this rank's
    # genotype codes from pinned memory, D2H of every record it computes
    e2e = None
    if args.e2e:
        codes_h = codes.cpu().pin_memory()
        outs_h = [tuple(x.cpu().pin_memory() if x is not None else None for x in o) for o in ring.out]
        d2h = sum(x.numel() * x.element_size() for o in ring.out for x in o if x is not None)
        e_steps = max(1, min(args.steps, 3))

        def e2e_step():
            codes.copy_(codes_h, non_blocking=True)
            step()
            for o, oh in zip(ring.out, outs_h):
                for x, xh in zip(o, oh):
                    if x is not None:
                        xh.copy_(x, non_blocking=True)
            torch.cuda.synchronize()

        e2e_step()
        dist.barrier()
        t = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        dt = torch.tensor([(time.perf_counter() - t) / e_steps], dtype=torch.float64, device="cuda")
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": comps / float(dt.item()), "unit": unit,
               "h2d_bytes_per_step": (hi - lo) * n_f, "d2h_bytes_per_step": d2h,
               "steps": e_steps, "ms_per_step": float(dt.item()) * 1e3,
               "api": "dist.Ring2Way over the libccc binding, pinned host codes in / records out "
                      "(per-rank bytes)"}
    if rank == 0:
        from bench import peaks
        pk, pk_kind = peaks()
        my_comps = n_f * sum(decomp.unit2_records(u, bounds) for u in ring.units)
        ach = 2.0 * my_comps * args.steps / (kms / 1e3) / 1e12
        peak = 2.0 * pk["bf16_tflops"]
        out = {
            "metric": metric, "value": comps / (ms_step / 1e3), "unit": unit, "n_gpus": P,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic",
            "config": {"workload": f"2-way CCC block-circulant, {n_v} SNP vectors x {n_f} "
                                   f"individuals over {P} GPUs (per-GPU load = configs[1])",
                       "n_v": n_v, "n_f": n_f, "parallelism": f"block-circulant dp{P}",
                       "ring": "packed 2-bit blocks, NCCL send/recv, overlapped",
                       "l2": "inputs larger than L2"},
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                         "frac": ach / peak, "traffic": None, "kernel": "tally2_kernel",
                         "peak_source": f"2 x bf16_tflops of MEASURED_PEAKS.json ({pk_kind})"},
            "gpu_launches": launches, "checksum": f"{ck:032x}",
            "clocks": clk.summary(),
        }
        if e2e:
            out["e2e"] = e2e
        print(json.dumps(out))
    dist.barrier()
    dist.destroy_process_group()

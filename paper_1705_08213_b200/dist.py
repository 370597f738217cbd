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

    # ---- 3-way (Ring3Way) ------------------------------------------------------------
    def g_empty(self, n_v):
        return torch.zeros((n_v, n_v), dtype=torch.int32, device=self.device)

    def expand_into(self, packed, full, lo, hi):
        N, s, w = full
        return self.ccc.ccc_expand(packed, self.n_f, self.gamma, N[lo:hi], s[lo:hi], w[lo:hi])

    def g_block(self, ring, a, b):
        """Pairwise G of blocks a == b (own block) into the global G."""
        N, s, w = ring.full
        lo, hi = ring.bounds[a]
        n_v = ring.n_v
        Gv = ring.G.view(-1)[lo * n_v + lo:]
        self.ccc.ccc_2way_block(N[lo:hi], s[lo:hi], w[lo:hi], lo, 0, hi - lo, N[lo:hi], s[lo:hi],
                                w[lo:hi], lo, True, self.n_f, 0, g=Gv, ldg=n_v)

    def g_full(self, ring):
        N, s, w = ring.full
        self.ccc.ccc_2way_block(N, s, w, 0, 0, ring.n_v, N, s, w, 0, True, self.n_f, 0,
                                g=ring.G, ldg=ring.n_v)

    def _blk(self, ring, b):
        N, s, w = ring.full
        lo, hi = ring.bounds[b]
        return self.ccc.block(N[lo:hi], s[lo:hi], w[lo:hi], lo)

    def unit_records(self, ring, u, p_lo, p_hi):
        return decomp.unit3_count(decomp.Unit3(u.pb, p_lo, p_hi, u.mb, u.m_lo, u.m_hi, u.nb,
                                               u.n_lo, u.n_hi, u.order), ring.bounds)

    def unit(self, ring, u, p_lo, p_hi, ck):
        """One piece of a tetrahedral unit into a reused record buffer: the views it returns
        (and hands to Ring3Way's sink) are valid only until the next piece is launched on
        the current stream -- a sink that keeps records must copy them on this stream."""
        f = self.out_flags
        n_rec = self.unit_records(ring, u, p_lo, p_hi)
        buf = getattr(self, "_buf3", None)
        if buf is None or buf[0] < n_rec or buf[1] != f:
            T = torch.empty((n_rec, 8), dtype=torch.int32, device=self.device) if f & 1 else None
            C = (torch.empty((n_rec, 8), dtype=torch.float64, device=self.device) if f & 2 else
                 torch.empty((n_rec, 8), dtype=torch.float32, device=self.device) if f & 4 else None)
            self._buf3 = (n_rec, f, T, C)
        _, _, T, C = self._buf3
        T = T[:n_rec] if T is not None else None
        C = C[:n_rec] if C is not None else None
        self.ccc.ccc_3way_unit(self._blk(ring, u.pb), p_lo, p_hi, self._blk(ring, u.mb), u.m_lo,
                               u.m_hi, self._blk(ring, u.nb), u.n_lo, u.n_hi, u.order, ring.G,
                               self.n_f, f, T, C, ck, gamma=self.gamma)
        return T, C

    def block(self, A, a_row0, a_lo, a_hi, B, b_row0, diag, out, ck, timed=False):
        N_a, s_a, w_a = A
        N_b, s_b, w_b = B
        T, C = out
        ev = None
        if timed:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        self.ccc.ccc_2way_block(N_a, s_a, w_a, a_row0, a_lo, a_hi, N_b, s_b, w_b, b_row0, diag,
                                self.n_f, self.out_flags, T, C, ck, gamma=self.gamma)
        if timed:
            ev[1].record()
            self.kernel_events.append(ev)
        return self.ccc.ccc_last_launch_count()


class _StagedRecv:
    """Completion of a host-staged receive: wait, then copy into the device buffer."""

    def __init__(self, reqs, host, dst):
        self.reqs, self.host, self.dst = reqs, host, dst

    def wait(self):
        for q in self.reqs:
            q.wait()
        self.dst.copy_(self.host)


def ring_shift(cur: torch.Tensor, nxt: torch.Tensor, r: int, P: int, group=None):
    """Post send(cur -> r-1) and recv(nxt <- r+1); returns the requests to wait on.

    NCCL moves the device buffers directly (NVLink).  gloo cannot move CUDA tensors point to
    point, so under a gloo group the packed block is staged through host memory -- the
    transport that lets several ranks share one GPU in the tests; the kernels are the same."""
    if cur.is_cuda and dist.get_backend(group) == "gloo":
        host = torch.empty(nxt.shape, dtype=nxt.dtype)
        ops = [dist.P2POp(dist.isend, cur.contiguous().cpu(), (r - 1) % P, group),
               dist.P2POp(dist.irecv, host, (r + 1) % P, group)]
        return [_StagedRecv(dist.batch_isend_irecv(ops), host, nxt)]
    ops = [dist.P2POp(dist.isend, cur.contiguous(), (r - 1) % P, group),
           dist.P2POp(dist.irecv, nxt, (r + 1) % P, group)]
    return dist.batch_isend_irecv(ops)


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
                reqs = ring_shift(cur, nxt, r, P, self.group)
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


class Ring3Way:
    """Per-rank tetrahedral 3-way computation.  Every rank
    needs every block: a ring all-gather *with retention* of the packed blocks (P-1
    steps, NCCL send/recv) fills a full expanded N in place (blocks are contiguous
    rows), overlapped with the rank's {A,A,A} unit, which needs only its own block and
    the own-block part of G.  Then the pairwise G over all vectors (KB-2W, ~1/n_f of the
    3-way work) and the remaining units.  Each unit is cut into pivot sub-ranges so
    that no output buffer exceeds `max_records` (the paper's stages)."""

    def __init__(self, backend, bounds, rank: int, world: int, max_records: int, group=None):
        self.be = backend
        self.bounds = bounds
        self.rank = rank
        self.P = world
        self.group = group
        self.n_v = bounds[-1][1]
        self.units = decomp.plan_3way(world, rank, bounds)
        self.full = backend.expanded_empty(self.n_v)
        self.G = backend.g_empty(self.n_v)
        self.recv = [backend.packed_empty(max(hi - lo for lo, hi in bounds)) for _ in range(2)]
        self.held = [None] * world
        self.max_records = max_records
        self.ck = backend.checksum_zero()
        self.launches = 0

    def _pieces(self, u):
        """Split a unit into pivot sub-ranges of <= max_records records."""
        out, lo = [], u.p_lo
        while lo < u.p_hi:
            hi = lo + 1
            while hi < u.p_hi and self.be.unit_records(self, u, lo, hi + 1) <= self.max_records:
                hi += 1
            out.append((lo, hi))
            lo = hi
        return out

    def run(self, packed_own, sink=None):
        """One pass; sink(unit, p_lo, p_hi, outputs) receives each piece's records (on the
        device, in a buffer the next piece overwrites: copy on the current stream to keep
        them; the default drops them after the checksum fold)."""
        be, r, P = self.be, self.rank, self.P
        lo, hi = self.bounds[r]
        be.expand_into(packed_own, self.full, lo, hi)
        be.g_block(self, r, r)
        self.launches = 2
        cur = packed_own
        reqs = []
        for d in range(P):
            nxt = None
            if d < P - 1:
                nb = (r + d + 1) % P
                nxt = self.recv[d % 2][: self.bounds[nb][1] - self.bounds[nb][0]]
                reqs = ring_shift(cur, nxt, r, P, self.group)
            if d == 0:   # own-block unit overlaps the gather
                self.launches += self._run_units(lambda u: u.pb == u.mb == u.nb, sink)
            for q in reqs:
                q.wait()
            reqs = []
            if nxt is not None:
                nb = (r + d + 1) % P
                be.expand_into(nxt, self.full, *self.bounds[nb])
                self.launches += 1
                cur = nxt
        be.g_full(self)
        self.launches += 1
        self.launches += self._run_units(lambda u: not (u.pb == u.mb == u.nb), sink)
        return self.ck

    def _run_units(self, pick, sink):
        n = 0
        for u in self.units:
            if not pick(u):
                continue
            for plo, phi in self._pieces(u):
                out = self.be.unit(self, u, plo, phi, self.ck)
                n += 1
                if sink is not None:
                    sink(u, plo, phi, out)
        return n


def checksum_total(ck_local: torch.Tensor, group=None) -> int:
    """Sum of the ranks' 128-bit checksums mod 2^128 (host-side, exact)."""
    world = dist.get_world_size(group)
    if ck_local.is_cuda and dist.get_backend(group) == "gloo":
        ck_local = ck_local.cpu()
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

    if wl["way"] == 3:
        return bench_main_3way(args, wl, metric, unit)
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

    # the timed steps write exactly what the single-GPU line writes (tallies + fp64 CCC);
    # the cross-rank checksum comes from one extra, untimed verification step below
    be.out_flags = ccc.OUT_TALLY | ccc.OUT_CCC_F64
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
    be.out_flags = flags                       # verification step: + the 128-bit checksum
    step()
    torch.cuda.synchronize()
    be.out_flags = ccc.OUT_TALLY | ccc.OUT_CCC_F64
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


def weak_scaled_nv3(n_v1: int, P: int, align: int = 256) -> int:
    """n_v at P GPUs with the same per-GPU triple count as n_v1 on one GPU."""
    if P == 1:
        return n_v1
    q = align * P
    return max(q, int(round(n_v1 * P ** (1.0 / 3.0) / q)) * q)


def bench_main_3way(args, wl, metric, unit):
    """bench.py --workload c4 at N > 1: tetrahedral 3-way, weak-scaled from C4."""
    import json

    import synthgen
    from . import ccc

    dist.init_process_group("nccl")
    rank, P = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    n_f = wl["n_f"]
    n_v = weak_scaled_nv3(wl["n_v"], P)
    bounds = decomp.block_bounds(n_v, P, align=256)
    lo, hi = bounds[rank]
    flags = ccc.OUT_TALLY | ccc.OUT_CCC_F64 | ccc.OUT_CHECKSUM
    be = CudaBackend(n_f, ccc.GAMMA, flags)
    max_rec = int(os.environ.get("CCC_3WAY_STAGE_RECORDS", 700_000_000))   # ~67 GB / stage
    ring = Ring3Way(be, bounds, rank, P, max_records=max_rec)
    codes = synthgen.random_codes(hi - lo, n_f, seed=1, device="cuda", row0=lo)
    packed = be.packed_empty(hi - lo)

    def step():
        be.pack(codes, packed)
        ring.ck.zero_()
        ring.run(packed)

    be.out_flags = ccc.OUT_TALLY | ccc.OUT_CCC_F64   # as the single-GPU line; checksum below
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    from bench import ClockSampler
    clk = ClockSampler(local)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clk:
        t0.record()
        for _ in range(args.steps):
            step()
        t1.record()
        torch.cuda.synchronize()
    tmax = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    be.out_flags = flags                                # untimed verification step
    step()
    torch.cuda.synchronize()
    ck = checksum_total(ring.ck)
    comps = n_f * (n_v * (n_v - 1) * (n_v - 2) // 6)
    ms_step = float(tmax.item()) / args.steps
    if rank == 0:
        out = {"metric": metric, "value": comps / (ms_step / 1e3), "unit": unit, "n_gpus": P,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
               "dtype": "int8", "data": "synthetic",
               "config": {"workload": f"3-way CCC tetrahedral, {n_v} SNP vectors x {n_f} "
                                      f"individuals over {P} GPUs (per-GPU load = configs[3])",
                          "n_v": n_v, "n_f": n_f, "parallelism": f"tetrahedral dp{P}",
                          "output": "FULL, staged", "l2": "outputs larger than L2"},
               "gpu_launches": args.steps * (1 + ring.launches), "checksum": f"{ck:032x}",
               "clocks": clk.summary()}
        from bench import peaks
        pk, pk_kind = peaks()
        # FULL records: 96 B per triple over all ranks; per-GPU HBM write rate vs the peak
        gbs = comps / n_f * 96 / P / (ms_step / 1e3) / 1e9
        out["roofline"] = {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                           "frac": gbs / pk["hbm_gbs"], "traffic": None, "kernel": "tally3_kernel",
                           "peak_source": f"hbm_gbs of MEASURED_PEAKS.json ({pk_kind}); per GPU, "
                                          "whole step (96 B/triple)"}
        print(json.dumps(out))
    dist.barrier()
    dist.destroy_process_group()

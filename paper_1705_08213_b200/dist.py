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

    def g_pair(self, ring, a, b):
        """Pairwise G between blocks a < b (all of a's vectors precede b's) into the global G."""
        N, s, w = ring.full
        (alo, ahi), (blo, bhi) = ring.bounds[a], ring.bounds[b]
        n_v = ring.n_v
        Gv = ring.G.view(-1)[alo * n_v + blo:]
        self.ccc.ccc_2way_block(N[alo:ahi], s[alo:ahi], w[alo:ahi], alo, 0, ahi - alo, N[blo:bhi], s[blo:bhi],
                                w[blo:bhi], blo, False, self.n_f, 0, g=Gv, ldg=n_v)

    def _blk(self, ring, b):
        N, s, w = ring.full
        lo, hi = ring.bounds[b]
        return self.ccc.block(N[lo:hi], s[lo:hi], w[lo:hi], lo)

    def unit_records(self, ring, u, p_lo, p_hi):
        return decomp.unit3_count(decomp.Unit3(u.pb, p_lo, p_hi, u.mb, u.m_lo, u.m_hi, u.nb,
                                               u.n_lo, u.n_hi, u.order), ring.bounds)

    def reserve_unit_records(self, n_rec):
        f = self.out_flags
        self._buf3 = None
        T = torch.empty((n_rec, 8), dtype=torch.int32, device=self.device) if f & 1 else None
        C = (torch.empty((n_rec, 8), dtype=torch.float64, device=self.device) if f & 2 else
             torch.empty((n_rec, 8), dtype=torch.float32, device=self.device) if f & 4 else None)
        self._buf3 = (n_rec, f, T, C)

    def unit(self, ring, u, p_lo, p_hi, ck):
        """One piece of a tetrahedral unit into a reused record buffer: the views it returns
        (and hands to Ring3Way's sink) are valid only until the next piece is launched on
        the current stream -- a sink that keeps records must copy them on this stream."""
        f = self.out_flags
        n_rec = self.unit_records(ring, u, p_lo, p_hi)
        buf = getattr(self, "_buf3", None)
        if buf is None or buf[0] < n_rec or (buf[1] & 7) != (f & 7):
            T = torch.empty((n_rec, 8), dtype=torch.int32, device=self.device) if f & 1 else None
            C = (torch.empty((n_rec, 8), dtype=torch.float64, device=self.device) if f & 2 else
                 torch.empty((n_rec, 8), dtype=torch.float32, device=self.device) if f & 4 else None)
            self._buf3 = None
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


def ring_shift(cur: torch.Tensor, nxt: torch.Tensor, r: int, P: int, group=None, ranks=None):
    """Post send(cur -> r-1) and recv(nxt <- r+1); returns the requests to wait on.
    r, P: position and size of the ring; ranks[k] = global rank of ring position k (a
    sub-ring of a process grid), default k itself.

    NCCL moves the device buffers directly (NVLink).  gloo cannot move CUDA tensors point to
    point, so under a gloo group the packed block is staged through host memory -- the
    transport that lets several ranks share one GPU in the tests; the kernels are the same."""
    to = ranks[(r - 1) % P] if ranks is not None else (r - 1) % P
    frm = ranks[(r + 1) % P] if ranks is not None else (r + 1) % P
    if cur.is_cuda and dist.get_backend(group) == "gloo":
        host = torch.empty(nxt.shape, dtype=nxt.dtype)
        ops = [dist.P2POp(dist.isend, cur.contiguous().cpu(), to, group),
               dist.P2POp(dist.irecv, host, frm, group)]
        return [_StagedRecv(dist.batch_isend_irecv(ops), host, nxt)]
    ops = [dist.P2POp(dist.isend, cur.contiguous(), to, group),
           dist.P2POp(dist.irecv, nxt, frm, group)]
    return dist.batch_isend_irecv(ops)


def row_bands(u, bounds, max_records):
    """Cut a 2-way unit into row bands of at most max_records records each -- the paper's
    2-way "phases" (§7 item 3: compute a subset of the blocks per run so the
    results fit in memory).  A band never splits a row; a single row above the bound is a
    band of its own.  None = the whole unit."""
    if max_records is None:
        return [(u.a_lo, u.a_hi)]
    n_b = bounds[u.b][1] - bounds[u.b][0]
    out, lo, acc = [], u.a_lo, 0
    for i in range(u.a_lo, u.a_hi):
        r = (n_b - 1 - i) if u.diag else n_b
        if acc and acc + r > max_records:
            out.append((lo, i))
            lo, acc = i, 0
        acc += r
    if u.a_hi > lo:
        out.append((lo, u.a_hi))
    return out


def band_records(u, bounds, lo, hi) -> int:
    n_b = bounds[u.b][1] - bounds[u.b][0]
    if u.diag:
        return sum(n_b - 1 - i for i in range(lo, hi))
    return (hi - lo) * n_b


class Ring2Way:
    """Per-rank state of the block-circulant 2-way computation (buffers are reused
    across calls so a bench step does no allocation).

    max_records = None: every unit keeps its own record buffers (`run` returns them).
    max_records = M: every unit is cut into row-band phases of <= M records (row_bands)
    and all phases write into ONE reused buffer; `sink(unit, a_lo, a_hi, (T, C))` sees each
    phase's records before the next phase overwrites them (copy on the current stream to
    keep them).  This is how configs[2] (614 GB of records at P = 1) runs in FULL mode."""

    def __init__(self, backend, bounds, rank: int, world: int, group=None, max_records=None):
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
        self.own = backend.expanded_empty(rows[rank])
        self.max_records = max_records
        self.phases = [row_bands(u, bounds, max_records) for u in self.units]
        if max_records is None:
            self.out = [backend.outputs(decomp.unit2_records(u, bounds)) for u in self.units]
        else:
            big = max(band_records(u, bounds, lo, hi) for u, ph in zip(self.units, self.phases)
                      for lo, hi in ph)
            self.buf = backend.outputs(big)
            self.out = None
        self.ck = backend.checksum_zero()
        self.launches = 0

    def _rows(self, b):
        return self.bounds[b][1] - self.bounds[b][0]

    def n_phases(self) -> int:
        return sum(len(ph) for ph in self.phases)

    def run(self, packed_own, timed=False, sink=None):
        """One pass over this rank's units.  packed_own: the rank's packed block."""
        be, r, P = self.be, self.rank, self.P
        own = be.expand(packed_own, self.own)
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
                assert u.a == r or u.b == r
                assert held in (u.a, u.b)
                for lo, hi in self.phases[ui]:
                    if self.out is not None:
                        out = self.out[ui]
                    else:
                        n = band_records(u, self.bounds, lo, hi)
                        out = tuple(x[:n] if x is not None else None for x in self.buf)
                    self.launches += be.block(A, self.bounds[u.a][0], lo, hi, B,
                                              self.bounds[u.b][0], u.diag, out, self.ck,
                                              timed=timed)
                    if sink is not None:
                        sink(u, lo, hi, out)
            for q in reqs:
                q.wait()
            if nxt is not None:
                cur = nxt
        return self.out


class Ring3Way:
    """Per-rank tetrahedral 3-way computation.  Every rank
    needs every block: a ring all-gather *with retention* of the packed blocks (P-1
    steps, NCCL send/recv) fills a full expanded N in place (blocks are contiguous
    rows).  Each unit runs as soon as its blocks are resident, while the next block is in
    flight: first the pairwise G among its blocks (KB-2W block GEMMs, ~1/n_f of the 3-way
    work, each block pair once), then the unit cut into pivot sub-ranges so that no output
    buffer exceeds `max_records` (the paper's stages)."""

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
        if hasattr(backend, "reserve_unit_records"):
            # one record buffer sized for the largest piece up front (no regrowth mid-run)
            backend.reserve_unit_records(max((backend.unit_records(self, u, lo, hi)
                                              for u in self.units for lo, hi in self._pieces(u)),
                                             default=0))

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
        them; the default drops them after the checksum fold).

        Every unit runs as soon as its three blocks have arrived -- while the next block is
        in flight round the ring -- after the pairwise G among those blocks (the epilogue's
        G_pm, G_pn, G_mn) has been computed block pair by block pair."""
        be, r, P = self.be, self.rank, self.P
        lo, hi = self.bounds[r]
        be.expand_into(packed_own, self.full, lo, hi)
        self.launches = 1
        self.arrived = {r}
        self.g_done = set()
        done = [False] * len(self.units)
        cur = packed_own
        reqs = []
        for d in range(P):
            nxt = None
            if d < P - 1:
                nb = (r + d + 1) % P
                nxt = self.recv[d % 2][: self.bounds[nb][1] - self.bounds[nb][0]]
                reqs = ring_shift(cur, nxt, r, P, self.group)
            self._run_ready(done, sink)          # overlaps the block in flight
            for q in reqs:
                q.wait()
            reqs = []
            if nxt is not None:
                nb = (r + d + 1) % P
                be.expand_into(nxt, self.full, *self.bounds[nb])
                self.arrived.add(nb)
                self.launches += 1
                cur = nxt
        self._run_ready(done, sink)
        assert all(done)
        return self.ck

    def _g(self, a, b):
        """The pairwise G of blocks a, b (once per pass)."""
        a, b = min(a, b), max(a, b)
        if (a, b) in self.g_done:
            return
        if a == b:
            self.be.g_block(self, a, a)
        else:
            self.be.g_pair(self, a, b)
        self.g_done.add((a, b))
        self.launches += 1

    def _run_ready(self, done, sink):
        for k, u in enumerate(self.units):
            blocks = {u.pb, u.mb, u.nb}
            if done[k] or not blocks <= self.arrived:
                continue
            for a in blocks:
                for b in blocks:
                    if a <= b:
                        self._g(a, b)
            for plo, phi in self._pieces(u):
                out = self.be.unit(self, u, plo, phi, self.ck)
                self.launches += 1
                if sink is not None:
                    sink(u, plo, phi, out)
            done[k] = True


def checksum_total(ck_local: torch.Tensor, group=None) -> int:
    """Sum of the ranks' 128-bit checksums mod 2^128 (host-side, exact); a world of one
    without a process group returns the local value."""
    if not dist.is_available() or not dist.is_initialized():
        lo, hi = (int(x) & ((1 << 64) - 1) for x in ck_local.cpu().tolist())
        return (hi << 64) | lo
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


def weak_scaled_nv3(n_v1: int, P: int, align: int = 256) -> int:
    """n_v at P GPUs with the same per-GPU triple count as n_v1 on one GPU."""
    if P == 1:
        return n_v1
    q = align * P
    return max(q, int(round(n_v1 * P ** (1.0 / 3.0) / q)) * q)


# ----------------------------------------------------------------------------- bench
class _World:
    """One process per GPU: torch.distributed over NCCL when launched by torchrun
    (WORLD_SIZE > 1), a world of one without a process group otherwise."""

    def __init__(self):
        self.P = int(os.environ.get("WORLD_SIZE", "1"))
        # CCC_DIST_BACKEND=gloo is the functional test of this N > 1 path on a one-GPU box:
        # the ranks share the visible GPU(s) and the ring moves packed blocks through host
        # memory (ring_shift); a timing taken that way is not a multi-GPU number.
        self.backend = os.environ.get("CCC_DIST_BACKEND", "nccl")
        if self.P > 1:
            dist.init_process_group(self.backend)
            self.rank, self.P = dist.get_rank(), dist.get_world_size()
        else:
            self.rank = 0
        self.local = int(os.environ.get("LOCAL_RANK", self.rank))
        if self.backend == "gloo":
            global _SHARE
            n_dev = torch.cuda.device_count()
            self.local %= n_dev
            _SHARE = -(-self.P // n_dev)
        torch.cuda.set_device(self.local)

    def barrier(self):
        if self.P > 1:
            dist.barrier()

    def max(self, v: float) -> float:
        if self.P == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.P > 1:
            dist.barrier()
            dist.destroy_process_group()


_SHARE = 1   # ranks per GPU: > 1 only under the gloo test hook (_World)


def record_budget(bytes_per_record: int, reserve_bytes: int) -> int:
    """Records that fit in the free HBM after `reserve_bytes` more are set aside (ranks that
    share a GPU under the test hook each get an equal part of its total memory)."""
    free, total = torch.cuda.mem_get_info()
    if _SHARE > 1:
        free = total // _SHARE
    return max(1, int((free - reserve_bytes - (6 << 30)) // bytes_per_record))


def _timed(W, step, args):
    """W warm-ups, barrier + synchronize, exactly K steps between CUDA events on the
    launching stream (NVML clocks sampled meanwhile), max over ranks."""
    from bench import ClockSampler
    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    W.barrier()
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    clk = ClockSampler(W.local)
    torch.cuda.synchronize()
    W.barrier()
    with clk:
        ev[0].record(stream)
        for k in range(args.steps):
            step(True)
            ev[k + 1].record(stream)
        torch.cuda.synchronize()
    per = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    ms = W.max(ev[0].elapsed_time(ev[-1]))
    per_max = [W.max(x) for x in per]
    return ms, per_max, clk.summary()


def bench_main(args, wl, metric, unit):  # noqa: C901
    """bench.py through the decompositions: N > 1 (torchrun, NCCL) or the strong-scaled
    BASELINE configs (c3, c5) at any N.  2-way: block-circulant ring with row-band phases
    when the records exceed HBM; 3-way: tetrahedral units cut into pivot pieces.  After
    the timed steps, one untimed step with the 128-bit checksum is summed over the ranks
    and compared with a single-GPU CHECKSUM-mode run of the whole problem on rank 0 (the
    paper's bit-for-bit check across decompositions)."""
    import json

    import synthgen
    from . import ccc

    W = _World()
    rank, P = W.rank, W.P
    strong = wl.get("strong", False)
    way = wl["way"]
    n_f = wl["n_f"]
    gshape = getattr(args, "grid", None)
    if gshape is not None:
        if way != 2 or decomp.Grid(*gshape).world != P:
            raise SystemExit("--grid n_pv,n_pr,n_pf is a 2-way decomposition of all ranks (product = N)")
    if way == 2:
        n_v = wl["n_v"] if strong else weak_scaled_nv(wl["n_v"], P)
    else:
        n_v = wl["n_v"] if strong else weak_scaled_nv3(wl["n_v"], P)
    bounds = decomp.block_bounds(n_v, P, align=256)
    lo, hi = bounds[rank]
    full = ccc.OUT_TALLY | ccc.OUT_CCC_F64
    be = CudaBackend(n_f, ccc.GAMMA, full)
    codes = synthgen.random_codes(hi - lo, n_f, seed=1, device="cuda", row0=lo)
    packed = be.packed_empty(hi - lo)
    k_pad, stride = ccc.ccc_k_pad(n_f), ccc.ccc_packed_stride(n_f)
    rec_bytes = 48 if way == 2 else 96
    if way == 2 and gshape is not None:
        # the paper's process grid: vector blocks x result parts x field slices
        from .fieldsplit import field_slices
        from .grid import CudaGridBackend, Grid2Way
        G = decomp.Grid(*gshape)
        v, _, f = G.coords(rank)
        bounds = decomp.block_bounds(n_v, G.n_pv, align=256)
        lo, hi = bounds[v]
        f0, f1 = field_slices(n_f, G.n_pf)[f]
        be = CudaGridBackend(f1 - f0, n_f, ccc.GAMMA, full)
        codes = synthgen.random_codes(hi - lo, n_f, seed=1, device="cuda", row0=lo)[:, f0:f1].contiguous()
        packed = be.packed_empty(hi - lo)
        k_pad, stride = ccc.ccc_k_pad(f1 - f0), ccc.ccc_packed_stride(f1 - f0)
        parts = [decomp.split_rows(u, bounds, G.n_pr)[G.coords(rank)[1]]
                 for u in decomp.plan_2way(G.n_pv, v, bounds)]
        my_rec = sum(decomp.unit2_records(decomp.Unit2(u.a, u.b, a, b, u.diag, u.step), bounds)
                     for u, (a, b) in zip(decomp.plan_2way(G.n_pv, v, bounds), parts))
        max_rows = max(b - a for a, b in bounds)
        fixed = 2 * max_rows * k_pad + 2 * max_rows * stride + (2 << 30)   # + slot buffers
        budget = record_budget(rec_bytes, fixed)
        max_rec = None if my_rec <= budget else budget
        ring = Grid2Way(be, G, rank, bounds, max_records=max_rec)
        phases = sum(len(b) for b in ring.bands)
        my_rec = my_rec // G.n_pf     # records this rank writes (its owned tiles)
    elif way == 2:
        units = decomp.plan_2way(P, rank, bounds)
        my_rec = sum(decomp.unit2_records(u, bounds) for u in units)
        max_rows = max(b - a for a, b in bounds)
        fixed = 2 * max_rows * k_pad + 2 * max_rows * stride          # own + other N, recv
        budget = record_budget(rec_bytes, fixed)
        max_rec = None if my_rec <= budget else budget
        ring = Ring2Way(be, bounds, rank, P, max_records=max_rec)
        phases = ring.n_phases()
    else:
        my_rec = decomp.total_triples(P, bounds) // P
        fixed = n_v * k_pad + 4 * n_v * n_v + 2 * max(b - a for a, b in bounds) * stride
        max_rec = min(record_budget(rec_bytes, fixed), 1 << 40)
        ring = Ring3Way(be, bounds, rank, P, max_records=max_rec)
        phases = sum(len(ring._pieces(u)) for u in ring.units)
    launches = [0]

    def step(timed):
        be.pack(codes, packed)
        ring.ck.zero_()
        if way == 2 and gshape is None:
            ring.run(packed, timed=timed)
        else:
            ring.run(packed)
        if timed:
            launches[0] += 1 + ring.launches

    ms, per, clk = _timed(W, step, args)
    kms = sum(a.elapsed_time(b) for a, b in be.kernel_events) if (way == 2 and gshape is None) else None
    if kms is not None:
        kms = W.max(kms)
    # verification: + the checksum, summed over ranks
    be.out_flags = full | ccc.OUT_CHECKSUM
    step(False)
    torch.cuda.synchronize()
    ck = checksum_total(ring.ck)
    be.out_flags = full
    comps = n_f * (n_v * (n_v - 1) // 2 if way == 2 else n_v * (n_v - 1) * (n_v - 2) // 6)
    ms_step = ms / args.steps
    e2e = None
    if args.e2e and way == 2 and gshape is None and ring.out is not None:
        # the same step through the public API with host buffers: H2D of this rank's genotype
        # codes from pinned memory, D2H of every record it computes, max over ranks
        import time
        codes_h = codes.cpu().pin_memory()
        outs_h = [tuple(x.cpu().pin_memory() if x is not None else None for x in o) for o in ring.out]
        d2h = sum(x.numel() * x.element_size() for o in ring.out for x in o if x is not None)
        e_steps = max(1, min(args.steps, 3))

        def e2e_step():
            codes.copy_(codes_h, non_blocking=True)
            step(False)
            for o, oh in zip(ring.out, outs_h):
                for x, xh in zip(o, oh):
                    if x is not None:
                        xh.copy_(x, non_blocking=True)
            torch.cuda.synchronize()

        e2e_step()
        W.barrier()
        t = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        dt = W.max((time.perf_counter() - t) / e_steps)
        e2e = {"value": comps / dt, "unit": unit, "h2d_bytes_per_step": (hi - lo) * n_f,
               "d2h_bytes_per_step": d2h, "steps": e_steps, "ms_per_step": dt * 1e3,
               "api": "dist.Ring2Way over the libccc binding, pinned host codes in / records out "
                      "(per-rank bytes)"}
        del outs_h, codes_h
    # the single-GPU CHECKSUM-mode reference run of the whole problem (rank 0, untimed)
    ring_phases = phases
    if gshape is not None:
        ring.close()
    del ring
    torch.cuda.empty_cache()
    ref = None
    if rank == 0:
        all_codes = codes if P == 1 else synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
        pk_all = ccc.ccc_pack(all_codes)
        del all_codes
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        if way == 2:
            _, _, ck1 = ccc.ccc_2way(pk_all, n_f, out_flags=ccc.OUT_CHECKSUM)
        else:
            _, _, ck1 = ccc.ccc_3way(pk_all, n_f, out_flags=ccc.OUT_CHECKSUM)
        t1.record()
        torch.cuda.synchronize()
        ref = {"single_gpu_checksum": f"{ccc.checksum_int(ck1):032x}",
               "match": ccc.checksum_int(ck1) == ck,
               "ms": t0.elapsed_time(t1),
               "how": ("ccc_2way" if way == 2 else "ccc_3way (1 stage)") + " of all %d vectors on "
                      "rank 0's GPU in CHECKSUM mode vs the sum of the ranks' checksums of the "
                      "decomposed run (P:651-656)" % n_v}
    if rank == 0:
        from bench import INT8_OPS_PER_CLK_SM, NOMINAL_INT8_TOPS, peaks
        pk, pk_kind = peaks()
        per_s = sorted(per)
        mhz = clk.get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)
        pipe = 148 * INT8_OPS_PER_CLK_SM * mhz * 1e6 / 1e12
        from bench import config_of
        cfg = config_of(wl, P)
        if gshape is not None:
            cfg["parallelism"] = "process grid n_pv x n_pr x n_pf = %d x %d x %d" % tuple(gshape)
            cfg["ring"] = ("packed 2-bit blocks round each (r, f) sub-ring, NCCL send/recv; field groups: "
                           "partial tiles stored from the GEMM epilogue into the owners' CUDA IPC slots, "
                           "stream-ordered barrier, owner finish (P:583-606)")
        out = {"metric": metric, "value": comps / (ms_step / 1e3), "unit": unit, "n_gpus": P,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
               "ms_per_step_median": per_s[len(per_s) // 2], "ms_per_step_best": per_s[0],
               "higher_is_better": True, "scaling": "strong" if strong else "weak",
               "vs_baseline": None, "dtype": "int8", "data": "synthetic", "config": cfg,
               "gpu_launches": launches[0], "checksum": f"{ck:032x}",
               "decomposition_check": ref, "clocks": clk,
               "phases_per_rank": ring_phases if max_rec is not None else 1}
        step_tops = 2.0 * comps / P / (ms_step / 1e3) / 1e12
        if way == 2:
            # grid: the export GEMMs + finishes of a rank are the whole step (no per-kernel
            # events), so the achieved rate is taken over the step
            ach = 2.0 * n_f * my_rec * args.steps / ((kms if kms else ms) / 1e3) / 1e12
            peak = 2.0 * pk["bf16_tflops"]
            out["roofline"] = {
                "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "traffic": None, "kernel": "tally2_kernel",
                "peak_source": f"2 x bf16_tflops of MEASURED_PEAKS.json ({pk_kind}); per GPU (rank 0)",
                "int8_pipe_at_clock": {"sm_mhz": mhz, "TOPS": pipe, "kernel_frac": ach / pipe,
                                       "step_frac": step_tops / pipe},
                "nominal_int8": {"TOPS": NOMINAL_INT8_TOPS, "kernel_frac": ach / NOMINAL_INT8_TOPS,
                                 "step_frac": step_tops / NOMINAL_INT8_TOPS}}
        else:
            gbs = comps / n_f * rec_bytes / P / (ms_step / 1e3) / 1e9
            out["roofline"] = {
                "bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": gbs / pk["hbm_gbs"], "traffic": None, "kernel": "tally3_kernel",
                "peak_source": f"hbm_gbs of MEASURED_PEAKS.json ({pk_kind}); per GPU, whole step "
                               "(96 B/triple)",
                "tensor": {"int8_pipe_at_clock": {"sm_mhz": mhz, "TOPS": pipe, "step_frac": step_tops / pipe},
                           "nominal_int8": {"TOPS": NOMINAL_INT8_TOPS,
                                            "step_frac": step_tops / NOMINAL_INT8_TOPS}}}
        if W.backend != "nccl":
            out["transport"] = ("%s test hook (CCC_DIST_BACKEND): %d ranks share %d GPU(s), blocks staged "
                                "through host memory; a functional run of the N > 1 path, not a "
                                "multi-GPU timing" % (W.backend, P, torch.cuda.device_count()))
        out["e2e"] = e2e
        if e2e is None:
            out["e2e_note"] = ("not measured on this workload: one step's records (%.0f GB) are "
                               "written in phases and exceed host memory; e2e is measured on the "
                               "configs[1] line" % (comps / n_f * rec_bytes / 1e9))
        print(json.dumps(out))
    W.close()

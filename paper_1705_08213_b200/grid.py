"""The 2-way CCC on the paper's process grid: n_pv vector blocks x n_pr result parts x
n_pf field slices (§4).

  * n_pv: vector blocks, block-circulant ring of packed blocks (dist.Ring2Way's scheme,
    P:596-606): rank (v, r, f) computes block row v of the pair matrix.
  * n_pr: "the n_pr parallel axis is used to parallelize the computation of the blocks of
    this block row": every unit of block row v is cut into n_pr row ranges
    with equal record counts (decomp.split_rows); part r is rank (v, r, f)'s.
  * n_pf: field slices.  "The n_pf parallelism axis requires a parallel reduction
    operation": the n_pf ranks (v, r, *) hold the same two blocks over their own
    fields; for every unit (band) the tally GEMM of each slice stores its partial tiles
    straight into the slot of the tile's owner (t mod n_pf) from the GEMM epilogue -- the
    scatter half of a reduce-scatter fused onto the GEMM, over NVLink through CUDA IPC
    peer pointers -- and after a stream-ordered barrier each owner reduces its tiles and
    writes their records (ccc_2way_fs_block_export / ccc_2way_fs_block_finish).

Ring traffic runs on the ring group of (r, f), the barrier and the allele-sum all-reduce on
the field group of (v, r).  Outputs stay on the owning rank in ccc_2way_block's layout of
the unit band (global indices implied by the unit).  The kernels come from a backend: the
product one is `CudaGridBackend` (libccc.so); the CPU tests inject their own (gloo).
`run_grid_simulated` runs every rank's work of a grid on the current GPU (local slots).
"""
from __future__ import annotations

import torch

from . import decomp
from .dist import CudaBackend, ring_shift, row_bands
from .fieldsplit import field_slices, waves


def make_groups(grid: decomp.Grid, rank: int):
    """(ring group, field group) of `rank`; every rank must call this (torch.distributed
    creates groups collectively).  (None, None) without an initialised process group."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or grid.world == 1:
        return None, None
    v, r, f = grid.coords(rank)
    ring = field = None
    for rr in range(grid.n_pr):
        for ff in range(grid.n_pf):
            g = dist.new_group(grid.ring_ranks(rr, ff))
            if (rr, ff) == (r, f):
                ring = g
    for vv in range(grid.n_pv):
        for rr in range(grid.n_pr):
            g = dist.new_group(grid.field_ranks(vv, rr))
            if (vv, rr) == (v, r):
                field = g
    return ring, field


class Grid2Way:
    """Per-rank state of the 2-way computation on a Grid (buffers reused across runs).

    bounds: the n_pv vector blocks; the rank's packed input is block v over its field
    slice.  max_records / sink: the row-band phases of dist.Ring2Way (one reused record
    buffer); wave_tiles bounds the slot memory of one export/finish wave."""

    def __init__(self, backend, grid: decomp.Grid, rank: int, bounds, max_records=None, wave_tiles=None,
                 groups=None):
        self.be = backend
        self.grid = grid
        self.rank = rank
        self.v, self.r, self.f = grid.coords(rank)
        self.bounds = bounds
        self.ring_group, self.field_group = groups if groups is not None else make_groups(grid, rank)
        self.ring_ranks = grid.ring_ranks(self.r, self.f)
        self.units = []
        for u in decomp.plan_2way(grid.n_pv, self.v, bounds):
            lo, hi = decomp.split_rows(u, bounds, grid.n_pr)[self.r]
            self.units.append(decomp.Unit2(u.a, u.b, lo, hi, u.diag, u.step))
        self.steps = decomp.ring_steps_2way(grid.n_pv)
        self.bands = []      # per unit: [(lo, hi, [(t_lo, t_hi), ...]), ...]
        nbytes, big = 0, 0
        for u in self.units:
            bl = []
            if u.a_hi > u.a_lo:
                for lo, hi in row_bands(u, bounds, max_records):
                    tiles = backend.fs_tiles(self._rows(u.a), lo, hi, self._rows(u.b), u.diag)
                    wv = waves(tiles, wave_tiles)
                    nbytes = max([nbytes] + [backend.fs_slot_bytes(grid.n_pf, a, b) for a, b in wv])
                    big = max(big, decomp.unit2_records(decomp.Unit2(u.a, u.b, lo, hi, u.diag, u.step), bounds))
                    bl.append((lo, hi, wv))
            self.bands.append(bl)
        backend.fs_open(self.field_group, self.f, grid.n_pf, max(nbytes, 4))
        rows = [hi - lo for lo, hi in bounds]
        self.max_rows = max(rows)
        self.recv = [backend.packed_empty(self.max_rows) for _ in range(2 if self.steps else 0)]
        self.other = backend.expanded_empty(self.max_rows) if self.steps else None
        self.own = backend.expanded_empty(rows[self.v])
        self.s_own = backend.s_empty(rows[self.v])
        self.s_other = backend.s_empty(self.max_rows) if self.steps else None
        self.max_records = max_records
        if max_records is None:
            self.out = [backend.outputs(decomp.unit2_records(u, bounds)) for u in self.units]
            self.buf = None
        else:
            self.out = None
            self.buf = backend.outputs(big)
        self.ck = backend.checksum_zero()
        self.launches = 0

    def _rows(self, b):
        return self.bounds[b][1] - self.bounds[b][0]

    def n_waves(self) -> int:
        return sum(len(w) for bl in self.bands for _, _, w in bl)

    def run(self, packed_own, sink=None):
        """One pass over this rank's part of its block row.  packed_own: block v over this
        rank's field slice (packed).  sink(unit, a_lo, a_hi, (T, C)) sees every band's
        buffer after its owner tiles are written (only this rank's tiles are)."""
        be, v, P = self.be, self.v, self.grid.n_pv
        own = be.expand(packed_own, self.own)
        s_own = be.s_full(own, self.field_group, self.s_own)
        self.launches = 1
        cur = packed_own
        wave_no = 0
        for d in range(self.steps + 1):
            reqs, nxt = [], None
            if d < self.steps:
                nb = (v + d + 1) % P
                nxt = self.recv[d % 2][: self._rows(nb)]
                reqs = ring_shift(cur, nxt, v, P, self.ring_group, self.ring_ranks)
            if d == 0:
                held, s_held = own, s_own
            else:
                held = be.expand(cur, self.other)
                s_held = be.s_full(held, self.field_group, self.s_other)
                self.launches += 1
            for ui, u in enumerate(self.units):
                if u.step != d:
                    continue
                A, sA = (own, s_own) if (u.a == v or d == 0) else (held, s_held)
                B, sB = (own, s_own) if (u.b == v or d == 0) else (held, s_held)
                for lo, hi, wv in self.bands[ui]:
                    if self.out is not None:
                        out = self.out[ui]
                    else:
                        n = decomp.unit2_records(decomp.Unit2(u.a, u.b, lo, hi, u.diag, u.step), self.bounds)
                        out = tuple(x[:n] if x is not None else None for x in self.buf)
                    for t_lo, t_hi in wv:
                        k = wave_no & 1
                        wave_no += 1
                        be.fs_export(A, B, lo, hi, u.diag, t_lo, t_hi, k)
                        be.fs_barrier(k)
                        be.fs_finish(sA, self.bounds[u.a][0], lo, hi, sB, self.bounds[u.b][0], u.diag,
                                     t_lo, t_hi, k, out, self.ck)
                        self.launches += 2
                    if sink is not None:
                        sink(u, lo, hi, out)
            for q in reqs:
                q.wait()
            if nxt is not None:
                cur = nxt
        return self.out

    def close(self):
        self.be.fs_close()


class CudaGridBackend(CudaBackend):
    """libccc kernels for Grid2Way on the current CUDA device: pack / expand of the rank's
    field slice (n_f_slice fields), export GEMM into the field group's slot buffers (CUDA
    IPC handles exchanged in the field group), finish with the full n_f."""

    def __init__(self, n_f_slice: int, n_f: int, gamma: float, out_flags: int):
        super().__init__(n_f_slice, gamma, out_flags)
        self.n_f_full = n_f
        self.bufs, self.opened, self.tables = [], [], []
        self.group = None

    def s_empty(self, rows):
        return torch.empty(rows, dtype=torch.int32, device=self.device)

    def s_full(self, expanded, group, out):
        """Full allele sums of a block: the all-reduce of its slices' s over the field group."""
        s = out[: expanded[1].shape[0]]
        s.copy_(expanded[1])
        if group is not None:
            import torch.distributed as dist
            dist.all_reduce(s, group=group)
        return s

    def fs_tiles(self, n_a, lo, hi, n_b, diag):
        return self.ccc.ccc_2way_fs_block_tiles(n_a, lo, hi, n_b, diag)

    def fs_slot_bytes(self, n_pf, t_lo, t_hi):
        return self.ccc.ccc_2way_fs_slot_bytes(n_pf, t_lo, t_hi)

    def fs_open(self, group, f, n_pf, nbytes):
        """Two slot buffers (waves alternate), shared with the field group through CUDA IPC."""
        self.group, self.f, self.n_pf = group, f, n_pf
        self.bufs = [self.ccc.IpcBuffer(nbytes) for _ in range(2)]
        if group is None:
            handles = [[None, None]]
        else:
            import torch.distributed as dist
            handles = [None] * n_pf
            dist.all_gather_object(handles, [b.handle() for b in self.bufs], group=group)
        self.tables = []
        for k in range(2):
            ptrs = []
            for q in range(n_pf):
                if q == f:
                    ptrs.append(self.bufs[k].ptr)
                else:
                    p = self.ccc.ipc_open(handles[q][k])
                    self.opened.append(p)
                    ptrs.append(p)
            self.tables.append(torch.tensor(ptrs, dtype=torch.int64, device=self.device))
        self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)

    def fs_export(self, A, B, lo, hi, diag, t_lo, t_hi, k):
        self.ccc.ccc_2way_fs_block_export(A[0], A[1], lo, hi, B[0], B[1], diag, self.n_f, self.tables[k],
                                          self.f, self.n_pf, t_lo, t_hi)

    def fs_barrier(self, k):
        # stream-ordered: runs after this rank's exports and before its finish
        if self.group is not None:
            import torch.distributed as dist
            dist.all_reduce(self._flag, group=self.group)

    def fs_finish(self, sA, a_row0, lo, hi, sB, b_row0, diag, t_lo, t_hi, k, out, ck):
        T, C = out
        self.ccc.ccc_2way_fs_block_finish(None, sA, a_row0, lo, hi, sB, b_row0, diag, self.n_f_full, self.f,
                                          self.n_pf, t_lo, t_hi, self.out_flags, T, C, ck, gamma=self.gamma,
                                          slot_ptr=self.bufs[k].ptr)

    def fs_close(self):
        torch.cuda.synchronize()
        if self.group is not None:
            import torch.distributed as dist
            dist.barrier(group=self.group)
        for p in self.opened:
            self.ccc.ipc_close(p)
        self.opened = []
        for b in self.bufs:
            b.free()
        self.bufs = []


def run_grid_simulated(codes: torch.Tensor, grid: decomp.Grid, out_flags: int, wave_tiles=None,
                       gamma: float | None = None, align: int = 1):
    """Every rank's work of `grid` on the current GPU: the block / part / slice geometry,
    the export GEMMs of every slice into local slot buffers and every owner's finish --
    the kernels and slot addressing of Grid2Way minus the transports.  Returns
    ([(unit, a_lo, a_hi, T, C)], checksum) with one entry per (rank row, unit) part."""
    from . import ccc
    gamma = ccc.GAMMA if gamma is None else gamma
    n_v, n_f = codes.shape
    dev = codes.device
    bounds = decomp.block_bounds(n_v, grid.n_pv, align)
    slices = field_slices(n_f, grid.n_pf)
    ex, s_full = {}, {}
    for b, (lo, hi) in enumerate(bounds):
        parts = []
        for f0, f1 in slices:
            pk = ccc.ccc_pack(codes[lo:hi, f0:f1].contiguous())
            parts.append(ccc.ccc_expand(pk, f1 - f0, gamma))
        ex[b] = parts
        s_full[b] = torch.stack([p[1] for p in parts]).sum(0, dtype=torch.int32)   # the s all-reduce
    _, _, ck = ccc._outputs(0, 4, ccc.OUT_CHECKSUM, dev)
    results = []
    for v in range(grid.n_pv):
        for u0 in decomp.plan_2way(grid.n_pv, v, bounds):
            for r, (lo, hi) in enumerate(decomp.split_rows(u0, bounds, grid.n_pr)):
                if hi == lo:
                    continue
                u = decomp.Unit2(u0.a, u0.b, lo, hi, u0.diag, u0.step)
                n_a, n_b = bounds[u.a][1] - bounds[u.a][0], bounds[u.b][1] - bounds[u.b][0]
                n_rec = decomp.unit2_records(u, bounds)
                T, C, _ = ccc._outputs(n_rec, 4, out_flags & ~ccc.OUT_CHECKSUM, dev)
                tiles = ccc.ccc_2way_fs_block_tiles(n_a, lo, hi, n_b, u.diag)
                plan = waves(tiles, wave_tiles)
                nbytes = max(ccc.ccc_2way_fs_slot_bytes(grid.n_pf, a, b) for a, b in plan)
                slots = [torch.empty(max(1, nbytes // 4), dtype=torch.int32, device=dev) for _ in range(grid.n_pf)]
                ptrs = torch.tensor([t.data_ptr() for t in slots], dtype=torch.int64, device=dev)
                for t_lo, t_hi in plan:
                    for f, (f0, f1) in enumerate(slices):
                        Na, sa, _ = ex[u.a][f]
                        Nb, sb, _ = ex[u.b][f]
                        ccc.ccc_2way_fs_block_export(Na, sa, lo, hi, Nb, sb, u.diag, f1 - f0, ptrs, f, grid.n_pf,
                                                     t_lo, t_hi)
                    for f in range(grid.n_pf):
                        ccc.ccc_2way_fs_block_finish(slots[f], s_full[u.a], bounds[u.a][0], lo, hi, s_full[u.b],
                                                     bounds[u.b][0], u.diag, n_f, f, grid.n_pf, t_lo, t_hi,
                                                     out_flags, T, C, ck if out_flags & ccc.OUT_CHECKSUM else None,
                                                     gamma=gamma)
                results.append((u, lo, hi, T, C))
    return results, ck

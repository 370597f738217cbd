"""Field-axis split of the 2-way CCC (§4): `world`
ranks share the n_f fields of every vector, each tallies its slice on its own GPU, and
the reduce-scatter of the partial tallies is fused onto the GEMM (include/ccc.h, "f3").

Per wave of tiles [t_lo, t_hi):
  1. export: the tally GEMM of the rank's slice stores every partial tile straight into
     the slot buffer of the tile's owner (t mod world) -- a peer-mapped CUDA IPC pointer,
     i.e. NVLink stores issued from the GEMM epilogue while later tiles are multiplied;
  2. a stream-ordered barrier (an NCCL all-reduce of one element);
  3. finish: the owner sums the world partials of its tiles and writes their records.
Slot buffers are double-buffered across waves: the barrier of wave w+1 orders every
owner's finish of wave w-1 before the exports of wave w+1 reuse its buffer.

`run_simulated` runs every slice on the current GPU with local slot buffers: the same
kernels, slot addressing and reduction as the multi-GPU run minus the NVLink transport
(the only form the single-GPU test box can execute).  `FieldSplit2Way` is the one-process-
per-GPU orchestration (torchrun, NCCL + CUDA IPC).  There is no CPU path.
"""
from __future__ import annotations

import torch

from . import ccc


def field_slices(n_f: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced field ranges [f0, f1), one per rank (P:583-591's n_pf split)."""
    if world < 1 or n_f < world:
        raise ValueError("need 1 <= world <= n_f")
    return [(r * n_f // world, (r + 1) * n_f // world) for r in range(world)]


def waves(total_tiles: int, wave_tiles: int | None) -> list[tuple[int, int]]:
    """Tile ranges of the schedule processed per wave (bounded slot memory)."""
    w = total_tiles if not wave_tiles else max(1, wave_tiles)
    return [(t, min(total_tiles, t + w)) for t in range(0, total_tiles, w)]


def run_simulated(codes: torch.Tensor, world: int, out_flags: int = ccc.OUT_TALLY | ccc.OUT_CCC_F64,
                  wave_tiles: int | None = None, gamma: float = ccc.GAMMA):
    """All field slices on the current GPU; returns the records of ccc_2way (T, C, ck)."""
    n_v, n_f = codes.shape
    dev = codes.device
    prepared = []
    for f0, f1 in field_slices(n_f, world):
        packed = ccc.ccc_pack(codes[:, f0:f1].contiguous())
        N, s, _ = ccc.ccc_expand(packed, f1 - f0, gamma)
        prepared.append((N, s, f1 - f0))
    s_full = torch.stack([p[1] for p in prepared]).sum(0, dtype=torch.int32)   # the s all-reduce
    total = ccc.ccc_2way_fs_tiles(n_v)
    plan = waves(total, wave_tiles)
    nbytes = max(ccc.ccc_2way_fs_slot_bytes(world, a, b) for a, b in plan) if plan else 0
    slots = [torch.empty(max(1, nbytes // 4), dtype=torch.int32, device=dev) for _ in range(world)]
    ptrs = torch.tensor([t.data_ptr() for t in slots], dtype=torch.int64, device=dev)
    m = ccc.ccc_num_unique(2, n_v)
    T, C, ck = ccc._outputs(m, 4, out_flags, dev)
    for t_lo, t_hi in plan:
        for r, (N, s, nf_r) in enumerate(prepared):
            ccc.ccc_2way_fs_export(N, s, nf_r, ptrs, r, world, t_lo, t_hi)
        for r in range(world):
            ccc.ccc_2way_fs_finish(slots[r], s_full, n_f, r, world, t_lo, t_hi, out_flags, T, C, ck,
                                   gamma=gamma)
    return T, C, ck


class FieldSplit2Way:
    """One process per GPU; rank r owns field slice r of every vector (torchrun, NCCL)."""

    def __init__(self, rank: int, world: int, n_v: int, n_f: int, wave_tiles: int | None = None,
                 out_flags: int = ccc.OUT_TALLY | ccc.OUT_CCC_F64, gamma: float = ccc.GAMMA,
                 group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank, self.world, self.n_v, self.n_f = rank, world, n_v, n_f
        self.f0, self.f1 = field_slices(n_f, world)[rank]
        self.out_flags, self.gamma = out_flags, gamma
        self.plan = waves(ccc.ccc_2way_fs_tiles(n_v), wave_tiles)
        nbytes = max(ccc.ccc_2way_fs_slot_bytes(world, a, b) for a, b in self.plan)
        self.dev = torch.device("cuda", torch.cuda.current_device())
        # two slot buffers (waves alternate), shared with every peer through CUDA IPC
        self.bufs = [ccc.IpcBuffer(nbytes) for _ in range(2)]
        handles = [None] * world
        dist.all_gather_object(handles, [b.handle() for b in self.bufs], group=group)
        self.opened = []
        tables = []
        for k in range(2):
            ptrs = []
            for q in range(world):
                if q == rank:
                    ptrs.append(self.bufs[k].ptr)
                else:
                    p = ccc.ipc_open(handles[q][k])
                    self.opened.append(p)
                    ptrs.append(p)
            tables.append(torch.tensor(ptrs, dtype=torch.int64, device=self.dev))
        self.tables = tables
        self._flag = torch.zeros(1, dtype=torch.int32, device=self.dev)

    def _barrier(self):
        # stream-ordered: NCCL runs after the exports queued on this stream and before the
        # finish kernel queued next
        self.dist.all_reduce(self._flag, group=self.group)

    def run(self, codes_slice: torch.Tensor):
        """codes_slice: uint8 [n_v][f1 - f0] of this rank's fields, resident on its GPU.
        Returns this rank's records (T, C, ck) in the ccc_2way layout (own tiles only)."""
        nf_r = self.f1 - self.f0
        packed = ccc.ccc_pack(codes_slice)
        N, s, _ = ccc.ccc_expand(packed, nf_r, self.gamma)
        s_full = s.clone()
        self.dist.all_reduce(s_full, group=self.group)          # full allele sums
        m = ccc.ccc_num_unique(2, self.n_v)
        T, C, ck = ccc._outputs(m, 4, self.out_flags, self.dev)
        for w, (t_lo, t_hi) in enumerate(self.plan):
            k = w & 1
            ccc.ccc_2way_fs_export(N, s, nf_r, self.tables[k], self.rank, self.world, t_lo, t_hi)
            self._barrier()
            ccc._check(ccc.lib().ccc_2way_fs_finish(
                self.bufs[k].ptr, ccc._p(s_full), self.n_v, self.n_f, self.gamma, self.rank, self.world,
                t_lo, t_hi, self.out_flags, ccc._p(T), ccc._p(C), ccc._p(ck), ccc._stream(None)))
        return T, C, ck

    def close(self):
        torch.cuda.synchronize()
        self.dist.barrier(group=self.group)
        for p in self.opened:
            ccc.ipc_close(p)
        self.opened = []
        for b in self.bufs:
            b.free()

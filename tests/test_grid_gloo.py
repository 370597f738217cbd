"""The 2-way process grid n_pv x n_pr x n_pf (§4) on
CPU with gloo at world sizes 2-8.

grid.Grid2Way's orchestration runs unchanged -- the sub-rings of the vector-block ring,
the n_pr row split of every unit, the field groups' all-reduce of the allele sums, the
export / barrier / finish wave protocol with alternating slot buffers, phases, the
checksum -- with the kernels replaced by an oracle-backed CPU backend defined here (test
code only): a rank's "export" is the oracle's tallies of its field slice (tallies are sums
over fields, so slices add up exactly), the field-group "barrier" all-reduces them, and a
rank's "finish" writes the records of the rows it owns (tile = row, owner = tile mod
n_pf).  Every pair must be produced exactly once, by its owner, with the oracle's values.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synthgen
from paper_1705_08213_b200 import decomp


class GridOracleBackend:
    """CPU stand-in for CudaGridBackend: 'packed' = the slice's raw codes."""

    def __init__(self, n_f_slice, n_f, gamma=oracle.GAMMA):
        self.n_f, self.n_f_full, self.gamma = n_f_slice, n_f, gamma
        self.pending = [None, None]
        self.log = []          # record indices written since the sink last looked

    # pack / expand: identity on the slice's codes
    def pack(self, codes, out=None):
        if out is not None:
            out.copy_(codes)
            return out
        return codes.clone()

    def packed_empty(self, rows):
        return torch.zeros((rows, self.n_f), dtype=torch.uint8)

    def expand(self, packed, out=None):
        return (packed.clone(), None, None)

    def expanded_empty(self, rows):
        return (torch.zeros((rows, self.n_f), dtype=torch.uint8), None, None)

    def s_empty(self, rows):
        return torch.zeros((rows, 2), dtype=torch.int64)

    def s_full(self, expanded, group, out):
        s = out[: expanded[0].shape[0]]
        s.copy_(torch.from_numpy(oracle.allele_sums(expanded[0].numpy())))
        if group is not None:
            dist.all_reduce(s, group=group)
        return s

    def outputs(self, n_rec):
        return (torch.full((n_rec, 4), -1, dtype=torch.int64), torch.zeros((n_rec, 4), dtype=torch.float64))

    def checksum_zero(self):
        return torch.zeros(2, dtype=torch.int64)

    # field-split protocol (tile = one row of the band)
    def fs_tiles(self, n_a, lo, hi, n_b, diag):
        return hi - lo

    def fs_slot_bytes(self, n_pf, t_lo, t_hi):
        return 4 * (t_hi - t_lo)

    def fs_open(self, group, f, n_pf, nbytes):
        self.group, self.f, self.n_pf = group, f, n_pf

    def _pairs(self, lo, hi, n_b, diag, t_lo, t_hi):
        return [(i, j) for i in range(lo + t_lo, lo + t_hi) for j in range(i + 1 if diag else 0, n_b)]

    def fs_export(self, A, B, lo, hi, diag, t_lo, t_hi, k):
        ca, cb = A[0].numpy(), B[0].numpy()
        idx = np.array([(i, ca.shape[0] + j) for i, j in self._pairs(lo, hi, cb.shape[0], diag, t_lo, t_hi)],
                       dtype=np.int64).reshape(-1, 2)
        T, _ = oracle.pairs(np.concatenate([ca, cb]), idx)
        self.pending[k] = torch.from_numpy(T)

    def fs_barrier(self, k):
        if self.group is not None:
            dist.all_reduce(self.pending[k], group=self.group)

    def fs_finish(self, sA, a_row0, lo, hi, sB, b_row0, diag, t_lo, t_hi, k, out, ck):
        T_all = self.pending[k].numpy()
        n_a, n_b = sA.shape[0], sB.shape[0]
        two_nf = 2.0 * self.n_f_full
        rows_done = 0
        for t in range(t_lo, t_hi):
            i = lo + t
            js = list(range(i + 1 if diag else 0, n_b))
            if t % self.n_pf == self.f:
                T = T_all[rows_done: rows_done + len(js)]
                base = (sum(n_a - 1 - x for x in range(lo, i)) if diag else (i - lo) * n_b)
                for q, j in enumerate(js):
                    rec = base + q
                    out[0][rec] = torch.from_numpy(T[q])
                    wi = [1 - self.gamma * float(sA[i][a]) / two_nf for a in (0, 1)]
                    wj = [1 - self.gamma * float(sB[j][b]) / two_nf for b in (0, 1)]
                    out[1][rec] = torch.tensor([T[q][2 * a + b] / (4.0 * self.n_f_full) * wi[a] * wj[b]
                                                for a in (0, 1) for b in (0, 1)])
                    self.log.append(rec)
                    v = oracle.checksum(2, np.array([[a_row0 + i, b_row0 + j]]), T[q:q + 1])
                    cur = (int(ck[1]) & ((1 << 64) - 1)) << 64 | (int(ck[0]) & ((1 << 64) - 1))
                    s = (cur + v) & ((1 << 128) - 1)
                    to_i64 = lambda u: u - (1 << 64) if u >= (1 << 63) else u
                    ck[0] = to_i64(s & ((1 << 64) - 1))
                    ck[1] = to_i64(s >> 64)
            rows_done += len(js)

    def fs_close(self):
        pass


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, shape, port, n_v, n_f, max_rec, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    grid = decomp.Grid(*shape)
    dist.init_process_group("gloo", rank=rank, world_size=grid.world)
    try:
        from paper_1705_08213_b200.dist import checksum_total
        from paper_1705_08213_b200.fieldsplit import field_slices
        from paper_1705_08213_b200.grid import Grid2Way
        v, r, f = grid.coords(rank)
        bounds = decomp.block_bounds(n_v, grid.n_pv)
        f0, f1 = field_slices(n_f, grid.n_pf)[f]
        lo, hi = bounds[v]
        codes = synthgen.random_codes(n_v, n_f, seed=11)[lo:hi, f0:f1].contiguous()
        be = GridOracleBackend(f1 - f0, n_f)
        g = Grid2Way(be, grid, rank, bounds, max_records=max_rec, wave_tiles=2)
        got = []

        def sink(u, a_lo, a_hi, out):
            pairs = list(decomp.unit2_pairs(decomp.Unit2(u.a, u.b, a_lo, a_hi, u.diag, u.step), bounds))
            for rec in be.log:
                got.append((pairs[rec], out[0][rec].numpy().copy(), out[1][rec].numpy().copy()))
            be.log = []

        g.run(codes, sink=sink)
        ck = checksum_total(g.ck)
        g.close()
        q.put((rank, ck, got, g.n_waves()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,max_rec", [((2, 1, 2), None), ((1, 2, 2), None), ((2, 2, 1), None),
                                           ((1, 1, 3), 40), ((3, 1, 2), 25), ((2, 2, 2), None)])
def test_grid_2way_gloo(shape, max_rec):
    """Every pair exactly once over all ranks of the n_pv x n_pr x n_pf grid, with the
    oracle's tallies and CCC; the ranks' checksums sum to the oracle's."""
    n_v, n_f = 21, 29
    grid = decomp.Grid(*shape)
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, shape, port, n_v, n_f, max_rec, qq))
             for r in range(grid.world)]
    for p in procs:
        p.start()
    res = [qq.get(timeout=240) for _ in range(grid.world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    codes = synthgen.random_codes(n_v, n_f, seed=11)
    To, Co = oracle.all_pairs(codes)
    index = {tuple(p): k for k, p in enumerate(oracle.pair_list(n_v))}
    want_ck = oracle.checksum(2, oracle.pair_list(n_v), To)
    seen = set()
    for rank, ck, got, nw in res:
        assert ck == want_ck
        for pr, T, C in got:
            pr = tuple(int(x) for x in pr)
            assert pr not in seen
            seen.add(pr)
            np.testing.assert_array_equal(T, To[index[pr]])
            np.testing.assert_allclose(C, Co[index[pr]], rtol=1e-13)
    assert len(seen) == n_v * (n_v - 1) // 2


def test_grid_coords_and_groups():
    """Grid rank <-> (v, r, f) is a bijection; ring groups vary v, field groups vary f."""
    for shape in ((1, 1, 1), (2, 1, 2), (2, 3, 2), (4, 1, 2), (3, 2, 1)):
        g = decomp.Grid(*shape)
        seen = set()
        for rank in range(g.world):
            v, r, f = g.coords(rank)
            assert g.rank(v, r, f) == rank
            seen.add((v, r, f))
            assert rank in g.ring_ranks(r, f) and g.ring_ranks(r, f)[v] == rank
            assert rank in g.field_ranks(v, r) and g.field_ranks(v, r)[f] == rank
        assert len(seen) == g.world


@pytest.mark.parametrize("P,parts", [(1, 1), (1, 3), (2, 2), (4, 3), (5, 4)])
def test_split_rows(P, parts):
    """The n_pr split covers each unit's rows in order with near-equal record counts."""
    bounds = decomp.block_bounds(1003, P)
    for rank in range(P):
        for u in decomp.plan_2way(P, rank, bounds):
            sp = decomp.split_rows(u, bounds, parts)
            assert len(sp) == parts and sp[0][0] == u.a_lo and sp[-1][1] == u.a_hi
            assert all(a[1] == b[0] and a[0] <= a[1] for a, b in zip(sp, sp[1:]))
            recs = [decomp.unit2_records(decomp.Unit2(u.a, u.b, lo, hi, u.diag, u.step), bounds) for lo, hi in sp]
            assert sum(recs) == decomp.unit2_records(u, bounds)
            row_max = bounds[u.b][1] - bounds[u.b][0]
            assert max(recs) - min(recs) <= row_max

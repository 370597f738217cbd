"""World-size-2 (and 3, 4) gloo tests of the block-circulant ring orchestration on CPU.

The ring logic of paper_1705_08213_b200.dist (which block is resident at which step, the
A/B roles of every unit, record layouts, the 128-bit checksum reduction) runs unchanged;
the kernels are replaced by an oracle-backed CPU backend defined here (test code only).
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


class OracleBackend:
    """CPU stand-in: 'packed' = the raw codes, 'expanded' = (codes, None, None)."""

    def __init__(self, n_f):
        self.n_f = n_f

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

    def outputs(self, n_rec):
        return (torch.zeros((n_rec, 4), dtype=torch.int64), torch.zeros((n_rec, 4), dtype=torch.float64))

    def checksum_zero(self):
        return torch.zeros(2, dtype=torch.int64)

    def block(self, A, a_row0, a_lo, a_hi, B, b_row0, diag, out, ck, timed=False):
        ca, cb = A[0].numpy(), B[0].numpy()
        idx = []
        for il in range(a_lo, a_hi):
            for jl in range(il + 1 if diag else 0, cb.shape[0]):
                idx.append((il, ca.shape[0] + jl))
        both = np.concatenate([ca, cb])
        T, C = oracle.pairs(both, np.array(idx, dtype=np.int64).reshape(-1, 2))
        out[0][:] = torch.from_numpy(T)
        out[1][:] = torch.from_numpy(C)
        gidx = np.array([(a_row0 + i, b_row0 + j - ca.shape[0]) for i, j in idx]).reshape(-1, 2)
        v = oracle.checksum(2, gidx, T)
        lo, hi = v & ((1 << 64) - 1), v >> 64
        cur_lo, cur_hi = (int(x) & ((1 << 64) - 1) for x in ck.tolist())
        s = ((cur_hi << 64) | cur_lo) + ((hi << 64) | lo)
        s &= (1 << 128) - 1
        to_i64 = lambda u: u - (1 << 64) if u >= (1 << 63) else u
        ck[0] = to_i64(s & ((1 << 64) - 1))
        ck[1] = to_i64(s >> 64)
        return 1


def _worker(rank, world, port, n_v, n_f, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1705_08213_b200.dist import Ring2Way, checksum_total
        bounds = decomp.block_bounds(n_v, world)
        lo, hi = bounds[rank]
        codes = synthgen.random_codes(hi - lo, n_f, seed=5, row0=lo)
        ring = Ring2Way(OracleBackend(n_f), bounds, rank, world)
        outs = ring.run(codes)
        ck = checksum_total(ring.ck)
        recs = []
        for u, (T, C) in zip(ring.units, outs):
            pairs = list(decomp.unit2_pairs(u, bounds))
            recs.append((pairs, T.numpy(), C.numpy()))
        q.put((rank, ck, recs))
    finally:
        dist.destroy_process_group()


def _worker_phases(rank, world, port, n_v, n_f, max_rec, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1705_08213_b200.dist import Ring2Way, checksum_total
        bounds = decomp.block_bounds(n_v, world)
        lo, hi = bounds[rank]
        codes = synthgen.random_codes(hi - lo, n_f, seed=7, row0=lo)
        ring = Ring2Way(OracleBackend(n_f), bounds, rank, world, max_records=max_rec)
        got = []

        def sink(u, a_lo, a_hi, out):   # copy: the next phase overwrites the buffer
            sub = decomp.Unit2(u.a, u.b, a_lo, a_hi, u.diag, u.step)
            got.append((list(decomp.unit2_pairs(sub, bounds)), out[0].numpy().copy(),
                        out[1].numpy().copy()))

        assert ring.run(codes, sink=sink) is None
        q.put((rank, checksum_total(ring.ck), got, ring.n_phases(), ring.buf[0].shape[0]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,max_rec", [(1, 17), (2, 25), (3, 40), (4, 9)])
def test_ring_2way_phases_gloo(world, max_rec):
    """2-way phases: every unit cut into row bands of <= max_records records
    written into ONE reused buffer; the sink sees each band before it is overwritten.  All
    ranks' bands together cover every pair exactly once with the oracle's records."""
    n_v, n_f = 26, 31
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_phases, args=(r, world, port, n_v, n_f, max_rec, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    codes = synthgen.random_codes(n_v, n_f, seed=7)
    To, Co = oracle.all_pairs(codes)
    index = {tuple(p): r for r, p in enumerate(oracle.pair_list(n_v))}
    seen = set()
    for rank, ck, got, nph, cap in res:
        assert ck == oracle.checksum(2, oracle.pair_list(n_v), To)
        assert nph == len(got) > 1
        for pairs, T, C in got:
            rows = {i for i, _ in pairs}
            assert len(pairs) <= max(max_rec, max(sum(1 for p in pairs if p[0] == i) for i in rows))
            assert len(pairs) <= cap
            for k, pr in enumerate(pairs):
                assert pr not in seen
                seen.add(pr)
                np.testing.assert_array_equal(T[k], To[index[pr]])
                np.testing.assert_allclose(C[k], Co[index[pr]], rtol=1e-15)
    assert len(seen) == n_v * (n_v - 1) // 2


def test_row_bands():
    """Row bands never split a row, respect the bound unless one row exceeds it, and cover
    the unit's rows in order (pure host logic)."""
    from paper_1705_08213_b200.dist import band_records, row_bands
    bounds = decomp.block_bounds(1000, 4)
    for P, r in ((1, 0), (4, 0), (4, 3)):
        bounds = decomp.block_bounds(1000, P)
        for u in decomp.plan_2way(P, r, bounds):
            for m in (1, 50, 997, 10 ** 6):
                bands = row_bands(u, bounds, m)
                assert bands[0][0] == u.a_lo and bands[-1][1] == u.a_hi
                assert all(b[1] == c[0] for b, c in zip(bands, bands[1:]))
                assert sum(band_records(u, bounds, a, b) for a, b in bands) == decomp.unit2_records(u, bounds)
                for a, b in bands:
                    assert band_records(u, bounds, a, b) <= m or b - a == 1
            assert row_bands(u, bounds, None) == [(u.a_lo, u.a_hi)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3, 4])
def test_ring_2way_gloo(world):
    n_v, n_f = 23, 37
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_v, n_f, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    codes = synthgen.random_codes(n_v, n_f, seed=5)
    To, Co = oracle.all_pairs(codes)
    index = {tuple(p): r for r, p in enumerate(oracle.pair_list(n_v))}
    seen = set()
    for rank, ck, recs in res:
        assert ck == oracle.checksum(2, oracle.pair_list(n_v), To)   # same on every rank
        for pairs, T, C in recs:
            for k, pr in enumerate(pairs):
                assert pr not in seen
                seen.add(pr)
                np.testing.assert_array_equal(T[k], To[index[pr]])
                np.testing.assert_allclose(C[k], Co[index[pr]], rtol=1e-15)
    assert len(seen) == n_v * (n_v - 1) // 2


class Oracle3Backend(OracleBackend):
    """CPU stand-in for the 3-way ring: 'expanded' full matrix = the raw codes."""

    def expanded_empty(self, rows):
        return (torch.zeros((rows, self.n_f), dtype=torch.uint8), None, None)

    def g_empty(self, n_v):
        return None

    def expand_into(self, packed, full, lo, hi):
        full[0][lo:hi] = packed

    def g_block(self, ring, a, b):
        ring.g_log = getattr(ring, "g_log", set()) | {(a, b)}

    def g_pair(self, ring, a, b):
        assert a < b and {a, b} <= ring.arrived        # both blocks resident
        ring.g_log = getattr(ring, "g_log", set()) | {(a, b)}

    def g_full(self, ring):
        pass

    def unit_records(self, ring, u, p_lo, p_hi):
        return decomp.unit3_count(decomp.Unit3(u.pb, p_lo, p_hi, u.mb, u.m_lo, u.m_hi, u.nb,
                                               u.n_lo, u.n_hi, u.order), ring.bounds)

    def unit(self, ring, u, p_lo, p_hi, ck):
        # a unit runs only once its blocks are resident and their pairwise G is computed
        blocks = {u.pb, u.mb, u.nb}
        assert blocks <= ring.arrived
        assert all((a, b) in ring.g_log for a in blocks for b in blocks if a <= b)
        sub = decomp.Unit3(u.pb, p_lo, p_hi, u.mb, u.m_lo, u.m_hi, u.nb, u.n_lo, u.n_hi, u.order)
        tr = np.array(list(decomp.unit3_triples(sub, ring.bounds)), dtype=np.int64).reshape(-1, 3)
        codes = ring.full[0].numpy()
        T, C = oracle.triples(codes, tr)
        v = oracle.checksum(3, tr, T)
        cur_lo, cur_hi = (int(x) & ((1 << 64) - 1) for x in ck.tolist())
        tot = (((cur_hi << 64) | cur_lo) + v) & ((1 << 128) - 1)
        to_i64 = lambda x: x - (1 << 64) if x >= (1 << 63) else x
        ck[0] = to_i64(tot & ((1 << 64) - 1))
        ck[1] = to_i64(tot >> 64)
        return tr, T


def _worker3(rank, world, port, n_v, n_f, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1705_08213_b200.dist import Ring3Way, checksum_total
        bounds = decomp.block_bounds(n_v, world)
        lo, hi = bounds[rank]
        codes = synthgen.random_codes(hi - lo, n_f, seed=6, row0=lo)
        ring = Ring3Way(Oracle3Backend(n_f), bounds, rank, world, max_records=150)
        got = []
        ring.run(codes, sink=lambda u, plo, phi, out: got.append((phi - plo,) + tuple(out)))
        q.put((rank, checksum_total(ring.ck), got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_ring_3way_gloo(world):
    n_v, n_f = 17, 29
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker3, args=(r, world, port, n_v, n_f, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    codes = synthgen.random_codes(n_v, n_f, seed=6)
    To, _ = oracle.all_triples(codes)
    index = {tuple(t): r for r, t in enumerate(oracle.triple_list(n_v))}
    seen = set()
    for rank, ck, got in res:
        assert ck == oracle.checksum(3, oracle.triple_list(n_v), To)
        for npiv, tr, T in got:
            assert len(tr) <= 150 or npiv == 1         # stage pieces respect the bound
            for k, t in enumerate(map(tuple, tr)):
                assert t not in seen
                seen.add(t)
                np.testing.assert_array_equal(T[k], To[index[t]])
    assert len(seen) == len(To)

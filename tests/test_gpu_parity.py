"""Parity of the CUDA path (through the C ABI) with the CPU oracle, on a B200.

Bars: tallies bit-exact; CCC |x - y| <= 1e-12 |y| in fp64 (1e-6 for the
fp32 variant), x == 0 exactly where the tally is 0; checksums equal.
"""
import numpy as np
import pytest
import torch

import oracle
import synthgen

pytestmark = pytest.mark.gpu

ccc = pytest.importorskip("paper_1705_08213_b200.ccc")

F64, F32, TAL, CK = ccc.OUT_CCC_F64, ccc.OUT_CCC_F32, ccc.OUT_TALLY, ccc.OUT_CHECKSUM


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


def _t(t):
    """device int32 tally tensor -> numpy int64 (uint32 bit patterns)."""
    return t.cpu().numpy().astype(np.int64) & 0xFFFFFFFF


def _ccc_close(got, want, rtol=1e-12):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert np.all((want == 0) == (got == 0))
    nz = want != 0
    rel = np.abs(got[nz] - want[nz]) / np.abs(want[nz])
    assert rel.size == 0 or rel.max() <= rtol, rel.max()


def _codes(kind, n_v, n_f, seed=None):
    return synthgen.make_codes(kind, n_v, n_f, seed)


# ------------------------------------------------------------------- pack / expand
@pytest.mark.parametrize("n_v,n_f", [(1, 1), (3, 63), (5, 64), (7, 65), (9, 1000), (33, 4111), (11, 4100), (6, 12500)])
def test_pack_expand(n_v, n_f):
    codes = _codes("random", n_v, n_f, seed=n_f)
    packed = ccc.ccc_pack(codes.cuda())
    # expected packing (layout of include/ccc.h, built independently here)
    c = codes.numpy().astype(np.uint32)
    stride = ccc.ccc_packed_stride(n_f)
    exp = np.zeros((n_v, stride), np.uint8)
    for q in range(n_f):
        exp[:, q // 4] |= ((c[:, q] & 3) << (2 * (q % 4))).astype(np.uint8)
    np.testing.assert_array_equal(packed.cpu().numpy(), exp)
    N, s, w = ccc.ccc_expand(packed, n_f)
    S = oracle.allele_sums(codes)
    n1 = ((codes.numpy() >> 1) & 1) + (codes.numpy() & 1)
    Nn = N.cpu().numpy()
    np.testing.assert_array_equal(Nn[:, :n_f], n1)
    assert np.all(Nn[:, n_f:] == 0)
    np.testing.assert_array_equal(s.cpu().numpy(), S[:, 1])
    f = oracle.frequencies(codes)
    np.testing.assert_allclose(w.cpu().numpy(), 1.0 - oracle.GAMMA * f, rtol=1e-15, atol=0)
    # the single-GPU fused pass (unpacked codes -> N, s, w) is bit-identical to pack + expand
    N2, s2, w2 = ccc.ccc_expand_codes(codes.cuda())
    assert bool((N2 == N).all()) and bool((s2 == s).all()) and bool((w2 == w).all())


@pytest.mark.parametrize("n_v,n_f,offset", [(9, 1, 1), (33, 65, 3), (40, 1000, 0), (17, 1024, 4), (8, 4097, 2)])
def test_expand_codes_alignment_and_high_bits(n_v, n_f, offset):
    """ccc_expand_codes on rows that are not 16-B aligned (odd n_f, a base offset) and on
    bytes with garbage above the 2 code bits: N, s, w as the oracle's Eq.1 of the codes."""
    codes = _codes("random", n_v, n_f, seed=n_f + offset)
    junk = torch.randint(0, 64, (n_v, n_f), dtype=torch.uint8) << 2
    buf = torch.empty(n_v * n_f + offset, dtype=torch.uint8, device="cuda")
    view = buf[offset:].view(n_v, n_f)
    view.copy_((codes | junk).cuda())
    N, s, w = ccc.ccc_expand_codes(view)
    n1 = ((codes.numpy() >> 1) & 1) + (codes.numpy() & 1)
    Nn = N.cpu().numpy()
    np.testing.assert_array_equal(Nn[:, :n_f], n1)
    assert np.all(Nn[:, n_f:] == 0)
    np.testing.assert_array_equal(s.cpu().numpy(), oracle.allele_sums(codes)[:, 1])
    np.testing.assert_allclose(w.cpu().numpy(), 1.0 - oracle.GAMMA * oracle.frequencies(codes), rtol=1e-15, atol=0)


# ------------------------------------------------------------------- 2-way, full
def _check_2way_full(codes, flags=TAL | F64 | CK, gamma=oracle.GAMMA):
    n_v, n_f = codes.shape
    T, C, ck = ccc.two_way(codes.cuda(), gamma=gamma, out_flags=flags)
    torch.cuda.synchronize()
    To, Co = oracle.all_pairs(codes, gamma)
    if flags & TAL:
        np.testing.assert_array_equal(_t(T), To)
    if flags & F64:
        _ccc_close(C.cpu().numpy(), Co)
    if flags & F32:
        _ccc_close(C.cpu().numpy(), Co, rtol=1e-6)
    if flags & CK:
        assert ccc.checksum_int(ck) == oracle.checksum(2, oracle.pair_list(n_v), To)


def test_2way_C1_full():
    """configs[0]: 64 vectors x 1,024 individuals, bit-exact against the brute force."""
    _check_2way_full(_codes("random", 64, 1024, seed=1))


@pytest.mark.parametrize("n_v", [2, 3, 63, 64, 65, 127, 129, 257, 300])
@pytest.mark.parametrize("n_f", [1, 63, 65, 127, 1000])
def test_2way_ragged_shapes(n_v, n_f):
    if n_v * n_v * n_f > 2e8:
        pytest.skip("covered by smaller combos")
    codes = _codes("random", n_v, n_f, seed=n_v * 1000 + n_f)
    _check_2way_full(codes)                        # generic epilogue (+ checksum)
    _check_2way_full(codes, flags=TAL | F64)       # the flag-free FULL specialisation


@pytest.mark.parametrize("kind", ["hwe", "planted"])
def test_2way_other_inputs(kind):
    _check_2way_full(_codes(kind, 200, 777))


def test_2way_f32_and_gamma():
    codes = _codes("random", 150, 300, seed=5)
    _check_2way_full(codes, flags=TAL | F32)
    _check_2way_full(codes, flags=F64, gamma=0.0)
    _check_2way_full(codes, flags=F32 | CK, gamma=0.5)


def test_2way_checksum_only_and_tally_only():
    codes = _codes("random", 333, 257, seed=6)
    _check_2way_full(codes, flags=CK)
    _check_2way_full(codes, flags=TAL)


def test_2way_degenerate_inputs():
    for codes in (torch.zeros(70, 300, dtype=torch.uint8), torch.ones(70, 300, dtype=torch.uint8),
                  torch.full((70, 300), 3, dtype=torch.uint8)):
        _check_2way_full(codes)
    assert ccc.two_way(torch.zeros(1, 5, dtype=torch.uint8).cuda())[0].shape == (0, 4)


def test_2way_planted_closed_form_every_record():
    n_v, n_f = 700, 3001
    codes, L, H, _ = synthgen.planted_codes(n_v, n_f, seed=3)
    T, _, _ = ccc.two_way(codes.cuda(), out_flags=TAL)
    T = _t(T)
    for r, (i, j) in enumerate(oracle.pair_list(n_v)):
        if r % 7:           # every 7th record through the closed form (35k records)
            continue
        assert list(T[r]) == oracle.planted_tally2(L, H, n_f, i, j)


def test_2way_block_rect_and_row_split():
    """Off-diagonal blocks (block-circulant) and the antipodal row split."""
    n_v, n_f = 400, 517
    codes = _codes("random", n_v, n_f, seed=8)
    packed = ccc.ccc_pack(codes.cuda())
    N, s, w = ccc.ccc_expand(packed, n_f)
    To, Co = oracle.all_pairs(codes)
    a0, a1, b0, b1 = 0, 150, 150, 400         # A = rows [0,150), B = rows [150,400)
    lo, hi = 40, 131                          # rows [40,131) of A only
    nA, nB = a1 - a0, b1 - b0
    m = (hi - lo) * nB
    T = torch.empty((m, 4), dtype=torch.int32, device="cuda")
    C = torch.empty((m, 4), dtype=torch.float64, device="cuda")
    ck = torch.zeros(2, dtype=torch.int64, device="cuda")
    ccc.ccc_2way_block(N[a0:a1], s[a0:a1], w[a0:a1], a0, lo, hi, N[b0:b1], s[b0:b1], w[b0:b1], b0,
                       False, n_f, TAL | F64 | CK, T, C, ck)
    T, C = _t(T), C.cpu().numpy()
    idx = [(a0 + i, b0 + j) for i in range(lo, hi) for j in range(nB)]
    rows = [ccc.ccc_pair_index(n_v, i, j) for i, j in idx]
    np.testing.assert_array_equal(T, To[rows])
    _ccc_close(C, Co[rows])
    assert ccc.checksum_int(ck) == oracle.checksum(2, np.array(idx), To[rows])
    # diag block with a row range: records start at row lo
    Td = torch.empty((ccc.ccc_pair_index(n_v, 0, 1) + 1, 4), dtype=torch.int32, device="cuda")
    lo, hi = 100, 230
    m = sum(n_v - 1 - i for i in range(lo, hi))
    Td = torch.empty((m, 4), dtype=torch.int32, device="cuda")
    ccc.ccc_2way_block(N, s, w, 0, lo, hi, N, s, w, 0, True, n_f, TAL, Td)
    r0 = ccc.ccc_pair_index(n_v, lo, lo + 1)
    np.testing.assert_array_equal(_t(Td), To[r0:r0 + m])


def test_2way_host_e2e_api():
    codes = _codes("random", 300, 999, seed=12)
    T, C, ck = ccc.ccc_2way_host(codes.pin_memory(), out_flags=TAL | F64 | CK)
    To, Co = oracle.all_pairs(codes)
    np.testing.assert_array_equal(T.numpy().astype(np.int64) & 0xFFFFFFFF, To)
    _ccc_close(C.numpy(), Co)
    assert ccc.checksum_int(ck) == oracle.checksum(2, oracle.pair_list(300), To)


# ------------------------------------------------------------------- 2-way at C2 size
def test_2way_C2_full_size_sampled_and_invariants():
    """configs[1]: 20,000 x 50,000 in the launch configuration bench.py times.
    Sampled records against the brute force, the whole T(1,1) against an independent
    cuBLASLt int8 GEMM (torch._int_mm), sum T = 4 n_f for every record."""
    n_v, n_f = 20000, 50000
    codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
    T, C, _ = ccc.two_way(codes, out_flags=TAL | F64)
    torch.cuda.synchronize()
    assert bool((T.sum(1, dtype=torch.int64) == 4 * n_f).all())
    rng = np.random.default_rng(2)
    edges = [0, 1, 127, 128, 129, 255, 256, 257, 2047, 2048, 4095, 4096, n_v - 2, n_v - 1]
    ii = list(rng.integers(0, n_v - 1, 6000)) + edges
    pairs = []
    for i in ii:
        i = int(min(i, n_v - 2))
        j = int(rng.integers(i + 1, n_v))
        pairs.append((i, j))
        pairs.append((i, n_v - 1))
        pairs.append((i, i + 1))
    pairs = np.array(sorted(set(pairs)), dtype=np.int64)
    rows = torch.tensor([ccc.ccc_pair_index(n_v, int(i), int(j)) for i, j in pairs], device="cuda")
    Tg, Cg = _t(T[rows]), C[rows].cpu().numpy()
    codes_h = codes.cpu()
    To, Co = oracle.pairs(codes_h, pairs)
    np.testing.assert_array_equal(Tg, To)
    _ccc_close(Cg, Co)
    # independent library GEMM for T(1,1) on every record
    n1 = ((codes >> 1) & 1) + (codes & 1)
    n1 = n1.to(torch.int8)
    K = (n_f + 31) // 32 * 32
    A = torch.zeros((n_v, K), dtype=torch.int8, device="cuda")
    A[:, :n_f] = n1
    del n1
    G = torch._int_mm(A, A.t().contiguous())
    iu = torch.triu_indices(n_v, n_v, 1, device="cuda")
    assert bool((G[iu[0], iu[1]] == T[:, 3]).all())


# ------------------------------------------------------------------- 3-way
def _check_3way_full(codes, n_stages=1, flags=TAL | F64 | CK, gamma=oracle.GAMMA):
    n_v, n_f = codes.shape
    To, Co = oracle.all_triples(codes, gamma)
    packed = ccc.ccc_pack(codes.cuda())
    ws = ccc.ccc_3way_prepare(packed, n_f, gamma)
    Ts, Cs, cks = [], [], 0
    for st in range(n_stages):
        T, C, ck = ccc.ccc_3way_stage(n_v, n_f, n_stages, st, ws, out_flags=flags, gamma=gamma)
        if flags & TAL:
            Ts.append(_t(T))
        if flags & (F64 | F32):
            Cs.append(C.cpu().numpy())
        if flags & CK:
            cks = (cks + ccc.checksum_int(ck)) % (1 << 128)
    if flags & TAL:
        np.testing.assert_array_equal(np.concatenate(Ts), To)
    if flags & F64:
        _ccc_close(np.concatenate(Cs), Co)
    if flags & F32:
        _ccc_close(np.concatenate(Cs), Co, rtol=1e-6)
    if flags & CK:
        assert cks == oracle.checksum(3, oracle.triple_list(n_v), To)


@pytest.mark.parametrize("n_v,n_f", [(3, 1), (4, 65), (5, 127), (40, 200), (130, 65),
                                     (131, 300), (260, 129)])
def test_3way_full(n_v, n_f):
    _check_3way_full(_codes("random", n_v, n_f, seed=n_v + n_f))


@pytest.mark.parametrize("n_v,n_f,n_stages", [(385, 77, 1), (385, 77, 5), (513, 130, 3), (300, 64, 7)])
def test_3way_pivot_pairs_full_epilogue(n_v, n_f, n_stages):
    """The flag-free FULL epilogue (tallies + fp64 CCC, gamma = 2/3) on the pivot-pair units:
    several 128-row tiles and 256-column tiles, stages that cut the pivot range mid-pair
    (odd pivot counts per tile leave the follower CTA without a pivot), aligned record
    groups with every row offset mod 4 -- against the oracle record by record."""
    _check_3way_full(_codes("random", n_v, n_f, seed=n_v * 7 + n_stages), n_stages=n_stages, flags=TAL | F64)
    _check_3way_full(_codes("hwe", n_v, n_f, seed=n_v + n_stages), n_stages=n_stages, flags=TAL | F64 | CK)


def test_3way_stages_and_variants():
    codes = _codes("hwe", 150, 333)
    _check_3way_full(codes, n_stages=7)
    _check_3way_full(codes, n_stages=3, flags=TAL | F32)
    _check_3way_full(_codes("planted", 90, 250), n_stages=2)
    _check_3way_full(torch.full((70, 130), 3, dtype=torch.uint8))


@pytest.mark.parametrize("gamma", [0.0, 0.5, 1.0])
def test_3way_general_gamma(gamma):
    """gamma != 2/3 takes the epilogue that reads the stored weights w (the integer form
    only holds for the paper's 2/3)."""
    _check_3way_full(_codes("hwe", 140, 301), n_stages=2, flags=TAL | F64, gamma=gamma)
    _check_3way_full(_codes("random", 70, 97), flags=F32, gamma=gamma)


def test_3way_C4_full_size_stage_sampled():
    """configs[3]: 4,096 x 16,384, 16 stages; first and last stage checked on samples."""
    n_v, n_f, n_st = 4096, 16384, 16
    codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
    packed = ccc.ccc_pack(codes)
    ws = ccc.ccc_3way_prepare(packed, n_f)
    codes_h = codes.cpu()
    rng = np.random.default_rng(4)
    for st in (0, n_st - 1):
        ib, ie, rb, rc = ccc.ccc_stage_range(n_v, n_st, st)
        T, C, _ = ccc.ccc_3way_stage(n_v, n_f, n_st, st, ws, out_flags=TAL | F64)
        assert bool((T.sum(1, dtype=torch.int64) == 8 * n_f).all())
        trip = set()
        for _ in range(1500):
            i = int(rng.integers(ib, ie))
            if i > n_v - 3:
                continue
            j = int(rng.integers(i + 1, n_v - 1))
            k = int(rng.integers(j + 1, n_v))
            trip.add((i, j, k))
            trip.add((i, i + 1, n_v - 1))
            trip.add((i, j, j + 1))
        trip = np.array(sorted(trip), dtype=np.int64)
        rows = torch.tensor([ccc.ccc_triple_index(n_v, *map(int, t)) - rb for t in trip],
                            device="cuda")
        To, Co = oracle.triples(codes_h, trip)
        np.testing.assert_array_equal(_t(T[rows]), To)
        _ccc_close(C[rows].cpu().numpy(), Co)
        del T, C
        torch.cuda.empty_cache()


# ------------------------------------------------------------------- multi-GPU schedules
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_block_circulant_units_on_one_gpu(P):
    """Every rank's block-circulant units (diagonal, off-diagonal, split antipodal block)
    computed by the CUDA kernels from per-block packed data; the union equals the
    single-GPU result record for record and the checksums agree."""
    from paper_1705_08213_b200 import decomp
    n_v, n_f = 1100, 333
    codes = _codes("random", n_v, n_f, seed=21)
    To, Co = oracle.all_pairs(codes)
    bounds = decomp.block_bounds(n_v, P)
    packed = [ccc.ccc_pack(codes[lo:hi].contiguous().cuda()) for lo, hi in bounds]
    exp = [ccc.ccc_expand(p, n_f) for p in packed]
    flags = TAL | F64 | CK
    total_ck = 0
    seen = np.zeros(len(To), dtype=np.int64)
    for r in range(P):
        ck = torch.zeros(2, dtype=torch.int64, device="cuda")
        for u in decomp.plan_2way(P, r, bounds):
            m = decomp.unit2_records(u, bounds)
            T = torch.empty((max(m, 1), 4), dtype=torch.int32, device="cuda")
            C = torch.empty((max(m, 1), 4), dtype=torch.float64, device="cuda")
            Na, sa, wa = exp[u.a]
            Nb, sb, wb = exp[u.b]
            ccc.ccc_2way_block(Na, sa, wa, bounds[u.a][0], u.a_lo, u.a_hi, Nb, sb, wb,
                               bounds[u.b][0], u.diag, n_f, flags, T, C, ck)
            rows = np.array([ccc.ccc_pair_index(n_v, i, j) for i, j in decomp.unit2_pairs(u, bounds)],
                            dtype=np.int64)
            if m:
                np.testing.assert_array_equal(_t(T)[:m], To[rows])
                _ccc_close(C.cpu().numpy()[:m], Co[rows])
                seen[rows] += 1
        total_ck = (total_ck + ccc.checksum_int(ck)) % (1 << 128)
    assert np.all(seen == 1)
    assert total_ck == oracle.checksum(2, oracle.pair_list(n_v), To)


def _nccl_worker(rank, world, port, n_v, n_f, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    from paper_1705_08213_b200 import decomp, dist as cdist
    bounds = decomp.block_bounds(n_v, world)
    lo, hi = bounds[rank]
    be = cdist.CudaBackend(n_f, ccc.GAMMA, TAL | CK)
    ring = cdist.Ring2Way(be, bounds, rank, world)
    codes = synthgen.random_codes(hi - lo, n_f, seed=5, row0=lo, device="cuda")
    ring.run(be.pack(codes))
    q.put(cdist.checksum_total(ring.ck))
    dist.destroy_process_group()


def test_ring_nccl_two_gpus():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    n_v, n_f = 900, 500
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_nccl_worker, args=(r, 2, port, n_v, n_f, q)) for r in range(2)]
    [p.start() for p in ps]
    cks = [q.get(timeout=300) for _ in range(2)]
    [p.join(timeout=60) for p in ps]
    To, _ = oracle.all_pairs(synthgen.random_codes(n_v, n_f, seed=5))
    assert cks[0] == cks[1] == oracle.checksum(2, oracle.pair_list(n_v), To)


def _gloo_ring_worker(rank, world, port, n_v2, n_v3, n_f, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1705_08213_b200 import decomp, dist as cdist
    be = cdist.CudaBackend(n_f, ccc.GAMMA, TAL | CK)
    res = {"rank": rank}
    bounds = decomp.block_bounds(n_v2, world)
    lo, hi = bounds[rank]
    r2 = cdist.Ring2Way(be, bounds, rank, world)
    r2.run(be.pack(synthgen.random_codes(hi - lo, n_f, seed=5, row0=lo, device="cuda")))
    res["ck2"] = cdist.checksum_total(r2.ck)
    bounds = decomp.block_bounds(n_v3, world)
    lo, hi = bounds[rank]
    r3 = cdist.Ring3Way(be, bounds, rank, world, max_records=3000)
    r3.run(be.pack(synthgen.random_codes(hi - lo, n_f, seed=6, row0=lo, device="cuda")))
    res["ck3"] = cdist.checksum_total(r3.ck)
    dist.destroy_process_group()
    q.put(res)


@pytest.mark.parametrize("world", [2, 3])
def test_rings_multi_rank_one_gpu(world):
    """Ring2Way / Ring3Way with the CUDA backend at world 2 and 3: every rank a process on
    cuda:0 (gloo, packed blocks staged through host memory -- the only multi-rank form a
    one-GPU box can run); the ranks' checksums add up to the oracle's over all pairs and
    all triples."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    n_v2, n_v3, n_f = 700, 130, 333
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_ring_worker, args=(r, world, port, n_v2, n_v3, n_f, q))
          for r in range(world)]
    [p.start() for p in ps]
    res = [q.get(timeout=300) for _ in range(world)]
    [p.join(timeout=60) for p in ps]
    T2, _ = oracle.all_pairs(synthgen.random_codes(n_v2, n_f, seed=5))
    T3, _ = oracle.all_triples(synthgen.random_codes(n_v3, n_f, seed=6))
    ck2 = oracle.checksum(2, oracle.pair_list(n_v2), T2)
    ck3 = oracle.checksum(3, oracle.triple_list(n_v3), T3)
    for r in res:
        assert r["ck2"] == ck2 and r["ck3"] == ck3, r["rank"]


@pytest.mark.parametrize("P,gamma", [(1, oracle.GAMMA), (2, oracle.GAMMA), (3, oracle.GAMMA),
                                     (4, oracle.GAMMA), (3, 0.25)])
def test_tetrahedral_units_on_one_gpu(P, gamma):
    """Every rank's tetrahedral 3-way units ({A,A,A}, {D,D,S} both orders, the three
    parts of {A<B<C}) through ccc_3way_unit on per-block expanded data; union equals the
    single-GPU result triple for triple and the unit checksums add up."""
    from paper_1705_08213_b200 import decomp
    n_v, n_f = 150, 197
    codes = _codes("random", n_v, n_f, seed=31)
    To, Co = oracle.all_triples(codes, gamma)
    # global pairwise G by the 2-way kernel on the whole matrix (what each rank builds
    # after the all-gather)
    N, s, w = ccc.ccc_expand(ccc.ccc_pack(codes.cuda()), n_f)
    G = torch.zeros((n_v, n_v), dtype=torch.int32, device="cuda")
    ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, 0, g=G, ldg=n_v)
    bounds = decomp.block_bounds(n_v, P)
    exp = [ccc.ccc_expand(ccc.ccc_pack(codes[lo:hi].contiguous().cuda()), n_f, gamma)
           for lo, hi in bounds]
    blks = [ccc.block(*exp[b], bounds[b][0]) for b in range(P)]
    seen = np.zeros(len(To), dtype=np.int64)
    total_ck = 0
    for r in range(P):
        for u in decomp.plan_3way(P, r, bounds):
            ck = torch.zeros(2, dtype=torch.int64, device="cuda")
            T, C, ck = ccc.ccc_3way_unit(blks[u.pb], u.p_lo, u.p_hi, blks[u.mb], u.m_lo, u.m_hi,
                                         blks[u.nb], u.n_lo, u.n_hi, u.order, G, n_f,
                                         TAL | F64 | CK, checksum=ck, gamma=gamma)
            tr = list(decomp.unit3_triples(u, bounds))
            assert T.shape[0] == len(tr) == decomp.unit3_count(u, bounds)
            if not tr:
                continue
            rows = np.array([ccc.ccc_triple_index(n_v, *t) for t in tr], dtype=np.int64)
            np.testing.assert_array_equal(_t(T), To[rows])
            _ccc_close(C.cpu().numpy(), Co[rows])
            seen[rows] += 1
            total_ck = (total_ck + ccc.checksum_int(ck)) % (1 << 128)
    assert np.all(seen == 1)
    assert total_ck == oracle.checksum(3, oracle.triple_list(n_v), To)


def test_3way_unit_pivot_subranges_as_stages():
    """A distinct-block unit and a {D,D,S} unit split into pivot sub-ranges (stages) give
    the same records as the whole unit."""
    from paper_1705_08213_b200 import decomp
    n_v, n_f = 120, 300
    codes = _codes("hwe", n_v, n_f)
    N, s, w = ccc.ccc_expand(ccc.ccc_pack(codes.cuda()), n_f)
    G = torch.zeros((n_v, n_v), dtype=torch.int32, device="cuda")
    ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, 0, g=G, ldg=n_v)
    bounds = decomp.block_bounds(n_v, 3)
    exp = [ccc.ccc_expand(ccc.ccc_pack(codes[lo:hi].contiguous().cuda()), n_f) for lo, hi in bounds]
    b = [ccc.block(*exp[i], bounds[i][0]) for i in range(3)]
    for (pb, mb, nb, order) in [(1, 0, 2, ("m", "p", "n")), (2, 2, 0, ("n", "p", "m"))]:
        n_p = bounds[pb][1] - bounds[pb][0]
        full, _, _ = ccc.ccc_3way_unit(b[pb], 0, n_p, b[mb], 0, b[mb].rows, b[nb], 0, b[nb].rows,
                                       order, G, n_f, TAL)
        parts = []
        for lo, hi in [(0, 7), (7, 20), (20, n_p)]:
            T, _, _ = ccc.ccc_3way_unit(b[pb], lo, hi, b[mb], 0, b[mb].rows, b[nb], 0,
                                        b[nb].rows, order, G, n_f, TAL)
            parts.append(_t(T))
        np.testing.assert_array_equal(np.concatenate(parts), _t(full))


def _ring_world1(q, port, n_v2, n_v3, n_f):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    from paper_1705_08213_b200 import decomp, dist as cdist
    res = {}
    be = cdist.CudaBackend(n_f, ccc.GAMMA, TAL | CK)
    codes = synthgen.random_codes(n_v2, n_f, seed=9, device="cuda")
    r2 = cdist.Ring2Way(be, decomp.block_bounds(n_v2, 1), 0, 1)
    r2.run(be.pack(codes))
    res["ck2"] = cdist.checksum_total(r2.ck)
    codes = synthgen.random_codes(n_v3, n_f, seed=9, device="cuda")
    r3 = cdist.Ring3Way(be, decomp.block_bounds(n_v3, 1), 0, 1, max_records=5000)
    pieces = []
    r3.run(be.pack(codes), sink=lambda u, lo, hi, out: pieces.append((lo, hi, _t(out[0]).tolist())))
    res["ck3"] = cdist.checksum_total(r3.ck)
    res["pieces"] = pieces
    dist.destroy_process_group()
    q.put(res)


def test_rings_world1_nccl():
    """The CUDA backend methods of Ring2Way / Ring3Way (expand into the full buffer, own-block
    and full G, staged units) under a 1-rank NCCL group."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    n_v2, n_v3, n_f = 300, 90, 211
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_ring_world1, args=(q, port, n_v2, n_v3, n_f))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    T2, _ = oracle.all_pairs(synthgen.random_codes(n_v2, n_f, seed=9))
    assert res["ck2"] == oracle.checksum(2, oracle.pair_list(n_v2), T2)
    T3, _ = oracle.all_triples(synthgen.random_codes(n_v3, n_f, seed=9))
    assert res["ck3"] == oracle.checksum(3, oracle.triple_list(n_v3), T3)
    got = np.concatenate([np.array(t, dtype=np.int64).reshape(-1, 8) for _, _, t in res["pieces"]])
    np.testing.assert_array_equal(got, T3)
    assert len(res["pieces"]) > 1                     # the stage split was exercised


def test_3way_epilogue_form_boundaries():
    """The 3-way epilogue picks its cell formula by n_f: T U_p U_m < 2^52 (n_f <= 38,000:
    one DFMA per cell) or not (two-multiply form), and 8 n_f < 2^23 for the FP32-only
    fp32-CCC path.  Records on both sides of each boundary against the oracle."""
    for n_v, n_f, flags in ((12, 38000, TAL | F64), (12, 38100, TAL | F64 | CK),
                            (6, (1 << 20) - 8, TAL | F32), (6, (1 << 20) + 8, TAL | F32)):
        _check_3way_full(_codes("random", n_v, n_f, seed=n_f), flags=flags)


def test_2way_C3_block_full_size():
    """configs[2] (160,000 x 100,000, block-circulant over 8 GPUs): rank 0's ring-step-1
    unit -- the full 20,000 x 20,000 off-diagonal block pair at n_f = 100,000, in the
    launch configuration of the multi-GPU bench (blocks aligned to 256) -- sampled pairs
    against the brute force, sum T = 4 n_f on every record."""
    from paper_1705_08213_b200 import decomp
    n_v, n_f, P = 160000, 100000, 8
    bounds = decomp.block_bounds(n_v, P, align=256)
    u = [x for x in decomp.plan_2way(P, 0, bounds) if not x.diag][0]
    (a0, a1), (b0, b1) = bounds[u.a], bounds[u.b]
    exp = []
    for lo, hi in ((a0, a1), (b0, b1)):
        c = synthgen.random_codes(hi - lo, n_f, seed=1, device="cuda", row0=lo)
        exp.append(ccc.ccc_expand(ccc.ccc_pack(c), n_f))
        del c
    m = decomp.unit2_records(u, bounds)
    T = torch.empty((m, 4), dtype=torch.int32, device="cuda")
    C = torch.empty((m, 4), dtype=torch.float64, device="cuda")
    ccc.ccc_2way_block(*exp[0], a0, u.a_lo, u.a_hi, *exp[1], b0, False, n_f, TAL | F64, T, C)
    torch.cuda.synchronize()
    assert bool((T.sum(1, dtype=torch.int64) == 4 * n_f).all())
    rng = np.random.default_rng(8)
    nb = b1 - b0
    loc = [(int(i), int(j)) for i, j in zip(rng.integers(u.a_lo, u.a_hi, 700), rng.integers(0, nb, 700))]
    loc += [(u.a_lo, 0), (u.a_hi - 1, nb - 1), (u.a_lo, nb - 1), (u.a_hi - 1, 0)]
    rows = torch.tensor([(i - u.a_lo) * nb + j for i, j in loc], device="cuda")
    glob = sorted({a0 + i for i, _ in loc} | {b0 + j for _, j in loc})
    pos = {g: t for t, g in enumerate(glob)}
    sub = torch.cat([synthgen.random_codes(1, n_f, seed=1, row0=g) for g in glob])
    To, Co = oracle.pairs(sub, np.array([(pos[a0 + i], pos[b0 + j]) for i, j in loc], dtype=np.int64))
    np.testing.assert_array_equal(_t(T[rows]), To)
    _ccc_close(C[rows].cpu().numpy(), Co)


def test_3way_C5_unit_full_size():
    """configs[4] (16,384 x 32,768, tetrahedral over 8 GPUs): a {A<B<C} part of rank 1's
    plan at full size (blocks of 2,048 vectors, n_f = 32,768, the pairwise G of all 16,384
    vectors by the 2-way kernel), first 4 pivots: sampled triples against the brute force
    and sum T = 8 n_f on every record."""
    from paper_1705_08213_b200 import decomp
    n_v, n_f, P = 16384, 32768, 8
    bounds = decomp.block_bounds(n_v, P, align=256)
    codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
    N, s, w = ccc.ccc_expand(ccc.ccc_pack(codes), n_f)
    del codes
    G = torch.zeros((n_v, n_v), dtype=torch.int32, device="cuda")
    ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, 0, g=G, ldg=n_v)
    blk = lambda b: ccc.block(N[bounds[b][0]:bounds[b][1]], s[bounds[b][0]:bounds[b][1]],
                              w[bounds[b][0]:bounds[b][1]], bounds[b][0])
    u = [x for x in decomp.plan_3way(P, 1, bounds) if x.order == ("m", "p", "n")][0]
    p_hi = u.p_lo + 4
    T, C, _ = ccc.ccc_3way_unit(blk(u.pb), u.p_lo, p_hi, blk(u.mb), u.m_lo, u.m_hi, blk(u.nb), u.n_lo,
                                u.n_hi, u.order, G, n_f, TAL | F64)
    torch.cuda.synchronize()
    nm, nn = u.m_hi - u.m_lo, u.n_hi - u.n_lo
    assert T.shape[0] == 4 * nm * nn
    assert bool((T.sum(1, dtype=torch.int64) == 8 * n_f).all())
    rng = np.random.default_rng(9)
    loc = [(int(p), int(m), int(k)) for p, m, k in
           zip(rng.integers(0, 4, 500), rng.integers(0, nm, 500), rng.integers(0, nn, 500))]
    loc += [(0, 0, 0), (3, nm - 1, nn - 1)]
    rows = torch.tensor([(p * nm + m) * nn + k for p, m, k in loc], device="cuda")
    p0, m0, n0 = bounds[u.pb][0] + u.p_lo, bounds[u.mb][0] + u.m_lo, bounds[u.nb][0] + u.n_lo
    trip = [(m0 + m, p0 + p, n0 + k) for p, m, k in loc]          # canonical (i < j < k)
    glob = sorted({g for t in trip for g in t})
    pos = {g: t for t, g in enumerate(glob)}
    sub = torch.cat([synthgen.random_codes(1, n_f, seed=1, row0=g) for g in glob])
    To, Co = oracle.triples(sub, np.array([[pos[x] for x in t] for t in trip], dtype=np.int64))
    np.testing.assert_array_equal(_t(T[rows]), To)
    _ccc_close(C[rows].cpu().numpy(), Co)


@pytest.mark.parametrize("n_stages", [1, 3, 7])
def test_3way_host_stage_streaming(n_stages):
    """f2 stage streaming: host codes in, every stage's records streamed to host buffers
    while the next stage computes; equals the oracle record for record."""
    n_v, n_f = 90, 333
    codes = _codes("random", n_v, n_f, seed=50 + n_stages)
    T, C, ck = ccc.ccc_3way_host(codes.contiguous(), out_flags=TAL | F64 | CK, n_stages=n_stages)
    To, Co = oracle.all_triples(codes)
    np.testing.assert_array_equal(T.numpy().astype(np.int64) & 0xFFFFFFFF, To)
    _ccc_close(C.numpy(), Co)
    assert ccc.checksum_int(ck) == oracle.checksum(3, oracle.triple_list(n_v), To)


def _golden_vec(spec):
    out = []
    for part in spec.split(","):
        if "*" in part:
            c, n = part.split("*")
            out += [int(c)] * int(n)
        else:
            out.append(int(part))
    return out


def test_golden_hand_values_through_the_kernels():
    """SPEC's hand values and our n_f = 1 figure-style examples (tests/golden/) through the
    CUDA path: tallies exact, CCC equal to the exact fractions (independent of the oracle)."""
    from fractions import Fraction
    from conftest import read_golden
    for name, inputs, expected, _ in read_golden("spec_hand_values.txt"):
        if name not in ("pair_tally", "ccc2", "ccc3", "reconstruct3"):
            continue
        a = dict(kv.strip().split("=") for kv in inputs.split(";"))
        vs = [_golden_vec(a[k]) for k in ("vi", "vj", "vk") if k in a]
        codes = torch.tensor(vs, dtype=torch.uint8).cuda()
        want = [Fraction(x) for x in expected.split("=")[1].split(",")]
        if name in ("pair_tally", "ccc2"):
            T, C, _ = ccc.two_way(codes, out_flags=TAL | F64)
        else:
            T, C, _ = ccc.three_way(codes, out_flags=TAL | F64)
        torch.cuda.synchronize()
        if name in ("pair_tally", "reconstruct3"):
            assert list(_t(T)[0]) == [int(x) for x in want], name
        else:
            _ccc_close(C.cpu().numpy()[0], np.array([float(x) for x in want]))
    for way, cs, expected, _ in read_golden("fig_examples_nf1.txt"):
        codes = torch.tensor([[int(c)] for c in cs.split()], dtype=torch.uint8).cuda()
        T = (ccc.two_way if way == "2" else ccc.three_way)(codes, out_flags=TAL)[0]
        torch.cuda.synchronize()
        assert list(_t(T)[0]) == [int(x) for x in expected.split(",")]


def test_expand_ignores_garbage_tail():
    """codes past n_f in the last packed word are not elements -- expand masks
    them, so caller-made packed rows with non-zero padding give the same N, s, w."""
    for n_f in (100, 65, 1):
        codes = _codes("random", 9, n_f, seed=n_f)
        packed = ccc.ccc_pack(codes.cuda())
        dirty = packed.clone()
        q = torch.arange(dirty.shape[1] * 4)
        byte_has_tail = torch.zeros(dirty.shape[1], dtype=torch.bool)
        byte_has_tail[(q[q >= n_f] // 4).unique()] = True
        for b in torch.nonzero(byte_has_tail).flatten().tolist():
            keep = 0
            for e in range(4):
                if 4 * b + e < n_f:
                    keep |= 3 << (2 * e)
            dirty[:, b] = (dirty[:, b] & keep) | (0xFF & ~keep)
        assert not torch.equal(dirty, packed)
        N0, s0, w0 = ccc.ccc_expand(packed, n_f)
        N1, s1, w1 = ccc.ccc_expand(dirty, n_f)
        assert torch.equal(N0, N1) and torch.equal(s0, s1) and torch.equal(w0, w1)
        np.testing.assert_array_equal(s1.cpu().numpy(), oracle.allele_sums(codes)[:, 1])


def test_3way_unit_rejects_noncanonical_orders():
    """with a shared pivot/row block the order must put p before m (with a shared
    row/column block m before n); other orders are INVALID_ARGUMENT, not silent garbage."""
    n_v, n_f = 64, 200
    N, s, w = ccc.ccc_expand(ccc.ccc_pack(_codes("random", n_v, n_f, seed=3).cuda()), n_f)
    G = torch.zeros((n_v, n_v), dtype=torch.int32, device="cuda")
    ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, 0, g=G, ldg=n_v)
    A = ccc.block(N[:32], s[:32], w[:32], 0)
    B = ccc.block(N[32:], s[32:], w[32:], 32)
    for order in range(6):
        ok_pm = order in (0, 1, 4)           # p before m
        ok_mn = order in (0, 2, 3)           # m before n
        for (bp, bm, bn, ok) in ((A, A, B, ok_pm), (B, A, A, ok_mn), (A, A, A, order == 0)):
            if ok:
                ccc.ccc_3way_unit(bp, 0, 2, bm, 0, 32, bn, 0, 32, order, G, n_f, TAL)
            else:
                with pytest.raises(ValueError, match="order must put"):
                    ccc.ccc_3way_unit(bp, 0, 2, bm, 0, 32, bn, 0, 32, order, G, n_f, TAL)


@pytest.mark.parametrize("n_v,n_f", [(2, 1), (3, 65), (127, 129), (129, 1000), (300, 777), (700, 4096),
                                     (1100, 2049)])
def test_2way_codes_overlapped_expand(n_v, n_f):
    """ccc_2way_codes (unpacked codes -> expand_codes -> tally GEMM) writes exactly ccc_2way's
    records on the packed path, and the oracle's; called twice on one workspace."""
    codes = _codes("random", n_v, n_f, seed=n_v * 7 + n_f)
    cd = codes.cuda()
    ws = ccc.workspace(2, n_v, n_f)
    T1, C1, k1 = ccc.ccc_2way(ccc.ccc_pack(cd), n_f, out_flags=TAL | F64 | CK)
    for _ in range(2):
        T2, C2, k2 = ccc.ccc_2way_codes(cd, out_flags=TAL | F64 | CK, ws=ws)
        torch.cuda.synchronize()
        assert bool((T1 == T2).all()) and bool((C1 == C2).all())
        assert ccc.checksum_int(k1) == ccc.checksum_int(k2)
    To, Co = oracle.all_pairs(codes)
    np.testing.assert_array_equal(_t(T2), To)
    _ccc_close(C2.cpu().numpy(), Co)


def test_2way_codes_c2_shape_equals_packed_path():
    """At configs[1]'s shape (20,000 x 50,000, bench.py's step): ccc_2way_codes' checksum
    equals the packed path's and a sample of records the oracle's."""
    n_v, n_f = 20000, 50000
    codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
    _, _, k1 = ccc.ccc_2way(ccc.ccc_pack(codes), n_f, out_flags=CK)
    T, C, k2 = ccc.ccc_2way_codes(codes, out_flags=TAL | F64 | CK)
    torch.cuda.synchronize()
    assert ccc.checksum_int(k1) == ccc.checksum_int(k2)
    rng = np.random.default_rng(3)
    i = rng.integers(0, n_v - 1, 2000)
    j = np.array([rng.integers(a + 1, n_v) for a in i])
    idx = np.stack([i, j], 1)
    rows = torch.tensor([ccc.ccc_pair_index(n_v, int(a), int(b)) for a, b in idx], device="cuda")
    To, Co = oracle.pairs(codes.cpu(), idx)
    np.testing.assert_array_equal(_t(T[rows]), To)
    _ccc_close(C[rows].cpu().numpy(), Co)


def test_2way_codes_compacted_equals_dense_filter():
    """ccc_2way_codes with threshold compaction (f2) keeps exactly the records
    of the dense output whose largest CCC cell exceeds theta, with their tallies and CCC."""
    n_v, n_f = 900, 3001
    codes = synthgen.random_codes(n_v, n_f, seed=41, device="cuda")
    T, C, _ = ccc.ccc_2way_codes(codes, out_flags=TAL | F64)
    mx = C.max(dim=1).values
    theta = float(torch.kthvalue(mx, mx.numel() - 300).values)
    cp = ccc.Compact(theta, 1000, 4)
    ccc.ccc_2way_codes(codes, out_flags=TAL | F64, compact=cp)
    n, keys, Tk, Ck = cp.result()
    want = torch.nonzero(mx > theta).flatten()
    assert n == want.numel() == 300
    idx = ccc.decode_keys(keys, 2).cpu().numpy()
    rows = torch.tensor([ccc.ccc_pair_index(n_v, int(i), int(j)) for i, j in idx], device="cuda")
    assert sorted(rows.tolist()) == want.tolist()
    assert bool((T[rows] == Tk).all()) and bool((C[rows] == Ck).all())

"""Full-size parity on EVERY record (SURVEY §8(c) protocol; VERDICT r1 "next" item 1).

The paper's second synthetic type exists "so that the correctness of every result value
can be verified analytically".  Here the planted type-2 input (seed 3) runs
through exactly the launch configuration bench.py times -- C2: ccc_pack -> ccc_expand ->
ccc_2way_block over the whole 20,000 x 50,000 matrix; C4: ccc_pack -> ccc_3way_prepare ->
16 x ccc_3way_stage into one reused stage buffer -- and every stored record (uint32
tallies + fp64 CCC) is copied back and compared, record by record, with the oracle's
closed form (oracle.planted_check, C + OpenMP on the host cores): tallies bit-exact, CCC
within 1e-12 relative and exactly 0 where the tally is 0.  The allele sums s of the
expand kernel are checked over the full matrix against the brute-force Eq.1 counts of the
oracle (and the closed form), for the planted and the timing (type-1) inputs.
"""

import numpy as np
import pytest
import torch

import oracle
import synthgen

pytestmark = pytest.mark.gpu

ccc = pytest.importorskip("paper_1705_08213_b200.ccc")

TAL, F64 = ccc.OUT_TALLY, ccc.OUT_CCC_F64


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


def check_records(way, L, H, n_f, rec0, T, C, chunk=1 << 25):
    """Copy device records T/C [n][cells] to pinned host buffers chunk by chunk (the next
    chunk's copy overlaps the current chunk's check) and compare every record with the
    oracle's planted closed form.  Returns the summed oracle.planted_check result."""
    n, cells = T.shape
    chunk = max(1, min(chunk, n))
    bufs = [(torch.empty((chunk, cells), dtype=torch.int32, pin_memory=True),
             torch.empty((chunk, cells), dtype=torch.float64, pin_memory=True)) for _ in range(2)]
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    events = [torch.cuda.Event(), torch.cuda.Event()]
    tot = {"bad_tallies": 0, "bad_ccc": 0, "first_bad": -1, "max_rel": 0.0, "records": 0}

    def issue(k):
        a, b = k * chunk, min(n, (k + 1) * chunk)
        Th, Ch = bufs[k % 2]
        with torch.cuda.stream(stream):
            Th[: b - a].copy_(T[a:b], non_blocking=True)
            Ch[: b - a].copy_(C[a:b], non_blocking=True)
            events[k % 2].record(stream)

    nchunks = (n + chunk - 1) // chunk
    if nchunks:
        issue(0)
    for k in range(nchunks):
        if k + 1 < nchunks:
            issue(k + 1)
        events[k % 2].synchronize()
        a, b = k * chunk, min(n, (k + 1) * chunk)
        Th, Ch = bufs[k % 2]
        r = oracle.planted_check(way, L, H, n_f, rec0 + a, b - a, Th[: b - a], Ch[: b - a])
        tot["bad_tallies"] += r["bad_tallies"]
        tot["bad_ccc"] += r["bad_ccc"]
        tot["max_rel"] = max(tot["max_rel"], r["max_rel"])
        if r["first_bad"] >= 0 and tot["first_bad"] < 0:
            tot["first_bad"] = rec0 + a + r["first_bad"]
        tot["records"] += b - a
    torch.cuda.synchronize()
    return tot


def _s_full_check(codes_dev, s, w, n_f):
    """s (and w) of the expand kernel over the whole matrix vs the brute-force Eq.1 sums."""
    S = oracle.allele_sums(codes_dev.cpu())
    np.testing.assert_array_equal(s.cpu().numpy(), S[:, 1])
    np.testing.assert_allclose(w.cpu().numpy(), 1.0 - oracle.GAMMA * S / (2.0 * n_f), rtol=1e-15, atol=0)


def test_C2_planted_every_record():
    """configs[1] 20,000 x 50,000, planted input, through bench.py's step (ccc_2way_codes:
    expand_codes + the flag-free FULL tally kernel): all 199,990,000 records (9.6 GB)."""
    n_v, n_f = 20000, 50000
    codes, L, H, _ = synthgen.planted_codes(n_v, n_f, seed=3, device="cuda")
    N, s, w = ccc.ccc_expand_codes(codes)
    _s_full_check(codes, s, w, n_f)
    np.testing.assert_array_equal(s.cpu().numpy(), oracle.planted_sums(L, H, n_f)[:, 1])
    del N, s, w
    m = ccc.ccc_num_unique(2, n_v)
    T = torch.empty((m, 4), dtype=torch.int32, device="cuda")
    C = torch.empty((m, 4), dtype=torch.float64, device="cuda")
    ccc.ccc_2way_codes(codes, ccc.GAMMA, TAL | F64, T, C)
    del codes
    r = check_records(2, L, H, n_f, 0, T, C)
    assert r["records"] == m
    assert (r["bad_tallies"], r["bad_ccc"]) == (0, 0), r
    assert r["max_rel"] <= 1e-12


def test_C2_planted_every_record_packed_path():
    """The same on the packed path (pack + expand + ccc_2way_block: the ring's kernels)."""
    n_v, n_f = 20000, 50000
    codes, L, H, _ = synthgen.planted_codes(n_v, n_f, seed=3, device="cuda")
    packed = ccc.ccc_pack(codes)
    del codes
    N, s, w = ccc.ccc_expand(packed, n_f)
    np.testing.assert_array_equal(s.cpu().numpy(), oracle.planted_sums(L, H, n_f)[:, 1])
    del packed
    m = ccc.ccc_num_unique(2, n_v)
    T = torch.empty((m, 4), dtype=torch.int32, device="cuda")
    C = torch.empty((m, 4), dtype=torch.float64, device="cuda")
    ccc.ccc_2way_block(N, s, w, 0, 0, n_v, N, s, w, 0, True, n_f, TAL | F64 | ccc.OUT_CHECKSUM, T, C,
                       torch.zeros(2, dtype=torch.int64, device="cuda"))
    r = check_records(2, L, H, n_f, 0, T, C)
    assert r["records"] == m
    assert (r["bad_tallies"], r["bad_ccc"]) == (0, 0), r
    assert r["max_rel"] <= 1e-12


def test_C2_timing_input_allele_sums_full():
    """The bench's own input (type 1, seed 1): s and w of every one of the 20,000 vectors
    against the brute-force Eq.1 counts."""
    n_v, n_f = 20000, 50000
    codes = synthgen.random_codes(n_v, n_f, seed=1, device="cuda")
    N, s, w = ccc.ccc_expand(ccc.ccc_pack(codes), n_f)
    _s_full_check(codes, s, w, n_f)
    N2, s2, w2 = ccc.ccc_expand_codes(codes)       # the bench step's fused pass: bit-identical
    assert bool((N2 == N).all()) and bool((s2 == s).all()) and bool((w2 == w).all())


def test_C4_planted_every_record_all_stages():
    """configs[3] 4,096 x 16,384, planted input, 16 stages in bench.py's configuration
    (one stage buffer reused): all 11,444,858,880 records (1.1 TB) checked."""
    n_v, n_f, n_st = 4096, 16384, 16
    codes, L, H, _ = synthgen.planted_codes(n_v, n_f, seed=3, device="cuda")
    packed = ccc.ccc_pack(codes)
    ws = ccc.ccc_3way_prepare(packed, n_f)
    rmax = max(ccc.ccc_stage_range(n_v, n_st, st)[3] for st in range(n_st))
    T = torch.empty((rmax, 8), dtype=torch.int32, device="cuda")
    C = torch.empty((rmax, 8), dtype=torch.float64, device="cuda")
    total = 0
    for st in range(n_st):
        ib, ie, rb, rc = ccc.ccc_stage_range(n_v, n_st, st)
        ccc.ccc_3way_stage(n_v, n_f, n_st, st, ws, TAL | F64, T[:rc], C[:rc])
        r = check_records(3, L, H, n_f, rb, T[:rc], C[:rc])
        assert r["records"] == rc
        assert (r["bad_tallies"], r["bad_ccc"]) == (0, 0), (st, r)
        assert r["max_rel"] <= 1e-12
        total += rc
    assert total == ccc.ccc_num_unique(3, n_v)


def test_ring2way_phases_planted_every_record():
    """2-way phases as the c3 bench runs them: Ring2Way at world 1 with a
    record bound that cuts the diagonal block into many row bands written into one reused
    buffer; every band's records checked against the planted closed form before the next
    band overwrites them."""
    from paper_1705_08213_b200 import decomp
    from paper_1705_08213_b200.dist import CudaBackend, Ring2Way
    n_v, n_f = 12000, 30000
    codes, L, H, _ = synthgen.planted_codes(n_v, n_f, seed=3, device="cuda")
    be = CudaBackend(n_f, oracle.GAMMA, TAL | F64)
    ring = Ring2Way(be, decomp.block_bounds(n_v, 1, align=256), 0, 1, max_records=7_000_000)
    assert ring.n_phases() >= 10
    seen = []

    def sink(u, lo, hi, out):
        rec0 = lo * (2 * n_v - lo - 1) // 2          # first pair (lo, lo+1) of the band
        r = check_records(2, L, H, n_f, rec0, out[0], out[1])
        assert (r["bad_tallies"], r["bad_ccc"]) == (0, 0), (lo, hi, r)
        seen.append(r["records"])

    ring.run(ccc.ccc_pack(codes), sink=sink)
    assert len(seen) == ring.n_phases() and sum(seen) == n_v * (n_v - 1) // 2


def test_ring3way_pieces_planted_every_record():
    """3-way pieces as the c5 bench runs them: Ring3Way at world 1 cuts the
    {A,A,A} unit into pivot pieces of bounded record count in one reused buffer; every
    piece checked against the planted closed form."""
    from paper_1705_08213_b200 import decomp
    from paper_1705_08213_b200.dist import CudaBackend, Ring3Way
    n_v, n_f = 2048, 8192
    codes, L, H, _ = synthgen.planted_codes(n_v, n_f, seed=3, device="cuda")
    be = CudaBackend(n_f, oracle.GAMMA, TAL | F64)
    ring = Ring3Way(be, decomp.block_bounds(n_v, 1, align=256), 0, 1, max_records=100_000_000)
    seen = []

    def sink(u, p_lo, p_hi, out):
        rec0 = sum((n_v - 1 - i) * (n_v - 2 - i) // 2 for i in range(p_lo))   # triples before p_lo
        r = check_records(3, L, H, n_f, rec0, out[0], out[1])
        assert (r["bad_tallies"], r["bad_ccc"]) == (0, 0), (p_lo, p_hi, r)
        seen.append(r["records"])

    ring.run(ccc.ccc_pack(codes), sink=sink)
    assert len(seen) >= 10 and sum(seen) == n_v * (n_v - 1) * (n_v - 2) // 6

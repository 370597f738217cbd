"""C-ABI library: loads, exports every symbol include/ccc.h declares, host helpers are
right, and arguments are validated before any launch (CPU only, no compute calls)."""
import ctypes
import re
import subprocess

import numpy as np
import pytest

import oracle
from paper_1705_08213_b200 import ccc


def test_library_exports_every_header_symbol():
    lib = ccc.lib()
    declared = ccc.header_symbols()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(lib, name), name
        assert name in ccc._SIGS, f"binding lacks {name}"
    out = subprocess.run(["nm", "-D", "--defined-only", ccc.lib_path()], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (ccc_[a-z0-9_]+)", out))
    assert set(declared) <= exported


def test_sm100a_cubin_has_tcgen05_and_tma():
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", ccc.lib_path()],
                          capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass            # tcgen05.mma kind::i8
    assert "UTMALDG" in sass            # TMA tile loads
    assert "LDTM" in sass               # tcgen05.ld
    assert "arch = sm_100a" in sass or "sm_100a" in sass


def test_counts_and_indices_against_enumeration():
    for n in range(0, 9):
        assert ccc.ccc_num_unique(2, n) == len(oracle.pair_list(n))
        assert ccc.ccc_num_unique(3, n) == len(oracle.triple_list(n))
        for r, (i, j) in enumerate(oracle.pair_list(n)):
            assert ccc.ccc_pair_index(n, int(i), int(j)) == r
        for r, (i, j, k) in enumerate(oracle.triple_list(n)):
            assert ccc.ccc_triple_index(n, int(i), int(j), int(k)) == r
    assert ccc.ccc_num_unique(4, 10) == -1
    assert ccc.ccc_pair_index(5, 3, 3) == -1 and ccc.ccc_pair_index(5, 3, 1) == -1
    assert ccc.ccc_triple_index(5, 0, 2, 2) == -1
    n = 160000
    assert ccc.ccc_num_unique(2, n) == n * (n - 1) // 2
    assert ccc.ccc_triple_index(n, n - 3, n - 2, n - 1) == n * (n - 1) * (n - 2) // 6 - 1


def test_strides():
    for n_f, ps, kp in [(1, 16, 128), (64, 16, 128), (65, 32, 128), (128, 32, 128),
                        (129, 48, 256), (50000, 12512, 50048), (100000, 25008, 100096)]:
        assert ccc.ccc_packed_stride(n_f) == ps
        assert ccc.ccc_k_pad(n_f) == kp


@pytest.mark.parametrize("n_v,n_st", [(3, 1), (10, 3), (24, 4), (100, 16), (5, 9)])
def test_stage_ranges_partition_triples(n_v, n_st):
    prev_end, prev_rec = 0, 0
    for s in range(n_st):
        ib, ie, rb, rc = ccc.ccc_stage_range(n_v, n_st, s)
        assert ib == prev_end and rb == prev_rec
        # records of the stage = triples whose first index lies in [ib, ie)
        assert rc == sum(1 for (i, _, _) in oracle.triple_list(n_v) if ib <= i < ie)
        prev_end, prev_rec = ie, rb + rc
    assert prev_end == n_v and prev_rec == n_v * (n_v - 1) * (n_v - 2) // 6


def test_stage_ranges_balanced():
    n_v, n_st = 4096, 16
    tot = n_v * (n_v - 1) * (n_v - 2) // 6
    counts = [ccc.ccc_stage_range(n_v, n_st, s)[3] for s in range(n_st)]
    assert sum(counts) == tot
    assert max(counts) < 1.05 * tot / n_st


def test_validation_before_launch():
    lib = ccc.lib()
    null = None
    # n_f < 1
    assert lib.ccc_pack(ctypes.c_void_p(16), 4, 0, ctypes.c_void_p(16), null) == ccc.ERR_INVALID_ARGUMENT
    # n_f too large
    assert lib.ccc_pack(ctypes.c_void_p(16), 4, 1 << 30, ctypes.c_void_p(16), null) == ccc.ERR_UNSUPPORTED
    # NULL pointers
    assert lib.ccc_pack(null, 4, 10, null, null) == ccc.ERR_INVALID_ARGUMENT
    assert "non-NULL" in lib.ccc_last_error().decode()
    # exclusive CCC flags
    st = lib.ccc_2way(ctypes.c_void_p(256), 4, 10, 2 / 3, ccc.OUT_CCC_F64 | ccc.OUT_CCC_F32,
                      null, ctypes.c_void_p(256), null, ctypes.c_void_p(256), 1 << 20, null, null)
    assert st == ccc.ERR_INVALID_ARGUMENT
    # missing tally buffer
    st = lib.ccc_2way(ctypes.c_void_p(256), 4, 10, 2 / 3, ccc.OUT_TALLY, null, null, null,
                      ctypes.c_void_p(256), 1 << 20, null, null)
    assert st == ccc.ERR_INVALID_ARGUMENT
    # workspace too small
    st = lib.ccc_2way(ctypes.c_void_p(256), 40, 10, 2 / 3, 0, null, null, null,
                      ctypes.c_void_p(256), 16, null, null)
    assert st == ccc.ERR_WORKSPACE
    # bad stage
    out = (ctypes.c_int64 * 4)()
    assert lib.ccc_stage_range(10, 3, 3, ctypes.cast(out, ctypes.c_void_p)) == ccc.ERR_INVALID_ARGUMENT
    with pytest.raises(ValueError):
        ccc.ccc_stage_range(10, 0, 0)
    # empty problems are valid and launch nothing
    assert lib.ccc_2way(null, 1, 10, 2 / 3, 0, null, null, null, null, 0, null, null) == ccc.OK
    assert lib.ccc_3way(null, 2, 10, 2 / 3, 0, 1, 0, null, null, null, null, 0, null, null) == ccc.OK
    assert lib.ccc_last_launch_count() == 0
    # diag block requires A == B
    st = lib.ccc_2way_block(ctypes.c_void_p(256), null, null, 8, 0, 0, 8, ctypes.c_void_p(512),
                            null, null, 8, 0, 1, 10, 2 / 3, 0, null, null, null, null, 0, null, null)
    assert st == ccc.ERR_INVALID_ARGUMENT
    # compacted output: counter required, NaN threshold refused
    cmp = ccc.CccCompact(0.5, 10, 256, None)
    st = lib.ccc_2way(ctypes.c_void_p(256), 40, 10, 2 / 3, 0, null, null, null,
                      ctypes.c_void_p(256), 1 << 30, ctypes.byref(cmp), null)
    assert st == ccc.ERR_INVALID_ARGUMENT and "count_d" in lib.ccc_last_error().decode()
    cmp = ccc.CccCompact(float("nan"), 10, 256, 512)
    st = lib.ccc_2way(ctypes.c_void_p(256), 40, 10, 2 / 3, 0, null, null, null,
                      ctypes.c_void_p(256), 1 << 30, ctypes.byref(cmp), null)
    assert st == ccc.ERR_INVALID_ARGUMENT and "NaN" in lib.ccc_last_error().decode()


def test_workspace_sizes():
    b2 = ccc.ccc_workspace_bytes(2, 20000, 50000)
    assert b2 >= 20000 * 50048 + 20000 * 20
    b3 = ccc.ccc_workspace_bytes(3, 4096, 16384)
    assert b3 >= 4096 * 16384 + 4096 * 4096 * 4
    assert ccc.ccc_workspace_bytes(5, 10, 10) == 0
    assert ccc.ccc_e2e_workspace_bytes(1000, 100, ccc.OUT_TALLY | ccc.OUT_CCC_F64) > 0


def test_header_compiles_as_c_and_links():
    """include/ccc.h is plain C: a C translation unit that takes the address of every
    declared function compiles with gcc and links against libccc.so."""
    import os
    import subprocess
    import tempfile
    syms = ccc.header_symbols()
    src = "#include <stddef.h>\n#include <stdint.h>\n#include \"ccc.h\"\n" \
          "void* table[] = {" + ", ".join(f"(void*)&{s}" for s in syms) + "};\n" \
          "int main(void) { return table[0] == 0; }\n"
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", inc, c, ccc.lib_path(),
                            "-o", os.path.join(d, "t")], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def test_validation_of_later_rows():
    """f1 3-way sparse, f3 field split, f4 baselines: synchronous argument checks."""
    lib = ccc.lib()
    null = None
    # field split: rank outside [0, world), ranges, empty waves launch nothing
    assert lib.ccc_2way_fs_export(ctypes.c_void_p(256), ctypes.c_void_p(256), 100, 64, ctypes.c_void_p(256),
                                  2, 2, 0, 1, null) == ccc.ERR_INVALID_ARGUMENT
    assert lib.ccc_2way_fs_export(ctypes.c_void_p(256), ctypes.c_void_p(256), 100, 64, ctypes.c_void_p(256),
                                  0, 2, 3, 1, null) == ccc.ERR_INVALID_ARGUMENT
    assert lib.ccc_2way_fs_export(null, null, 100, 64, null, 0, 2, 4, 4, null) == ccc.OK
    assert lib.ccc_2way_fs_finish(null, null, 100, 64, 2 / 3, 0, 2, 0, 0, 0, null, null, null, null) == ccc.OK
    assert lib.ccc_2way_fs_finish(ctypes.c_void_p(256), ctypes.c_void_p(256), 100, 64, 2 / 3, 0, 2, 0, 3,
                                  ccc.OUT_TALLY, null, null, null, null) == ccc.ERR_INVALID_ARGUMENT
    # popcount baseline: NULL packed
    assert lib.ccc_2way_popcount(null, 10, 10, 2 / 3, 0, null, null, null, ctypes.c_void_p(256), 1 << 20,
                                 null) == ccc.ERR_INVALID_ARGUMENT
    # sparse 3-way / paper route: small workspace, small scratch
    assert lib.ccc_3way_sparse_prepare(ctypes.c_void_p(256), 10, 10, 2 / 3, ctypes.c_void_p(256), 16,
                                       null) == ccc.ERR_WORKSPACE
    wsb = lib.ccc_sparse3_workspace_bytes(10, 10)
    assert lib.ccc_3way_sparse_stage(10, 10, 2 / 3, 1, 0, ccc.OUT_TALLY, ctypes.c_void_p(256), null, null,
                                     ctypes.c_void_p(256), wsb - 1, null, 0, null) == ccc.ERR_WORKSPACE
    assert lib.ccc_3way_sparse_scratch_bytes(10, 1, 0) == 0      # single pass: no stored forms
    assert lib.ccc_3way_sparse_stage(10, 10, 2 / 3, 1, 0, ccc.OUT_TALLY, null, null, null,
                                     ctypes.c_void_p(256), wsb, null, 0, null) == ccc.ERR_INVALID_ARGUMENT
    assert lib.ccc_3way_paper_scratch_bytes(10, 1, 0) == 2 * 120 * 4
    assert lib.ccc_3way_paper_workspace_bytes(10, 10) > 3 * 10 * 10 * 4
    assert lib.ccc_3way_paper_prepare(null, 2, 10, 2 / 3, null, 0, null) == ccc.OK   # n_v < 3: nothing


def test_product_path_fails_loudly_without_the_library():
    """No CPU fallback: with the library missing, the binding raises instead of computing
    anything (checked in a fresh interpreter so this process's loaded library is untouched)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_1705_08213_b200 import ccc\n"
            "try:\n    ccc.lib()\nexcept ImportError as e:\n    print('raised', e)\n"
            "else:\n    print('loaded')\n") % root
    env = dict(os.environ, CCC_LIB="/nonexistent/libccc.so")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert r.stdout.startswith("raised") and "no CPU fallback" in r.stdout, r.stdout + r.stderr


def test_product_package_does_not_import_the_oracle():
    """The product (paper_1705_08213_b200/) never imports oracle/ or baselines/ (DESIGN.md §3)."""
    import os
    import re
    pkg = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1705_08213_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+(oracle|baselines)\b", txt, re.M), f
                assert "ccc_oracle" not in txt and "liboracle" not in txt, f


def test_binding_rejects_bad_buffers_before_the_abi():
    """every wrapper checks device, dtype, contiguity and shape of its inputs and
    of caller-supplied outputs before a pointer reaches the C ABI (no CUDA needed: the
    checks raise first)."""
    import torch

    from paper_1705_08213_b200 import ccc
    cpu = torch.zeros((4, ccc.ccc_packed_stride(100)), dtype=torch.uint8)
    with pytest.raises(ValueError, match="CUDA"):
        ccc.ccc_expand(cpu, 100)
    with pytest.raises(ValueError, match="CUDA"):
        ccc.ccc_2way_popcount(cpu, 100)
    with pytest.raises(ValueError, match="CUDA"):
        ccc.ccc_3way_sparse_prepare(cpu, 100)
    with pytest.raises(ValueError, match="shape"):
        ccc._req(torch.zeros((4, 7), dtype=torch.uint8), torch.uint8, (None, ccc.ccc_packed_stride(100)),  # noqa: SLF001
                 "packed", cuda=False)
    with pytest.raises(ValueError, match="rows"):
        ccc._check_outs(10, 4, ccc.OUT_TALLY, torch.zeros((9, 4), dtype=torch.int32), None, None,  # noqa: SLF001
                        cuda=False)
    with pytest.raises(ValueError, match="float64"):
        ccc._check_outs(10, 4, ccc.OUT_CCC_F64, None, torch.zeros((10, 4), dtype=torch.float32), None,  # noqa: SLF001
                        cuda=False)
    with pytest.raises(ValueError, match="no buffer"):
        ccc._check_outs(10, 8, ccc.OUT_TALLY, None, None, None, cuda=False)   # noqa: SLF001
    with pytest.raises(ValueError, match="CUDA"):
        ccc._check_outs(1, 4, 0, None, None, torch.zeros(2, dtype=torch.int64), cuda=True)   # noqa: SLF001
    codes = torch.zeros((3, 100), dtype=torch.uint8)
    with pytest.raises(ValueError, match="tallies"):
        ccc.ccc_2way_host(codes, out_flags=ccc.OUT_TALLY, tallies_h=torch.zeros((2, 4), dtype=torch.int32),
                          dev_ws=torch.zeros(1, dtype=torch.uint8))

"""ctypes binding of libccc (include/ccc.h): the same names as the C ABI, argument
marshalling only.  Every step of the hot path runs in the CUDA kernels of libccc.so;
there is no CPU fallback -- if the library is missing or the device is not sm_100a,
calls raise.

Tensors are torch tensors used purely as device memory; launches go on torch's
current CUDA stream unless `stream` is given.
"""
from __future__ import annotations

import ctypes
import os
import re

import torch

from . import build as _build

OK, ERR_INVALID_ARGUMENT, ERR_UNSUPPORTED, ERR_CUDA, ERR_WORKSPACE = 0, 1, 2, 3, 4
OUT_TALLY, OUT_CCC_F64, OUT_CCC_F32, OUT_CHECKSUM = 1, 2, 4, 8
GAMMA = 2.0 / 3.0
HEADER = os.path.join(_build.ROOT, "include", "ccc.h")


class CCCError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class CccBlock(ctypes.Structure):
    """struct ccc_block of include/ccc.h."""
    _fields_ = [("N", ctypes.c_void_p), ("s", ctypes.c_void_p), ("w", ctypes.c_void_p),
                ("rows", ctypes.c_int64), ("row0", ctypes.c_int64)]


class CccCompact(ctypes.Structure):
    """struct ccc_compact of include/ccc.h."""
    _fields_ = [("threshold", ctypes.c_double), ("capacity", ctypes.c_int64),
                ("keys_d", ctypes.c_void_p), ("count_d", ctypes.c_void_p)]


class Compact:
    """Threshold-compacted output buffers (ccc_compact): records whose
    largest CCC cell exceeds `threshold` land in keys / tallies / ccc[:count] in arbitrary
    order.  Pass as `compact=` to ccc_2way / ccc_2way_block / ccc_3way_stage /
    ccc_3way_unit / ccc_3way; `count` accumulates across calls until reset()."""

    def __init__(self, threshold: float, capacity: int, cells: int,
                 out_flags: int = OUT_TALLY | OUT_CCC_F64, device="cuda"):
        self.threshold, self.capacity, self.cells = float(threshold), int(capacity), cells
        self.keys = torch.empty(self.capacity, dtype=torch.int64, device=device)
        self.count = torch.zeros(1, dtype=torch.int64, device=device)
        self.tallies = (torch.empty((self.capacity, cells), dtype=torch.int32, device=device)
                        if out_flags & OUT_TALLY else None)
        self.ccc = None
        if out_flags & OUT_CCC_F64:
            self.ccc = torch.empty((self.capacity, cells), dtype=torch.float64, device=device)
        elif out_flags & OUT_CCC_F32:
            self.ccc = torch.empty((self.capacity, cells), dtype=torch.float32, device=device)
        self._c = CccCompact(self.threshold, self.capacity, self.keys.data_ptr(),
                             self.count.data_ptr())

    def reset(self):
        self.count.zero_()

    def kept(self) -> int:
        return int(self.count.item())

    def result(self):
        """(count, keys, tallies, ccc) of the stored records (synchronises)."""
        n = self.kept()
        m = min(n, self.capacity)
        sl = lambda t: None if t is None else t[:m]
        return n, self.keys[:m], sl(self.tallies), sl(self.ccc)




def decode_keys(keys: torch.Tensor, num_way: int) -> torch.Tensor:
    """Compacted keys -> global indices [n][num_way]."""
    k = keys.to(torch.int64)
    if num_way == 2:
        return torch.stack([k >> 20, k & 0xFFFFF], 1)
    return torch.stack([k >> 40, (k >> 20) & 0xFFFFF, k & 0xFFFFF], 1)


_lib = None
_vp, _i64, _u32, _dbl, _int, _sz = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32,
                                    ctypes.c_double, ctypes.c_int, ctypes.c_size_t)
_SIGS = {
    "ccc_version": (_int, []),
    "ccc_status_string": (ctypes.c_char_p, [_int]),
    "ccc_last_error": (ctypes.c_char_p, []),
    "ccc_last_launch_count": (_i64, []),
    "ccc_num_unique": (_i64, [_int, _i64]),
    "ccc_pair_index": (_i64, [_i64, _i64, _i64]),
    "ccc_triple_index": (_i64, [_i64, _i64, _i64, _i64]),
    "ccc_packed_stride": (_i64, [_i64]),
    "ccc_k_pad": (_i64, [_i64]),
    "ccc_stage_range": (_int, [_i64, _i64, _i64, _vp]),
    "ccc_workspace_bytes": (_sz, [_int, _i64, _i64]),
    "ccc_pack": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "ccc_expand": (_int, [_vp, _i64, _i64, _dbl, _vp, _vp, _vp, _vp]),
    "ccc_expand_codes": (_int, [_vp, _i64, _i64, _dbl, _vp, _vp, _vp, _vp]),
    "ccc_2way": (_int, [_vp, _i64, _i64, _dbl, _u32, _vp, _vp, _vp, _vp, _sz, _vp, _vp]),
    "ccc_2way_codes": (_int, [_vp, _i64, _i64, _dbl, _u32, _vp, _vp, _vp, _vp, _sz, _vp, _vp]),
    "ccc_2way_popcount": (_int, [_vp, _i64, _i64, _dbl, _u32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "ccc_2way_fs_tiles": (_i64, [_i64]),
    "ccc_2way_fs_slot_bytes": (_sz, [_int, _i64, _i64]),
    "ccc_2way_fs_export": (_int, [_vp, _vp, _i64, _i64, _vp, _int, _int, _i64, _i64, _vp]),
    "ccc_2way_fs_finish": (_int, [_vp, _vp, _i64, _i64, _dbl, _int, _int, _i64, _i64, _u32, _vp, _vp,
                                  _vp, _vp]),
    "ccc_2way_fs_block_tiles": (_i64, [_i64, _i64, _i64, _i64, _int]),
    "ccc_2way_fs_block_export": (_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _int, _i64, _vp, _int,
                                        _int, _i64, _i64, _vp]),
    "ccc_2way_fs_block_finish": (_int, [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _i64, _i64, _int, _i64,
                                        _dbl, _int, _int, _i64, _i64, _u32, _vp, _vp, _vp, _vp]),
    "ccc_ipc_malloc": (_int, [_sz, _vp]),
    "ccc_ipc_free": (_int, [_vp]),
    "ccc_ipc_get_handle": (_int, [_vp, _vp]),
    "ccc_ipc_open": (_int, [_vp, _vp]),
    "ccc_ipc_close": (_int, [_vp]),
    "ccc_2way_block": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _i64, _i64,
                              _int, _i64, _dbl, _u32, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "ccc_3way_prepare": (_int, [_vp, _i64, _i64, _dbl, _vp, _sz, _vp]),
    "ccc_3way_stage": (_int, [_i64, _i64, _dbl, _i64, _i64, _u32, _vp, _vp, _vp, _vp, _sz, _vp,
                              _vp]),
    "ccc_3way": (_int, [_vp, _i64, _i64, _dbl, _u32, _i64, _i64, _vp, _vp, _vp, _vp, _sz, _vp,
                        _vp]),
    "ccc_3way_unit_records": (_i64, [_vp, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _i64]),
    "ccc_3way_unit": (_int, [_vp, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _i64, _int, _vp, _i64,
                             _i64, _dbl, _u32, _vp, _vp, _vp, _vp, _vp]),
    "ccc_sparse_rows": (_i64, [_i64]),
    "ccc_sparse_workspace_bytes": (_sz, [_i64, _i64]),
    "ccc_expand_sparse": (_int, [_vp, _i64, _i64, _dbl, _vp, _vp, _vp, _vp, _vp]),
    "ccc_2way_sparse_block": (_int, [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _i64, _int,
                                     _i64, _u32, _vp, _vp, _vp, _vp, _vp]),
    "ccc_2way_sparse": (_int, [_vp, _i64, _i64, _dbl, _u32, _vp, _vp, _vp, _vp, _sz, _vp, _vp]),
    "ccc_sparse3_workspace_bytes": (_sz, [_i64, _i64]),
    "ccc_3way_sparse_scratch_bytes": (_sz, [_i64, _i64, _i64]),
    "ccc_3way_sparse_prepare": (_int, [_vp, _i64, _i64, _dbl, _vp, _sz, _vp]),
    "ccc_3way_sparse_stage": (_int, [_i64, _i64, _dbl, _i64, _i64, _u32, _vp, _vp, _vp, _vp, _sz, _vp, _sz,
                                     _vp]),
    "ccc_3way_paper_workspace_bytes": (_sz, [_i64, _i64]),
    "ccc_3way_paper_scratch_bytes": (_sz, [_i64, _i64, _i64]),
    "ccc_3way_paper_prepare": (_int, [_vp, _i64, _i64, _dbl, _vp, _sz, _vp]),
    "ccc_3way_paper_stage": (_int, [_i64, _i64, _dbl, _i64, _i64, _u32, _vp, _vp, _vp, _vp, _sz, _vp, _sz,
                                    _vp]),
    "ccc_3way_host_workspace_bytes": (_sz, [_i64, _i64, _i64, _u32]),
    "ccc_3way_host": (_int, [_vp, _i64, _i64, _dbl, _u32, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "ccc_e2e_workspace_bytes": (_sz, [_i64, _i64, _u32]),
    "ccc_2way_host": (_int, [_vp, _i64, _i64, _dbl, _u32, _vp, _vp, _vp, _vp, _sz, _vp]),
}


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ccc_[a-z0-9_]+)\s*\(", txt)))


def lib_path() -> str:
    return _build.LIB


def lib():
    """Load libccc.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        path = os.environ.get("CCC_LIB", _build.LIB)   # alternate in-tree build variants
        if not os.path.exists(path):
            raise ImportError(f"libccc.so not built at {path}: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int):
    if status != OK:
        msg = lib().ccc_last_error().decode()
        name = lib().ccc_status_string(status).decode()
        if status == ERR_INVALID_ARGUMENT:
            raise ValueError(f"{name}: {msg}")
        raise CCCError(status, f"{name}: {msg}")


def _p(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, torch.cuda.Stream):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(stream)


def _req(t, dtype, shape, name, cuda=True, optional=True):
    """Validate a tensor crossing the ABI: device (CUDA or host), dtype, contiguity and the
    exact shape the C call will address (None in `shape` = any extent).  The C side only
    sees a raw pointer, so this is the one place a wrong buffer can be caught before a
    kernel or a D2H copy runs past its end."""
    if t is None:
        if optional:
            return
        raise ValueError(f"{name} is required")
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a torch tensor")
    if cuda and not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not cuda and t.is_cuda:
        raise ValueError(f"{name} must be a host (CPU) tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None:
        if t.dim() != len(shape) or any(e is not None and t.shape[d] != e for d, e in enumerate(shape)):
            raise ValueError(f"{name} must have shape {tuple('*' if e is None else e for e in shape)}, "
                             f"got {tuple(t.shape)}")


def _dev(t, dtype, name, shape=None):
    _req(t, dtype, shape, name, cuda=True)


def _bytes(t, need, name, cuda=True):
    """A uint8 scratch/workspace buffer of at least `need` bytes."""
    _req(t, torch.uint8, None, name, cuda=cuda, optional=False)
    if t.numel() < need:
        raise ValueError(f"{name} holds {t.numel()} bytes, needs {need}")


def _check_outs(n_rec, width, out_flags, tallies, ccc, checksum, cuda=True, require=True):
    """Caller-supplied record buffers must be [>= n_rec][width] of the flag's dtype (a reused
    larger buffer is fine: the records land in its first n_rec rows)."""
    cdt = (torch.float32 if out_flags & OUT_CCC_F32 and not out_flags & OUT_CCC_F64
           else torch.float64)
    for t, dt, name in ((tallies, torch.int32, "tallies"), (ccc, cdt, "ccc")):
        _req(t, dt, (None, width), name, cuda)
        if t is not None and t.shape[0] < n_rec:
            raise ValueError(f"{name} has {t.shape[0]} rows, the call writes {n_rec}")
    _req(checksum, torch.int64, (2,), "checksum", cuda)
    if not require:        # the caller allocates what is missing
        return
    for flag, t, name in ((OUT_TALLY, tallies, "tallies"), (OUT_CCC_F64 | OUT_CCC_F32, ccc, "ccc"),
                          (OUT_CHECKSUM, checksum, "checksum")):
        if out_flags & flag and t is None and n_rec:
            raise ValueError(f"out_flags asks for {name} but no buffer was given")


def _packed(packed, n_f, name="packed"):
    _dev(packed, torch.uint8, name, (None, ccc_packed_stride(n_f)))
    return packed.shape[0]


def _expanded(N, s, w, n_f, name):
    """(N int8 [rows][K_pad], s int32 [rows], w f64 [rows][2]) of one block."""
    rows = N.shape[0] if isinstance(N, torch.Tensor) else 0
    _dev(N, torch.int8, f"N_{name}", (rows, ccc_k_pad(n_f)))
    _dev(s, torch.int32, f"s_{name}", (rows,))
    _dev(w, torch.float64, f"w_{name}", (rows, 2))
    return rows


# ----------------------------------------------------------------------- host helpers
def ccc_version() -> int:
    return lib().ccc_version()


def ccc_last_launch_count() -> int:
    return lib().ccc_last_launch_count()


def ccc_num_unique(num_way: int, n_v: int) -> int:
    return lib().ccc_num_unique(num_way, n_v)


def ccc_pair_index(n_v: int, i: int, j: int) -> int:
    return lib().ccc_pair_index(n_v, i, j)


def ccc_triple_index(n_v: int, i: int, j: int, k: int) -> int:
    return lib().ccc_triple_index(n_v, i, j, k)


def ccc_packed_stride(n_f: int) -> int:
    return lib().ccc_packed_stride(n_f)


def ccc_k_pad(n_f: int) -> int:
    return lib().ccc_k_pad(n_f)


def ccc_stage_range(n_v: int, n_stages: int, stage: int):
    out = (ctypes.c_int64 * 4)()
    _check(lib().ccc_stage_range(n_v, n_stages, stage, ctypes.cast(out, ctypes.c_void_p)))
    return tuple(int(x) for x in out)


def ccc_workspace_bytes(num_way: int, n_v: int, n_f: int) -> int:
    return lib().ccc_workspace_bytes(num_way, n_v, n_f)


def ccc_e2e_workspace_bytes(n_v: int, n_f: int, out_flags: int) -> int:
    return lib().ccc_e2e_workspace_bytes(n_v, n_f, out_flags)


def workspace(num_way: int, n_v: int, n_f: int, device=None) -> torch.Tensor:
    n = max(ccc_workspace_bytes(num_way, n_v, n_f), 256)
    return torch.empty(n, dtype=torch.uint8, device=device or "cuda")


# ----------------------------------------------------------------------- device path
def ccc_pack(codes: torch.Tensor, packed: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    _dev(codes, torch.uint8, "codes", (None, None))
    n_v, n_f = codes.shape
    if packed is None:
        packed = torch.empty((n_v, ccc_packed_stride(n_f)), dtype=torch.uint8, device=codes.device)
    _dev(packed, torch.uint8, "packed", (n_v, ccc_packed_stride(n_f)))
    _check(lib().ccc_pack(_p(codes), n_v, n_f, _p(packed), _stream(stream)))
    return packed


def ccc_expand(packed: torch.Tensor, n_f: int, gamma: float = GAMMA, N=None, s=None, w=None,
               stream=None):
    n_v = _packed(packed, n_f)
    dev = packed.device
    if N is None:
        N = torch.empty((n_v, ccc_k_pad(n_f)), dtype=torch.int8, device=dev)
    if s is None:
        s = torch.empty(n_v, dtype=torch.int32, device=dev)
    if w is None:
        w = torch.empty((n_v, 2), dtype=torch.float64, device=dev)
    _dev(N, torch.int8, "N", (n_v, ccc_k_pad(n_f)))
    _dev(s, torch.int32, "s", (n_v,))
    _dev(w, torch.float64, "w", (n_v, 2))
    _check(lib().ccc_expand(_p(packed), n_v, n_f, gamma, _p(N), _p(s), _p(w), _stream(stream)))
    return N, s, w


def ccc_expand_codes(codes: torch.Tensor, gamma: float = GAMMA, N=None, s=None, w=None, stream=None):
    """Unpacked codes [n_v][n_f] -> (N, s, w) in one pass (= ccc_expand(ccc_pack(codes)))."""
    _dev(codes, torch.uint8, "codes", (None, None))
    n_v, n_f = codes.shape
    dev = codes.device
    if N is None:
        N = torch.empty((n_v, ccc_k_pad(n_f)), dtype=torch.int8, device=dev)
    if s is None:
        s = torch.empty(n_v, dtype=torch.int32, device=dev)
    if w is None:
        w = torch.empty((n_v, 2), dtype=torch.float64, device=dev)
    _dev(N, torch.int8, "N", (n_v, ccc_k_pad(n_f)))
    _dev(s, torch.int32, "s", (n_v,))
    _dev(w, torch.float64, "w", (n_v, 2))
    _check(lib().ccc_expand_codes(_p(codes), n_v, n_f, gamma, _p(N), _p(s), _p(w), _stream(stream)))
    return N, s, w


def _outputs(n_rec: int, width: int, out_flags: int, device, tallies=None, ccc=None,
             checksum=None):
    _check_outs(n_rec, width, out_flags, tallies, ccc, checksum, require=False)
    if out_flags & OUT_TALLY and tallies is None:
        tallies = torch.empty((n_rec, width), dtype=torch.int32, device=device)
    if out_flags & OUT_CCC_F64 and ccc is None:
        ccc = torch.empty((n_rec, width), dtype=torch.float64, device=device)
    if out_flags & OUT_CCC_F32 and ccc is None:
        ccc = torch.empty((n_rec, width), dtype=torch.float32, device=device)
    if out_flags & OUT_CHECKSUM and checksum is None:
        checksum = torch.zeros(2, dtype=torch.int64, device=device)
    return tallies, ccc, checksum


def _outs(n_rec, width, out_flags, device, tallies, ccc, checksum, compact):
    """Dense record buffers, or the compacted ones of `compact` (+ the checksum)."""
    if compact is None:
        return (None,) + _outputs(n_rec, width, out_flags, device, tallies, ccc, checksum)
    _, _, checksum = _outputs(0, width, out_flags & OUT_CHECKSUM, device, None, None, checksum)
    return ctypes.byref(compact._c), compact.tallies, compact.ccc, checksum


def ccc_2way(packed: torch.Tensor, n_f: int, gamma: float = GAMMA,
             out_flags: int = OUT_TALLY | OUT_CCC_F64, tallies=None, ccc=None, checksum=None,
             ws=None, stream=None, compact: Compact | None = None):
    """Tallies (uint32 bit patterns in an int32 tensor) [C(n_v,2)][4], CCC, checksum[2]
    (with `compact`: the compacted buffers of that object instead)."""
    n_v = _packed(packed, n_f)
    cp, tallies, ccc, checksum = _outs(ccc_num_unique(2, n_v), 4, out_flags, packed.device,
                                       tallies, ccc, checksum, compact)
    if ws is None:
        ws = workspace(2, n_v, n_f, packed.device)
    _bytes(ws, ccc_workspace_bytes(2, n_v, n_f), "ws")
    _check(lib().ccc_2way(_p(packed), n_v, n_f, gamma, out_flags, _p(tallies), _p(ccc),
                          _p(checksum), _p(ws), ws.numel(), cp, _stream(stream)))
    return tallies, ccc, checksum


def ccc_2way_codes(codes: torch.Tensor, gamma: float = GAMMA, out_flags: int = OUT_TALLY | OUT_CCC_F64,
                   tallies=None, ccc=None, checksum=None, ws=None, stream=None, compact: Compact | None = None):
    """All 2-way records from unpacked device codes [n_v][n_f]; the expand overlaps the
    tally GEMM (see include/ccc.h).  Returns (tallies, ccc, checksum) like ccc_2way."""
    _dev(codes, torch.uint8, "codes", (None, None))
    n_v, n_f = codes.shape
    cp, tallies, ccc, checksum = _outs(ccc_num_unique(2, n_v), 4, out_flags, codes.device,
                                       tallies, ccc, checksum, compact)
    if ws is None:
        ws = workspace(2, n_v, n_f, codes.device)
    _bytes(ws, ccc_workspace_bytes(2, n_v, n_f), "ws")
    _check(lib().ccc_2way_codes(_p(codes), n_v, n_f, gamma, out_flags, _p(tallies), _p(ccc),
                                _p(checksum), _p(ws), ws.numel(), cp, _stream(stream)))
    return tallies, ccc, checksum


def ccc_2way_popcount(packed: torch.Tensor, n_f: int, gamma: float = GAMMA,
                      out_flags: int = OUT_TALLY | OUT_CCC_F64, tallies=None, ccc=None, checksum=None,
                      ws=None, stream=None):
    """The paper's popcount tally (mGEMM2 idea) on CUDA cores: a comparison
    baseline with the outputs of ccc_2way."""
    n_v = _packed(packed, n_f)
    dev = packed.device
    T, C, ck = _outputs(ccc_num_unique(2, n_v), 4, out_flags, dev, tallies, ccc, checksum)
    if ws is None:
        ws = workspace(2, n_v, n_f, dev)
    _bytes(ws, ccc_workspace_bytes(2, n_v, n_f), "ws")
    _check(lib().ccc_2way_popcount(_p(packed), n_v, n_f, gamma, out_flags, _p(T), _p(C),
                                   _p(ck), _p(ws), ws.numel(), _stream(stream)))
    return T, C, ck


# ------------------------------------------------------------- f3: field-axis split
def ccc_2way_fs_tiles(n_v: int) -> int:
    return lib().ccc_2way_fs_tiles(n_v)


def ccc_2way_fs_slot_bytes(world: int, t_lo: int, t_hi: int) -> int:
    return lib().ccc_2way_fs_slot_bytes(world, t_lo, t_hi)


def ccc_2way_fs_export(N, s, n_f_slice: int, slot_ptrs: torch.Tensor, rank: int, world: int,
                       t_lo: int, t_hi: int, stream=None):
    """GEMM of this field slice; partial tiles go to the owners' slots (slot_ptrs: int64
    device tensor of `world` device addresses)."""
    n_v = N.shape[0] if isinstance(N, torch.Tensor) else 0
    _dev(N, torch.int8, "N", (n_v, ccc_k_pad(n_f_slice)))
    _dev(s, torch.int32, "s", (n_v,))
    _dev(slot_ptrs, torch.int64, "slot_ptrs", (world,))
    if not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    _check(lib().ccc_2way_fs_export(_p(N), _p(s), N.shape[0], n_f_slice, _p(slot_ptrs), rank, world,
                                    t_lo, t_hi, _stream(stream)))


def ccc_2way_fs_finish(slots: torch.Tensor, s, n_f: int, rank: int, world: int, t_lo: int, t_hi: int,
                       out_flags: int, tallies=None, ccc=None, checksum=None, gamma: float = GAMMA,
                       stream=None):
    """Reduce this owner's partial tiles and write their records (ccc_2way layout)."""
    _dev(s, torch.int32, "s", (None,))
    n_v = s.shape[0]
    _req(slots, torch.int32, None, "slots", optional=False)
    if slots.numel() * 4 < ccc_2way_fs_slot_bytes(world, t_lo, t_hi):
        raise ValueError("slots smaller than ccc_2way_fs_slot_bytes(world, t_lo, t_hi)")
    T, C, ck = _outputs(ccc_num_unique(2, n_v), 4, out_flags, s.device, tallies, ccc, checksum)
    _check(lib().ccc_2way_fs_finish(_p(slots), _p(s), n_v, n_f, gamma, rank, world, t_lo, t_hi,
                                    out_flags, _p(T), _p(C), _p(ck), _stream(stream)))
    return T, C, ck


def ccc_2way_fs_block_tiles(n_a: int, a_lo: int, a_hi: int, n_b: int, diag: bool) -> int:
    n = lib().ccc_2way_fs_block_tiles(n_a, a_lo, a_hi, n_b, int(bool(diag)))
    if n < 0:
        raise ValueError("invalid block geometry")
    return n


def block_records(n_a: int, a_lo: int, a_hi: int, n_b: int, diag: bool) -> int:
    """Records of ccc_2way_block's layout for this geometry (host arithmetic on indices)."""
    return sum(n_a - 1 - i for i in range(a_lo, a_hi)) if diag else (a_hi - a_lo) * n_b


def ccc_2way_fs_block_export(N_a, s_a, a_lo: int, a_hi: int, N_b, s_b, diag: bool, n_f_slice: int,
                             slot_ptrs: torch.Tensor, rank: int, world: int, t_lo: int, t_hi: int,
                             stream=None):
    """Export GEMM of one block of the vector decomposition on this field slice (2-D grid):
    partial tiles go to the owners' slots (slot_ptrs: int64 device tensor of `world`
    device addresses)."""
    n_a = N_a.shape[0] if isinstance(N_a, torch.Tensor) else 0
    n_b = N_b.shape[0] if isinstance(N_b, torch.Tensor) else 0
    _dev(N_a, torch.int8, "N_a", (n_a, ccc_k_pad(n_f_slice)))
    _dev(N_b, torch.int8, "N_b", (n_b, ccc_k_pad(n_f_slice)))
    _dev(s_a, torch.int32, "s_a", (n_a,))
    _dev(s_b, torch.int32, "s_b", (n_b,))
    _dev(slot_ptrs, torch.int64, "slot_ptrs", (world,))
    if not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    if diag and (N_a.data_ptr() != N_b.data_ptr() or s_a.data_ptr() != s_b.data_ptr()):
        raise ValueError("a diag block passes the same N / s for A and B")
    _check(lib().ccc_2way_fs_block_export(_p(N_a), _p(s_a), n_a, a_lo, a_hi, _p(N_b), _p(s_b), n_b,
                                          int(bool(diag)), n_f_slice, _p(slot_ptrs), rank, world, t_lo,
                                          t_hi, _stream(stream)))


def ccc_2way_fs_block_finish(slots, s_a, a_row0: int, a_lo: int, a_hi: int, s_b, b_row0: int, diag: bool,
                             n_f: int, rank: int, world: int, t_lo: int, t_hi: int, out_flags: int,
                             tallies=None, ccc=None, checksum=None, gamma: float = GAMMA, stream=None,
                             slot_ptr: int | None = None):
    """Reduce this owner's partial tiles of one block and write their records (the
    ccc_2way_block layout of the geometry).  s_a / s_b: the blocks' full allele sums.
    slots: this owner's int32 slot tensor, or slot_ptr (an IPC buffer's device address)."""
    _dev(s_a, torch.int32, "s_a", (None,))
    _dev(s_b, torch.int32, "s_b", (None,))
    n_a, n_b = s_a.shape[0], s_b.shape[0]
    if not 0 <= a_lo <= a_hi <= n_a:
        raise ValueError("row range [a_lo, a_hi) must lie inside block a")
    if slot_ptr is None:
        _req(slots, torch.int32, None, "slots", optional=False)
        if slots.numel() * 4 < ccc_2way_fs_slot_bytes(world, t_lo, t_hi):
            raise ValueError("slots smaller than ccc_2way_fs_slot_bytes(world, t_lo, t_hi)")
        sp = _p(slots)
    else:
        sp = ctypes.c_void_p(slot_ptr)
    n_rec = block_records(n_a, a_lo, a_hi, n_b, diag)
    T, C, ck = _outputs(n_rec, 4, out_flags, s_a.device, tallies, ccc, checksum)
    _check(lib().ccc_2way_fs_block_finish(sp, _p(s_a), n_a, a_row0, a_lo, a_hi, _p(s_b), n_b, b_row0,
                                          int(bool(diag)), n_f, gamma, rank, world, t_lo, t_hi, out_flags,
                                          _p(T), _p(C), _p(ck), _stream(stream)))
    return T, C, ck


class IpcBuffer:
    """A peer-shareable device buffer (ccc_ipc_malloc) with its CUDA IPC handle."""

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        _check(lib().ccc_ipc_malloc(nbytes, ctypes.byref(p)))
        self.ptr = p.value
        self.nbytes = nbytes

    def handle(self) -> bytes:
        h = ctypes.create_string_buffer(64)
        _check(lib().ccc_ipc_get_handle(self.ptr, h))
        return h.raw

    def free(self):
        if self.ptr:
            _check(lib().ccc_ipc_free(self.ptr))
            self.ptr = None


def ipc_open(handle: bytes) -> int:
    p = ctypes.c_void_p()
    _check(lib().ccc_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(p)))
    return p.value


def ipc_close(ptr: int):
    _check(lib().ccc_ipc_close(ptr))


def ccc_2way_block(N_a, s_a, w_a, a_row0, a_lo, a_hi, N_b, s_b, w_b, b_row0, diag: bool, n_f,
                   out_flags, tallies=None, ccc=None, checksum=None, g=None, ldg=0,
                   stream=None, gamma=GAMMA, compact: Compact | None = None):
    """gamma: the value the w arrays were expanded with (selects the kernel's arithmetic).
    Output buffers are the caller's (dense layout) or those of `compact`."""
    cp = None
    n_a = _expanded(N_a, s_a, w_a, n_f, "a")
    n_b = _expanded(N_b, s_b, w_b, n_f, "b")
    if not 0 <= a_lo <= a_hi <= n_a:
        raise ValueError("row range [a_lo, a_hi) must lie inside block a")
    n_rec = (sum(n_a - 1 - i for i in range(a_lo, a_hi)) if diag else (a_hi - a_lo) * n_b)
    if compact is not None:
        cp, tallies, ccc = ctypes.byref(compact._c), compact.tallies, compact.ccc
        _req(checksum, torch.int64, (2,), "checksum")
    else:
        _check_outs(n_rec, 4, out_flags, tallies, ccc, checksum)
    _req(g, torch.int32, None, "g")
    _check(lib().ccc_2way_block(_p(N_a), _p(s_a), _p(w_a), n_a, a_row0, a_lo, a_hi, _p(N_b),
                                _p(s_b), _p(w_b), n_b, b_row0, int(bool(diag)), n_f, gamma, out_flags,
                                _p(tallies), _p(ccc), _p(checksum), _p(g), ldg, cp,
                                _stream(stream)))
    return tallies, ccc, checksum


def ccc_3way_prepare(packed, n_f, gamma=GAMMA, ws=None, stream=None):
    n_v = _packed(packed, n_f)
    if ws is None:
        ws = workspace(3, n_v, n_f, packed.device)
    _bytes(ws, ccc_workspace_bytes(3, n_v, n_f), "ws")
    _check(lib().ccc_3way_prepare(_p(packed), n_v, n_f, gamma, _p(ws), ws.numel(),
                                  _stream(stream)))
    return ws


def ccc_3way_stage(n_v, n_f, n_stages, stage, ws, out_flags=OUT_TALLY | OUT_CCC_F64,
                   tallies=None, ccc=None, checksum=None, stream=None, gamma=GAMMA,
                   compact: Compact | None = None):
    """gamma: the value given to ccc_3way_prepare for this workspace."""
    _, _, _, rec_count = ccc_stage_range(n_v, n_stages, stage)
    _bytes(ws, ccc_workspace_bytes(3, n_v, n_f), "ws")
    cp, tallies, ccc, checksum = _outs(rec_count, 8, out_flags, ws.device, tallies, ccc,
                                       checksum, compact)
    _check(lib().ccc_3way_stage(n_v, n_f, gamma, n_stages, stage, out_flags, _p(tallies), _p(ccc),
                                _p(checksum), _p(ws), ws.numel(), cp, _stream(stream)))
    return tallies, ccc, checksum


def ccc_3way(packed, n_f, gamma=GAMMA, out_flags=OUT_TALLY | OUT_CCC_F64, n_stages=1, stage=0,
             tallies=None, ccc=None, checksum=None, ws=None, stream=None,
             compact: Compact | None = None):
    n_v = _packed(packed, n_f)
    _, _, _, rec_count = ccc_stage_range(n_v, n_stages, stage)
    cp, tallies, ccc, checksum = _outs(rec_count, 8, out_flags, packed.device, tallies, ccc,
                                       checksum, compact)
    if ws is None:
        ws = workspace(3, n_v, n_f, packed.device)
    _bytes(ws, ccc_workspace_bytes(3, n_v, n_f), "ws")
    _check(lib().ccc_3way(_p(packed), n_v, n_f, gamma, out_flags, n_stages, stage, _p(tallies),
                          _p(ccc), _p(checksum), _p(ws), ws.numel(), cp, _stream(stream)))
    return tallies, ccc, checksum


ORDERS = {("p", "m", "n"): 0, ("p", "n", "m"): 1, ("m", "p", "n"): 2, ("m", "n", "p"): 3,
          ("n", "p", "m"): 4, ("n", "m", "p"): 5}


def block(N, s, w, row0: int) -> CccBlock:
    """ccc_block descriptor of an expanded block (keep the tensors alive)."""
    rows = N.shape[0] if isinstance(N, torch.Tensor) else 0
    _dev(N, torch.int8, "N", (rows, None))
    _dev(s, torch.int32, "s", (rows,))
    _dev(w, torch.float64, "w", (rows, 2))
    return CccBlock(N.data_ptr(), s.data_ptr(), w.data_ptr(), N.shape[0], row0)


def ccc_3way_unit_records(bp, p_lo, p_hi, bm, m_lo, m_hi, bn, n_lo, n_hi) -> int:
    return lib().ccc_3way_unit_records(ctypes.byref(bp), p_lo, p_hi, ctypes.byref(bm), m_lo, m_hi,
                                       ctypes.byref(bn), n_lo, n_hi)


def ccc_3way_unit(bp, p_lo, p_hi, bm, m_lo, m_hi, bn, n_lo, n_hi, order, G, n_f,
                  out_flags=OUT_TALLY | OUT_CCC_F64, tallies=None, ccc=None, checksum=None,
                  stream=None, gamma=GAMMA, compact: Compact | None = None):
    """One tetrahedral 3-way unit; `order` is a role tuple like ("m", "p", "n") or 0..5;
    gamma: the value the blocks' w were expanded with."""
    if not isinstance(order, int):
        order = ORDERS[tuple(order)]
    n_rec = ccc_3way_unit_records(bp, p_lo, p_hi, bm, m_lo, m_hi, bn, n_lo, n_hi)
    if n_rec < 0:
        raise ValueError("invalid unit ranges")
    _dev(G, torch.int32, "G", (None, None))
    if G.shape[0] != G.shape[1]:
        raise ValueError("G must be the square [n_v][n_v] pairwise G")
    cp, tallies, ccc, checksum = _outs(n_rec, 8, out_flags, G.device, tallies, ccc, checksum,
                                       compact)
    _check(lib().ccc_3way_unit(ctypes.byref(bp), p_lo, p_hi, ctypes.byref(bm), m_lo, m_hi,
                               ctypes.byref(bn), n_lo, n_hi, order, _p(G), G.shape[-1], n_f,
                               gamma, out_flags, _p(tallies), _p(ccc), _p(checksum), cp,
                               _stream(stream)))
    return tallies, ccc, checksum


def ccc_2way_host(codes_h: torch.Tensor, gamma: float = GAMMA,
                  out_flags: int = OUT_TALLY | OUT_CCC_F64, tallies_h=None, ccc_h=None,
                  checksum_h=None, dev_ws=None, stream=None):
    """End-to-end 2-way with host (pinned) buffers in and out."""
    if codes_h.is_cuda or codes_h.dtype != torch.uint8 or not codes_h.is_contiguous():
        raise ValueError("codes_h must be a contiguous host uint8 tensor")
    n_v, n_f = codes_h.shape
    m = ccc_num_unique(2, n_v)
    pin = codes_h.is_pinned()
    if out_flags & OUT_TALLY and tallies_h is None:
        tallies_h = torch.empty((m, 4), dtype=torch.int32, pin_memory=pin)
    if out_flags & OUT_CCC_F64 and ccc_h is None:
        ccc_h = torch.empty((m, 4), dtype=torch.float64, pin_memory=pin)
    if out_flags & OUT_CCC_F32 and ccc_h is None:
        ccc_h = torch.empty((m, 4), dtype=torch.float32, pin_memory=pin)
    if out_flags & OUT_CHECKSUM and checksum_h is None:
        checksum_h = torch.zeros(2, dtype=torch.int64, pin_memory=pin)
    if dev_ws is None:
        dev_ws = torch.empty(ccc_e2e_workspace_bytes(n_v, n_f, out_flags), dtype=torch.uint8,
                             device="cuda")
    _check_outs(m, 4, out_flags, tallies_h, ccc_h, checksum_h, cuda=False)
    _bytes(dev_ws, ccc_e2e_workspace_bytes(n_v, n_f, out_flags), "dev_ws")
    _check(lib().ccc_2way_host(_p(codes_h), n_v, n_f, gamma, out_flags, _p(tallies_h), _p(ccc_h),
                               _p(checksum_h), _p(dev_ws), dev_ws.numel(), _stream(stream)))
    return tallies_h, ccc_h, checksum_h


# ----------------------------------------------------------------------- conveniences
def checksum_int(ck: torch.Tensor) -> int:
    """checksum tensor [2] (lo, hi as int64 bit patterns) -> Python int mod 2^128."""
    lo, hi = (int(x) & ((1 << 64) - 1) for x in ck.cpu().tolist())
    return (hi << 64) | lo


# ----------------------------------------------------------------------- sparse mode (f1)
def ccc_sparse_rows(n_v: int) -> int:
    return lib().ccc_sparse_rows(n_v)


def ccc_expand_sparse(packed: torch.Tensor, n_f: int, gamma: float = GAMMA, out=None,
                      stream=None):
    """packed -> (X int8 [ccc_sparse_rows(n_v)][K_pad], s, c int32 [n_v], w f64 [n_v][2])
    (written into `out` = (X, s, c, w) if given)."""
    n_v = _packed(packed, n_f)
    dev = packed.device
    if out is None:
        X = torch.empty((ccc_sparse_rows(n_v), ccc_k_pad(n_f)), dtype=torch.int8, device=dev)
        s = torch.empty(n_v, dtype=torch.int32, device=dev)
        c = torch.empty(n_v, dtype=torch.int32, device=dev)
        w = torch.empty((n_v, 2), dtype=torch.float64, device=dev)
    else:
        X, s, c, w = out
    _dev(X, torch.int8, "X", (ccc_sparse_rows(n_v), ccc_k_pad(n_f)))
    _dev(s, torch.int32, "s", (n_v,))
    _dev(c, torch.int32, "c", (n_v,))
    _dev(w, torch.float64, "w", (n_v, 2))
    _check(lib().ccc_expand_sparse(_p(packed), n_v, n_f, gamma, _p(X), _p(s), _p(c), _p(w),
                                   _stream(stream)))
    return X, s, c, w


def ccc_2way_sparse_block(X_a, w_a, n_a, a_row0, a_lo, a_hi, X_b, w_b, n_b, b_row0, diag, n_f,
                          out_flags, tallies=None, ccc=None, checksum=None, stream=None,
                          compact: Compact | None = None):
    cp = None
    for X, w, n, nm in ((X_a, w_a, n_a, "a"), (X_b, w_b, n_b, "b")):
        _dev(X, torch.int8, f"X_{nm}", (ccc_sparse_rows(n), ccc_k_pad(n_f)))
        _dev(w, torch.float64, f"w_{nm}", (n, 2))
    if not 0 <= a_lo <= a_hi <= n_a:
        raise ValueError("row range [a_lo, a_hi) must lie inside block a")
    n_rec = (sum(n_a - 1 - i for i in range(a_lo, a_hi)) if diag else (a_hi - a_lo) * n_b)
    if compact is not None:
        cp, tallies, ccc = ctypes.byref(compact._c), compact.tallies, compact.ccc
        _req(checksum, torch.int64, (2,), "checksum")
    else:
        _check_outs(n_rec, 4, out_flags, tallies, ccc, checksum)
    _check(lib().ccc_2way_sparse_block(_p(X_a), _p(w_a), n_a, a_row0, a_lo, a_hi, _p(X_b),
                                       _p(w_b), n_b, b_row0, int(bool(diag)), n_f, out_flags,
                                       _p(tallies), _p(ccc), _p(checksum), cp, _stream(stream)))
    return tallies, ccc, checksum


def ccc_2way_sparse(packed: torch.Tensor, n_f: int, gamma: float = GAMMA,
                    out_flags: int = OUT_TALLY | OUT_CCC_F64, tallies=None, ccc=None,
                    checksum=None, ws=None, stream=None, compact: Compact | None = None):
    """Sparse-mode 2-way (code 2 = (1,0) marks a missing entry): records as ccc_2way."""
    n_v = _packed(packed, n_f)
    cp, tallies, ccc, checksum = _outs(ccc_num_unique(2, n_v), 4, out_flags, packed.device,
                                       tallies, ccc, checksum, compact)
    if ws is None:
        ws = torch.empty(max(lib().ccc_sparse_workspace_bytes(n_v, n_f), 256), dtype=torch.uint8,
                         device=packed.device)
    _bytes(ws, lib().ccc_sparse_workspace_bytes(n_v, n_f), "ws")
    _check(lib().ccc_2way_sparse(_p(packed), n_v, n_f, gamma, out_flags, _p(tallies), _p(ccc),
                                 _p(checksum), _p(ws), ws.numel(), cp, _stream(stream)))
    return tallies, ccc, checksum


def two_way(codes: torch.Tensor, gamma: float = GAMMA, out_flags: int = OUT_TALLY | OUT_CCC_F64,
            stream=None):
    """codes uint8 [n_v][n_f] on the GPU -> (tallies, ccc, checksum) for all i<j."""
    packed = ccc_pack(codes, stream=stream)
    return ccc_2way(packed, codes.shape[1], gamma, out_flags, stream=stream)


def three_way(codes: torch.Tensor, gamma: float = GAMMA, out_flags: int = OUT_TALLY | OUT_CCC_F64,
              n_stages: int = 1, stage: int = 0, stream=None):
    packed = ccc_pack(codes, stream=stream)
    return ccc_3way(packed, codes.shape[1], gamma, out_flags, n_stages, stage, stream=stream)


# ------------------------------------------------------------- f1: sparse 3-way
def ccc_3way_sparse_prepare(packed: torch.Tensor, n_f: int, gamma: float = GAMMA, ws=None, stream=None):
    """Expand for the sparse 3-way mode: the workspace (X interleaved, s, c, w)."""
    n_v = _packed(packed, n_f)
    if ws is None:
        ws = torch.empty(max(256, lib().ccc_sparse3_workspace_bytes(n_v, n_f)), dtype=torch.uint8,
                         device=packed.device)
    _bytes(ws, lib().ccc_sparse3_workspace_bytes(n_v, n_f), "ws")
    _check(lib().ccc_3way_sparse_prepare(_p(packed), n_v, n_f, gamma, _p(ws), ws.numel(), _stream(stream)))
    return ws


def ccc_3way_sparse_stage(n_v: int, n_f: int, n_stages: int, stage: int, ws: torch.Tensor,
                          out_flags: int = OUT_TALLY | OUT_CCC_F64, tallies=None, ccc=None, checksum=None,
                          scratch=None, gamma: float = GAMMA, stream=None):
    """One stage of the sparse 3-way records (one pivot GEMM with all 8 forms)."""
    rc = ccc_stage_range(n_v, n_stages, stage)[3]
    T, C, ck = _outputs(rc, 8, out_flags, ws.device, tallies, ccc, checksum)
    nb = lib().ccc_3way_sparse_scratch_bytes(n_v, n_stages, stage)
    if scratch is None:
        scratch = torch.empty(max(16, nb), dtype=torch.uint8, device=ws.device)
    _bytes(ws, lib().ccc_sparse3_workspace_bytes(n_v, n_f), "ws")
    _bytes(scratch, nb, "scratch")
    _check(lib().ccc_3way_sparse_stage(n_v, n_f, gamma, n_stages, stage, out_flags, _p(T), _p(C), _p(ck),
                                       _p(ws), ws.numel(), _p(scratch), scratch.numel(), _stream(stream)))
    return T, C, ck


def three_way_sparse(codes: torch.Tensor, gamma: float = GAMMA, out_flags: int = OUT_TALLY | OUT_CCC_F64,
                     n_stages: int = 1):
    """Convenience: all sparse 3-way records of a device code matrix, stages concatenated;
    returns (T, C, [per-stage checksum tensors])."""
    n_v, n_f = codes.shape
    ws = ccc_3way_sparse_prepare(ccc_pack(codes), n_f, gamma)
    outs = [ccc_3way_sparse_stage(n_v, n_f, n_stages, st, ws, out_flags, gamma=gamma) for st in range(n_stages)]
    T = torch.cat([o[0] for o in outs]) if out_flags & OUT_TALLY else None
    C = torch.cat([o[1] for o in outs]) if out_flags & (OUT_CCC_F64 | OUT_CCC_F32) else None
    return T, C, [o[2] for o in outs] if out_flags & OUT_CHECKSUM else None


# ------------------------------------------------------------- f4(ii): the paper's 3-way route
def ccc_3way_paper_prepare(packed: torch.Tensor, n_f: int, gamma: float = GAMMA, ws=None, stream=None):
    n_v = _packed(packed, n_f)
    if ws is None:
        ws = torch.empty(max(256, lib().ccc_3way_paper_workspace_bytes(n_v, n_f)), dtype=torch.uint8,
                         device=packed.device)
    _bytes(ws, lib().ccc_3way_paper_workspace_bytes(n_v, n_f), "ws")
    _check(lib().ccc_3way_paper_prepare(_p(packed), n_v, n_f, gamma, _p(ws), ws.numel(), _stream(stream)))
    return ws


def ccc_3way_paper_stage(n_v: int, n_f: int, n_stages: int, stage: int, ws: torch.Tensor,
                         out_flags: int = OUT_TALLY | OUT_CCC_F64, tallies=None, ccc=None, checksum=None,
                         scratch=None, gamma: float = GAMMA, stream=None):
    rc = ccc_stage_range(n_v, n_stages, stage)[3]
    T, C, ck = _outputs(rc, 8, out_flags, ws.device, tallies, ccc, checksum)
    nb = lib().ccc_3way_paper_scratch_bytes(n_v, n_stages, stage)
    if scratch is None:
        scratch = torch.empty(max(16, nb), dtype=torch.uint8, device=ws.device)
    _bytes(ws, lib().ccc_3way_paper_workspace_bytes(n_v, n_f), "ws")
    _bytes(scratch, nb, "scratch")
    _check(lib().ccc_3way_paper_stage(n_v, n_f, gamma, n_stages, stage, out_flags, _p(T), _p(C), _p(ck),
                                      _p(ws), ws.numel(), _p(scratch), scratch.numel(), _stream(stream)))
    return T, C, ck


# ------------------------------------------------------------- f2: 3-way stage streaming to host
def ccc_3way_host(codes_h: torch.Tensor, gamma: float = GAMMA, out_flags: int = OUT_TALLY | OUT_CCC_F64,
                  n_stages: int = 1, tallies_h=None, ccc_h=None, checksum_h=None, ws=None, stream=None):
    """Host codes in, every 3-way record streamed stage by stage into host buffers (pinned
    for overlap); allocates the host outputs (pinned) when not given."""
    if codes_h.dtype != torch.uint8 or codes_h.device.type != "cpu" or not codes_h.is_contiguous():
        raise ValueError("codes_h must be a contiguous uint8 CPU tensor")
    n_v, n_f = codes_h.shape
    m = ccc_num_unique(3, n_v)
    if out_flags & OUT_TALLY and tallies_h is None:
        tallies_h = torch.empty((m, 8), dtype=torch.int32, pin_memory=True)
    if out_flags & OUT_CCC_F64 and ccc_h is None:
        ccc_h = torch.empty((m, 8), dtype=torch.float64, pin_memory=True)
    if out_flags & OUT_CCC_F32 and ccc_h is None:
        ccc_h = torch.empty((m, 8), dtype=torch.float32, pin_memory=True)
    if out_flags & OUT_CHECKSUM and checksum_h is None:
        checksum_h = torch.zeros(2, dtype=torch.int64)
    if ws is None:
        ws = torch.empty(lib().ccc_3way_host_workspace_bytes(n_v, n_f, n_stages, out_flags), dtype=torch.uint8,
                         device="cuda")
    _check_outs(m, 8, out_flags, tallies_h, ccc_h, checksum_h, cuda=False)
    _bytes(ws, lib().ccc_3way_host_workspace_bytes(n_v, n_f, n_stages, out_flags), "ws")
    _check(lib().ccc_3way_host(codes_h.data_ptr(), n_v, n_f, gamma, out_flags, n_stages,
                               tallies_h.data_ptr() if tallies_h is not None else None,
                               ccc_h.data_ptr() if ccc_h is not None else None,
                               checksum_h.data_ptr() if checksum_h is not None else None,
                               _p(ws), ws.numel(), _stream(stream)))
    return tallies_h, ccc_h, checksum_h

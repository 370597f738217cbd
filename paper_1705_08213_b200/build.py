"""Build libccc.so in-tree with nvcc for sm_100a only (no JIT, no torch extension)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libccc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
EXTRA = os.environ.get("CCC_NVCC_EXTRA", "").split()


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(
        os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "ccc.h"), __file__]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile every csrc/*.cu into one shared library.  `out`/`defines` build diagnostic
    variants (e.g. -DCCC_D3_NOXF) next to the product library; they are never loaded
    unless CCC_LIB points at them."""
    if not force and out == LIB and not defines and up_to_date():
        return LIB
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
           "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC] + EXTRA + [f"-D{d}" for d in defines] + [
           "-Xptxas", "-v" if verbose else "-O3",
           "-o", tmp] + sources()
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libccc.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    out = LIB
    if "--out" in args:
        out = os.path.abspath(args[args.index("--out") + 1])
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args or out != LIB, verbose="-v" in args, out=out, defines=defs))

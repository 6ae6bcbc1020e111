"""Build libcimcs_gpu.so in-tree for sm_100a (B200) with nvcc.

The kernels are compiled with -fmad=false so the elementwise MFZ update keeps
the reference's rounding; the contraction and Gram kernels use explicit fma.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libcimcs_gpu.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("runtime.cu",)]
DEPS = SOURCES + sorted(
    os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))
    if f.endswith((".cuh", ".hpp"))) + [os.path.join(ROOT, "include", "cimcs_gpu.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-fmad=false", "-Xcompiler", "-fPIC,-O3", "-shared", "-cudart", "static",
]
LIBS = ["-lnccl", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]


def _torch_nccl_dir():
    """torch's bundled libnccl.so.2 (newer than the system copy): linking and
    rpath-ing it first means whichever of torch / this library loads first, the
    process gets the one NCCL both can use."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        d = os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(d, "libnccl.so.2")):
            return d
    return None


_NCCL = _torch_nccl_dir()
if _NCCL:
    LIBS = ["-L" + _NCCL, "-Xlinker", "-rpath," + _NCCL, "-l:libnccl.so.2"] + LIBS[1:]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        cmd = [NVCC, *FLAGS, *os.environ.get("CIMCS_NVCC_EXTRA", "").split(), "-o", LIB, *SOURCES,
               *LIBS]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd, cwd=ROOT)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)

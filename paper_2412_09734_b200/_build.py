"""Builds the in-tree CUDA library libmpax_b200.so for sm_100a with nvcc.

Every .cu under csrc/ is compiled (-gencode arch=compute_100a,code=sm_100a,
-lineinfo, no fast-math: IEEE division / sqrt as the iteration contract needs)
and linked into one shared library next to this file.  Re-links only when a
source or header is newer than the library.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmpax_b200.so")
BUILD = os.path.join(HERE, "build")
DEBUG = bool(os.environ.get("MPAX_DEBUG_BUILD"))
TRACE = bool(os.environ.get("MPAX_TRACE_BUILD"))
if DEBUG:  # a separate library with device-side bounds checks (load it with MPAX_LIB=...)
    LIB = os.path.join(HERE, "libmpax_b200_debug.so")
    BUILD = os.path.join(HERE, "build_debug")
elif TRACE:  # a separate library whose grid kernel prints per-phase timings (experiments only)
    LIB = os.path.join(HERE, "libmpax_b200_trace.so")
    BUILD = os.path.join(HERE, "build_trace")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-fmad=true", "-prec-div=true", "-prec-sqrt=true", "-ftz=false", "-Xptxas", "-v"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _nccl_dirs():
    try:
        import nvidia.nccl as nn  # noqa: F401
        base = os.path.dirname(nn.__file__) if getattr(nn, "__file__", None) else list(nn.__path__)[0]
    except Exception:
        base = None
    if base and os.path.exists(os.path.join(base, "include", "nccl.h")):
        return os.path.join(base, "include"), os.path.join(base, "lib")
    return None, None


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nvcc = _nvcc()
    os.makedirs(BUILD, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    nccl_inc, nccl_lib = _nccl_dirs()
    defs = ["-DMPAX_DEBUG=1"] if DEBUG else (["-DMPAX_TRACE=1"] if TRACE else [])
    if nccl_inc:
        inc += ["-I", nccl_inc]
        defs += ["-DMPAX_HAVE_NCCL=1"]
    objs = []
    for src in sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *defs, *inc, "-c", src, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(res.stderr)
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(res.stderr)
        objs.append(obj)
    tmp = LIB + f".tmp{os.getpid()}"
    link = [nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    if nccl_lib:
        link += ["-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl_lib}"]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

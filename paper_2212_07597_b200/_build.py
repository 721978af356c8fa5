"""Build libscl.so in-tree for sm_100a (nvcc; no JIT cache, so the .so travels with the repo)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libscl.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I" + INCLUDE]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "scl.h")]


def up_to_date() -> bool:
    return os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(p) for p in deps())


def build(force: bool = False, verbose: bool = False, lib: str = LIB, extra=()) -> str:
    """Compile csrc/*.cu -> lib.  extra: additional nvcc flags (e.g. -DSCL_PROFILE for
    the debug build with per-role cycle counters, libscl_prof.so)."""
    if not force and lib == LIB and up_to_date():
        return LIB
    objs = []
    for src in sources():
        obj = os.path.join(CSRC, os.path.basename(src)[:-3] + (".prof.o" if extra else ".o"))
        cmd = [NVCC, *FLAGS, *extra, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode != 0:
            print(" ".join(cmd))
            print(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}")
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        print(r.stdout + r.stderr)
        raise RuntimeError("link of libscl.so failed")
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


PROF_LIB = os.path.join(HERE, "libscl_prof.so")

if __name__ == "__main__":
    import sys
    if "prof" in sys.argv[1:]:
        build(force=True, lib=PROF_LIB, extra=("-DSCL_PROFILE",))
    else:
        build(force=True, verbose=True)

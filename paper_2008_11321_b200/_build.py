"""In-tree build of libpgc.so (nvcc, sm_100a).  Used by __graft_entry__.build().

Each csrc/*.cu compiles to its own object under build/ (in parallel; an object
is rebuilt when its source, any csrc/*.cuh or include/pgc.h is newer), then
nvcc links the shared library.  No device code crosses translation units.
"""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libpgc.so")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "pgc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(INCLUDE, "pgc.h"),
                                                             os.path.join(INCLUDE, "pgc_debug.h")]


def deps():
    return sources() + headers()


def _obj(src):
    return os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")


def _stale_obj(src):
    o = _obj(src)
    if not os.path.exists(o):
        return True
    t = os.path.getmtime(o)
    return any(os.path.getmtime(p) > t for p in [src, *headers()])


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False, extra=()) -> str:
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    os.makedirs(OBJ, exist_ok=True)
    todo = [s for s in sources() if force or _stale_obj(s)]

    def cc(src):
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-I", INCLUDE, "-c", "-o", _obj(src), src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)

    if todo:
        with ThreadPoolExecutor(max_workers=len(todo)) as ex:
            list(ex.map(cc, todo))
    if todo or force or stale():
        subprocess.check_call([nvcc, *ARCH, "-shared", "-o", SO, *[_obj(s) for s in sources()]])
    return SO


if __name__ == "__main__":
    print(build(force=True, verbose=True))

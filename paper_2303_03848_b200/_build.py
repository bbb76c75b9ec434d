"""Builds the in-tree CUDA library (sm_100a) and, for the tests, the CPU oracle."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libparareal.so")
UNITS = ["parareal.cu", "res.cu", "streamed.cu", "pinn_smem.cu", "pinn_param.cu", "misc.cu", "pipe.cu", "pinn_tc.cu", "pinn_train.cu", "fine_grid.cu"]
HEADERS = ["launch.h", "fine_resident.cuh", "fine_streamed.cuh", "pinn_chain.cuh"]
SOURCES = UNITS + HEADERS
HEADER = os.path.join(ROOT, "include", "parareal.h")
HEADERS_ABI = [HEADER, os.path.join(ROOT, "include", "pinn_train.h")]

NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC"]
LINK_FLAGS = ["-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static", "-ldl"]
BUILD_DIR = os.path.join(ROOT, "build")


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + HEADERS_ABI
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    """Each translation unit: nvcc -gencode arch=compute_100a,code=sm_100a -c (in parallel), then
    link → paper_2303_03848_b200/libparareal.so (cudart static; NCCL is dlopen'ed at run time)."""
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(BUILD_DIR, exist_ok=True)
    nv = _nvcc()
    hdr_t = max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS + []) if HEADERS else 0
    hdr_t = max([hdr_t] + [os.path.getmtime(h) for h in HEADERS_ABI])

    def compile_unit(u):
        src = os.path.join(CSRC, u)
        obj = os.path.join(BUILD_DIR, u.replace(".cu", ".o"))
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(os.path.getmtime(src), hdr_t):
            return obj
        cmd = [nv] + NVCC_FLAGS + ["-c", "-o", obj + ".tmp", src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError("nvcc failed for %s:\n%s" % (u, r.stderr))
        os.replace(obj + ".tmp", obj)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(UNITS), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_unit, UNITS))
    tmp = LIB + ".tmp%d" % os.getpid()
    cmd = [nv] + LINK_FLAGS + ["-o", tmp] + objs
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_cuda(force, verbose)
    sys.path.insert(0, ROOT)
    import oracle  # noqa: E402  (test infrastructure: compiled here, never used by the product path)
    oracle.build(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)

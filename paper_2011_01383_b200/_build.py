"""Build libcx.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

Each .cu is compiled to an object in parallel (build/), then linked; the
shared library travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# CX_TRACE=1 selects the debug timeline build (-DCX_TRACE, libcx_trace.so, used by
# tools/trace_*.py); the default product library has no trace code on the hot path.
TRACE = os.environ.get("CX_TRACE", "0") not in ("", "0")
OBJ = os.path.join(PKG, "build_trace" if TRACE else "build")
LIB = os.path.join(PKG, "libcx_trace.so" if TRACE else "libcx.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-diag-suppress", "177"] + \
    (["-DCX_TRACE"] if TRACE else [])


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "cx.h")]


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    return _newest(sources() + _headers()) > os.path.getmtime(LIB)


def _obj(src):
    return os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = _newest(_headers())

    def compile_one(src):
        o = _obj(src)
        if not force and os.path.exists(o) and os.path.getmtime(o) >= max(hdr_t, os.path.getmtime(src)):
            return
        cmd = [NVCC] + ARCH + FLAGS + ["-c", src, "-o", o + ".tmp"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd, cwd=CSRC)
        os.replace(o + ".tmp", o)

    srcs = sources()
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        list(ex.map(compile_one, srcs))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + [_obj(s) for s in srcs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)

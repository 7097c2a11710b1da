"""Build the in-tree native libraries (sm_100a CUDA + host test build).

``libskr.so``           nvcc, -gencode arch=compute_100a,code=sm_100a, static cudart
``libskr_hostdense.so`` g++ build of csrc/dense.h + recycle.h for CPU unit tests

Rebuilds only when a source is newer than its output. Called by
``__graft_entry__.build()`` and lazily by ``_lib`` when a library is missing.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
ROOT = os.path.dirname(PKG)
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libskr.so")
HOSTLIB = os.path.join(PKG, "libskr_hostdense.so")

CUDA_SOURCES = ["gcrodr.cu", "sort.cu", "assemble.cu", "grf.cu", "precond.cu"]
HEADERS = ["dense.h", "recycle.h", "skr_device.cuh", "precond.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libskr.so")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _deps(srcs):
    return ([os.path.join(CSRC, s) for s in srcs] + [os.path.join(CSRC, h) for h in HEADERS]
            + [os.path.join(INCLUDE, "skr.h"), __file__])


def build_cuda(force: bool = False, verbose: bool = True) -> str:
    if not force and not _stale(LIB, _deps(CUDA_SOURCES)):
        return LIB
    nvcc = _nvcc()
    objs = []
    tmp = os.path.join(CSRC, "build")
    os.makedirs(tmp, exist_ok=True)
    procs = []
    for src in CUDA_SOURCES:
        obj = os.path.join(tmp, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-I", INCLUDE, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd))
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed")
    out_tmp = LIB + ".tmp"
    cmd = [nvcc, *ARCH, "-shared", "-o", out_tmp, *objs, "-lcudart_static", "-lrt", "-ldl",
           "-lpthread"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(out_tmp, LIB)
    return LIB


def build_host(force: bool = False, verbose: bool = True) -> str:
    src = os.path.join(CSRC, "host_dense.cpp")
    if not force and not _stale(HOSTLIB, _deps([]) + [src]):
        return HOSTLIB
    cxx = os.environ.get("CXX", "g++")
    cmd = [cxx, "-O2", "-std=c++17", "-fPIC", "-shared", src, "-o", HOSTLIB + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(HOSTLIB + ".tmp", HOSTLIB)
    return HOSTLIB


def build_all(force: bool = False, verbose: bool = True):
    build_host(force, verbose)
    build_cuda(force, verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)

"""Build libniyama.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python paper_2503_22562_b200/build.py [--force]     (or __graft_entry__.build())

kernels.cu (and gather.cu, the NCCL device-API unit) are compiled by nvcc with
-gencode arch=compute_100a,code=sm_100a -lineinfo; runtime.cpp, sched.cpp and
predictor.cpp by the host compiler; the shared library links the
static CUDA runtime and the NCCL that torch loads (site-packages/nvidia/nccl,
2.28.x) so a process never holds two NCCLs.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libniyama.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    purelib = sysconfig.get_paths()["purelib"]
    base = os.path.join(purelib, "nvidia", "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nccl_inc, nccl_lib = nccl_dirs()
    headers = [os.path.join(CSRC, f) for f in ("internal.h", "ptx.cuh")] + [os.path.join(INCLUDE, "niyama.h")]
    k_src = os.path.join(CSRC, "kernels.cu")
    r_src = os.path.join(CSRC, "runtime.cpp")
    k_obj = os.path.join(BUILD, "kernels.o")
    r_obj = os.path.join(BUILD, "runtime.o")
    s_src = os.path.join(CSRC, "sched.cpp")
    s_obj = os.path.join(BUILD, "sched.o")
    p_src = os.path.join(CSRC, "predictor.cpp")
    p_obj = os.path.join(BUILD, "predictor.o")
    g_src = os.path.join(CSRC, "gather.cu")
    g_obj = os.path.join(BUILD, "gather.o")
    common = ["-O3", "-std=c++17", "-I", INCLUDE, "-I", CSRC]
    if force or _stale(k_obj, [k_src] + headers):
        _run([NVCC, *ARCH, *common, "-lineinfo", "-Xptxas", "-v", "-Xcompiler", "-fPIC", "-c", k_src, "-o", k_obj])
    if force or _stale(g_obj, [g_src] + headers):
        _run([NVCC, *ARCH, *common, "-I", nccl_inc, "-Xcompiler", "-fPIC", "-c", g_src, "-o", g_obj])
    for src, obj in ((r_src, r_obj), (s_src, s_obj), (p_src, p_obj)):
        if force or _stale(obj, [src] + headers):
            _run([os.environ.get("CXX", "g++"), *common, "-I", os.path.join(CUDA, "include"), "-I", nccl_inc, "-fPIC",
                  "-Wall", "-Wextra", "-Wno-unused-parameter", "-c", src, "-o", obj])
    if force or _stale(LIB, [k_obj, g_obj, r_obj, s_obj, p_obj]):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, k_obj, g_obj, r_obj, s_obj, p_obj, "-lpthread",
              "-L", nccl_lib,
              "-l:libnccl.so.2", "-Xlinker", f"-rpath,{nccl_lib}", "-Xlinker", "--no-undefined"])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)

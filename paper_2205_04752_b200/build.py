"""In-tree native build of the package (no torch JIT, no pip install).

  lib/libhmgpu.so  -- CUDA kernels + C ABI of include/hmgpu.h (sm_100a,
                      cudart linked statically so the library loads on
                      machines without a GPU)
  lib/libhmbem.so  -- host C++ layer + C API of include/hmbem.h, linked
                      against libhmgpu.so (rpath $ORIGIN)

Run ``python paper_2205_04752_b200/build.py`` or call ``build()``.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "lib")
INC = os.path.join(ROOT, "include")
GPU_SRC = os.path.join(PKG, "csrc", "gpu")
HOST_SRC = os.path.join(PKG, "csrc", "host")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", shutil.which("g++") or "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

HOST_SOURCES = ["geometry.cpp", "cluster.cpp", "quadrature.cpp", "operator.cpp", "sparse_ops.cpp",
                "capi.cpp"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _glob(d: str, exts: tuple[str, ...]) -> list[str]:
    return [os.path.join(d, f) for f in sorted(os.listdir(d)) if f.endswith(exts)]


def build(force: bool = False, verbose_ptxas: bool = False) -> None:
    os.makedirs(LIB, exist_ok=True)
    gpu_so = os.path.join(LIB, "libhmgpu.so")
    gpu_deps = _glob(GPU_SRC, (".cu", ".cuh")) + [os.path.join(INC, "hmgpu.h")]
    if force or _newer(gpu_so, gpu_deps):
        # --fmad=false: every fused multiply-add in device code is an explicit
        # fma(), so the ACA arithmetic is bit-reproducible by the CPU oracle
        cmd = [NVCC, "-std=c++17", "-O3", *ARCH, "-lineinfo", "--fmad=false",
               "-Xcompiler", "-fPIC",
               "-Xcompiler", "-ffp-contract=off", "-I", INC, "-shared", "-cudart",
               "static", "-o", gpu_so, os.path.join(GPU_SRC, "hmgpu.cu")]
        if verbose_ptxas:
            cmd.insert(3, "-Xptxas=-v")
        _run(cmd)
    host_so = os.path.join(LIB, "libhmbem.so")
    host_deps = _glob(HOST_SRC, (".cpp", ".hpp")) + [os.path.join(INC, "hmbem.h"),
                                                      os.path.join(INC, "hmgpu.h"), gpu_so]
    if force or _newer(host_so, host_deps):
        _run([CXX, "-std=c++17", "-O3", "-DNDEBUG", "-ffp-contract=off", "-fPIC", "-shared",
              "-pthread", "-Wall", "-I", INC, "-I", HOST_SRC,
              *[os.path.join(HOST_SRC, s) for s in HOST_SOURCES],
              "-L", LIB, "-lhmgpu", "-Wl,-rpath,$ORIGIN", "-o", host_so])


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)

"""In-tree build of ``lib/libocto_b200.so`` (C ABI + C++ API + sm_100a kernels).

``python paper_2209_12310_b200/build.py`` (or ``__graft_entry__.build()``); it
is a standalone script so it never imports the package it builds.
The CUDA translation unit is compiled for sm_100a only
(``-gencode arch=compute_100a,code=sm_100a``) with FMA contraction disabled
(``-fmad=false``); host translation units use ``-ffp-contract=off`` and no
``-march`` so host-side binary64 arithmetic matches the reference objects.
The CUDA runtime is linked statically, so the library needs only the driver.
Rebuilds are incremental on source/header mtimes.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "build")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libocto_b200.so")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
CXX = os.environ.get("CXX", "g++")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-fmad=false", "-std=c++20",
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-I", INCLUDE, "-I", CSRC,
]
CXX_FLAGS = [
    "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-fopenmp",
    "-Wall", "-Wextra", "-I", INCLUDE, "-I", CSRC,
    "-I", os.path.join(CUDA_HOME, "include"),
]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(INCLUDE, "**", "*.h*"), recursive=True)


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build step failed ({r.returncode}):\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stdout.strip() or r.stderr.strip()):
        print(r.stdout + r.stderr, flush=True)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    hdrs = _headers()
    objs = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        if force or _stale(obj, [src] + hdrs):
            _run([NVCC] + NVCC_FLAGS + ["-c", src, "-o", obj], verbose)
        objs.append(obj)
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cpp"))):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        if force or _stale(obj, [src] + hdrs):
            _run([CXX] + CXX_FLAGS + ["-c", src, "-o", obj], verbose)
        objs.append(obj)
    if force or _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs +
             ["-Xcompiler", "-fopenmp", "-lgomp", "-lpthread"], verbose)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))

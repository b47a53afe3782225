"""Compile the sm_100a CUDA library (in-tree, so the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = os.path.join(PKG, "csrc", "sdedge.cu")
HDR = os.path.join(ROOT, "include", "sdedge.h")
LIB = os.environ.get("SDEDGE_LIB") or os.path.join(PKG, "libsdedge.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    lib = out or LIB
    stale = (not os.path.exists(lib) or
             os.path.getmtime(lib) < max(os.path.getmtime(SRC), os.path.getmtime(HDR)))
    if force or stale:
        cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
               "-o", lib, SRC]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
    return lib

"""Builds paper_2605_19893_b200/lib/libspecsv_b200.so for sm_100a (in-tree).

    python -m paper_2605_19893_b200.build          # incremental
    python -m paper_2605_19893_b200.build --force
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libspecsv_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["attend.cu", "route.cu", "route3.cu", "compress.cu", "draft_tree.cu", "abi.cpp", "policy.cpp", "planner.cpp"]
HEADERS = ["attend.h", "sm100.cuh", "policy.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(os.path.join(LIBDIR, "obj"), exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "specsv_b200", "nsa_verify.h"),
        os.path.join(ROOT, "include", "specsv_b200", "planner.h"),
        os.path.join(ROOT, "include", "specsv_b200", "draft_tree.h")]
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(LIBDIR, "obj", src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + hdrs):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", path, "-o", obj]
            if os.environ.get("SPECSV_TRACE_TILES"):  # diagnostics build: per-tile stamps (--force)
                cmd.append("-DSPECSV_TRACE_TILES")
            if src.endswith(".cu"):
                cmd += ["-Xptxas", "-v"] if verbose else []
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)

"""Build the sm_100a CUDA library in-tree (no GPU needed: nvcc cross-compiles).

Parity build flags: -fmad=false -prec-div=true
-prec-sqrt=true, no fast-math, so the float arithmetic matches the
reference's Solver<float> bit for bit.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", "apbf_gpu.cu")]
DEPS = [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))] + [
    os.path.join(ROOT, "include", "apbf_gpu.h")]
OUT = os.path.join(HERE, "libapbf_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=default", "-shared"]


def _stale(out, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


CHECKED = os.path.join(HERE, "libapbf_gpu_checked.so")


def build_cuda(force: bool = False, checked: bool = True) -> str:
    """libapbf_gpu.so (the product) and libapbf_gpu_checked.so: the same code
    with -DAPBF_CHECKED device asserts on every data-derived index (selected
    with APBF_LIB=libapbf_gpu_checked.so; tools/checked_run.sh)."""
    if force or _stale(OUT, DEPS):
        cmd = [NVCC, *FLAGS, "-o", OUT, *SOURCES]
        print("[build]", " ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    if checked and (force or _stale(CHECKED, DEPS)):
        cmd = [NVCC, *FLAGS, "-DAPBF_CHECKED", "-o", CHECKED, *SOURCES]
        print("[build]", " ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return OUT


def build_oracle() -> None:
    """oracle/liboracle.so always; oracle/_ref only when /root/reference exists."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "all"], check=True)
    # tools/_bin/e2e_cpp: the C++ drop-in timed end to end (bench.py e2e_cpp)
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools"), "all"], check=True)


if __name__ == "__main__":
    build_cuda(force="--force" in sys.argv)
    build_oracle()

"""Build libkep.so in-tree for sm_100a (nvcc; no torch JIT cache).

    python -m paper_1710_05134_b200.build      # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libkep.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
METIS = "/usr/local/cuda/lib64/libcusolver_metis_static.a"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
           "--expt-relaxed-constexpr", "-Xptxas", "-v"]
SOURCES_CU = ["api.cu", "kernels.cu", "kernels_front.cu", "kernels_fast.cu", "kernels_solve.cu", "kth.cu", "kernels_resid.cu", "kernels_small.cu", "kernels_big.cu"]
SOURCES_CPP = ["symbolic.cpp", "tridiag.cpp"]


def _run(cmd, log):
    log.write(" ".join(cmd) + "\n")
    log.flush()
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    log.write(r.stdout)
    if r.returncode != 0:
        sys.stderr.write(r.stdout)
        raise RuntimeError(f"build failed: {' '.join(cmd)}")
    return r.stdout


def build(verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    logpath = os.path.join(LIBDIR, "build.log")
    objs = []
    with open(logpath, "w") as log:
        for src in SOURCES_CU:
            obj = os.path.join(objdir, src + ".o")
            _run([NVCC, *ARCH, *CUFLAGS, "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, src), "-o", obj], log)
            objs.append(obj)
        for src in SOURCES_CPP:
            obj = os.path.join(objdir, src + ".o")
            _run(["g++", "-O3", "-std=c++17", "-fPIC", "-fvisibility=hidden", "-g",
                  "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, src), "-o", obj], log)
            objs.append(obj)
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, METIS, "-Xlinker", "--exclude-libs,ALL", "-Xlinker", "-z,defs",
              "-lm"], log)
    if verbose:
        print(open(logpath).read())
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))

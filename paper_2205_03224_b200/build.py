"""Build libgemslr.so in-tree: host setup (g++) + sm_100a kernels (nvcc).

Host setup code is compiled with -ffp-contract=off so its ILU arithmetic is
plain IEEE round-to-nearest (reading Q22); device code keeps nvcc's
default FMA contraction.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libgemslr.so")
BUILD = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# GEMSLR_TRACE=1: compile the clock64 trace of k_tri_reg in (tools/trace_reg.py)
TRACE = ["-DGEMSLR_TRACE"] if os.environ.get("GEMSLR_TRACE") == "1" else []
# experiments: GEMSLR_NVCC_DEFS="-DNAME=VALUE ..." extra defines (e.g. SPLIT_BACKOFF_NS)
TRACE += os.environ.get("GEMSLR_NVCC_DEFS", "").split()

CPP = ["partition.cpp", "ilu.cpp", "schedule.cpp", "hostplan.cpp", "schur.cpp"]
CU = ["context.cu"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[0]} {cmd[-1]}")
    return r


def sources():
    deps = [os.path.join(SRC, f) for f in os.listdir(SRC)]
    deps.append(os.path.join(ROOT, "include", "gemslr.h"))
    return deps


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(p) > t for p in sources())


def build(force=False, verbose=False):
    if not force and not needs_build():
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    inc = ["-I", os.path.join(ROOT, "include"), "-I", SRC]
    for f in CPP:
        o = os.path.join(BUILD, f + ".o")
        _run(["g++", "-std=c++17", "-O2", "-fPIC", "-fopenmp", "-ffp-contract=off", "-Wall", *inc, "-c",
              os.path.join(SRC, f), "-o", o])
        objs.append(o)
    for f in CU:
        o = os.path.join(BUILD, f + ".o")
        r = _run([NVCC, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xptxas", "-v", "-Xcompiler", "-fPIC,-fopenmp",
                  *TRACE, *inc, "-c", os.path.join(SRC, f), "-o", o])
        if verbose:
            sys.stderr.write(r.stderr)
        with open(os.path.join(BUILD, f + ".ptxas.txt"), "w") as fh:
            fh.write(r.stderr)
        objs.append(o)
    tmp = OUT + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fopenmp", "-lgomp"])
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)

"""Builds libslm.so in-tree: host planner (g++) + sm_100a runtime/kernels (nvcc).

The library is the product: `paper_1604_06174_b200._lib` loads it with ctypes and fails
loudly if it is missing.  nvcc cross-compiles sm_100a without a GPU.
"""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libslm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INC = ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC))


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]
    return all(os.path.getmtime(f) <= t for f in deps)


def build(force=False, verbose_ptxas=False):
    if not force and up_to_date():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    o = os.path.join(BUILD, "planner.o")
    _run(["g++", "-std=c++17", "-O2", "-fPIC", "-Wall", *INC, "-c", os.path.join(CSRC, "planner.cpp"), "-o", o])
    objs.append(o)
    o = os.path.join(BUILD, "runtime.o")
    flags = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", *ARCH, *INC]
    if verbose_ptxas:
        flags += ["-Xptxas", "-v"]
    _run([NVCC, *flags, "-c", os.path.join(CSRC, "runtime.cu"), "-o", o])
    objs.append(o)
    tmp = LIB + ".tmp"
    _run([NVCC, "-shared", *ARCH, "-o", tmp, *objs, "-cudart", "static", "-ldl", "-lpthread"])
    os.replace(tmp, LIB)
    return LIB


def build_variant(name, defines):
    """An experimental in-tree variant of the library (compile-time kernel experiments), loaded by
    setting SLM_LIB=<name> (paper_1604_06174_b200/_lib.py); not part of the product build."""
    os.makedirs(BUILD, exist_ok=True)
    po = os.path.join(BUILD, "planner.o")
    if not os.path.exists(po):
        _run(["g++", "-std=c++17", "-O2", "-fPIC", "-Wall", *INC, "-c", os.path.join(CSRC, "planner.cpp"), "-o", po])
    o = os.path.join(BUILD, f"runtime_{name}.o")
    _run([NVCC, "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", *ARCH, *INC, *["-D" + d for d in defines],
          "-c", os.path.join(CSRC, "runtime.cu"), "-o", o])
    out = os.path.join(PKG, name)
    _run([NVCC, "-shared", *ARCH, "-o", out, po, o, "-cudart", "static", "-ldl", "-lpthread"])
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:   # --variant NAME.so DEF1 DEF2 ...
        i = sys.argv.index("--variant")
        build_variant(sys.argv[i + 1], sys.argv[i + 2:])
    else:
        build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)

"""Build libgiga.so in-tree: nvcc for sm_100a (cross-compiles without a GPU).

The shared library is the product: the sm_100a kernels, the C ABI of include/giga.h and
the orchestration. NCCL is resolved at run time (dlopen), cudart is linked statically.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgiga.so")
DEBUG_LIB = os.path.join(HERE, "libgiga_debug.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["gemm_3xtf32.cu", "prep16.cu", "vecops.cu"]
CPP_SOURCES = ["api.cpp", "runtime.cpp", "pipeline_nccl.cpp", "p2p.cpp", "host_pipeline.cpp",
               "host_plan.cpp", "nccl_loader.cpp", "mcast.cpp"]
HEADERS = ["ptx.cuh", "split16.cuh", "kernels.h", "nccl_loader.h", "host_plan.h", "runtime.h", "debug_kernels.cu"]


def nccl_paths():
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        inc = os.path.join(base, "nccl", "include")
        lib = os.path.join(base, "nccl", "lib", "libnccl.so.2")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", ""


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    nccl_inc, nccl_lib = nccl_paths()
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES + CPP_SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "giga.h"), os.path.abspath(__file__)]
    if not force and not _stale(LIB, deps):
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
              "-I", nccl_inc, f'-DGIGA_NCCL_PATH="{nccl_lib}"']
    objs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        cmd = [NVCC, *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", *common, "-c", s, "-o", o]
        if s.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd += ["-x", "c++"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        objs.append(o)
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
                           "-ldl", "-lpthread"])
    os.replace(tmp, LIB)
    # bring-up probes (not the product path): debug kernels + the TMA encoder helper
    dsrc = os.path.join(CSRC, "debug_kernels.cu")
    do = os.path.join(objdir, "debug_kernels.cu.o")
    subprocess.check_call([NVCC, *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", *common, "-c",
                           dsrc, "-o", do])
    tmp = DEBUG_LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, do,
                           os.path.join(objdir, "gemm_3xtf32.cu.o"), "-ldl", "-lpthread"])
    os.replace(tmp, DEBUG_LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))

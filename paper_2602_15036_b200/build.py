"""Build the in-tree native library paper_2602_15036_b200/liblithogpu.so.

nvcc -gencode arch=compute_100a,code=sm_100a for the CUDA translation units,
g++ -fopenmp for the host kernel generator; one shared library, no torch
types in any signature (the C ABI is include/lithogpu.h).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "liblithogpu.so")
OBJ = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = ["csrc/capi.cu", "csrc/fast_rows.cu", "csrc/fast_cols.cu", "csrc/kernelgen.cu"]
CPP_SOURCES = ["host/socs_kernels.cpp", "host/layout_io.cpp"]
# nlohmann/json (header-only; the reference's own JSON library) for the layout reader
JSON_INC = os.environ.get("LITHO_JSON_INC", "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/"
                                           "cudnn_frontend/thirdparty/nlohmann")
CUDA_INC = "/usr/local/cuda/include"
_FAST = ["csrc/fast_common.cuh", "csrc/socs_fast.cuh", "csrc/fftr.cuh", "csrc/fft.cuh", "csrc/socs_fast.h",
         "csrc/geom.h"]
# per-source header dependencies (incremental rebuilds)
DEPS = {
    "csrc/capi.cu": ["csrc/fft.cuh", "csrc/geom.h", "csrc/socs_kernels.cuh", "csrc/raster_kernels.cuh",
                     "csrc/util_kernels.cuh", "csrc/socs_fast.h", "csrc/contour_kernels.cuh",
                     "../include/lithogpu.h"],
    "csrc/fast_rows.cu": _FAST,
    "csrc/fast_cols.cu": _FAST,
    "csrc/kernelgen.cu": ["../include/lithogpu.h"],
}


def _newer(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(os.path.join(HERE, s)) > t for s in sources)


def _run(cmd):
    r = subprocess.run(cmd, cwd=HERE, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=(), objdir: str = OBJ) -> str:
    """Compile the library (incrementally).  `defines` / `out` / `objdir`
    build an A/B variant of the same sources (e.g. -DLG_ADJROWS_MINB=4 into
    variants/<name>/liblithogpu.so, loaded with LITHOGPU_LIB)."""
    os.makedirs(objdir, exist_ok=True)
    jobs = []
    objs = []
    dflags = ["-D" + d for d in defines]
    for src in CU_SOURCES:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + DEPS[src] + [os.path.relpath(__file__, HERE)]):
            jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *dflags,
                         "-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj])
    for src in CPP_SOURCES:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _newer(obj, [src, "../include/lithogpu.h"]):
            jobs.append(["g++", "-O2", "-std=c++17", "-fPIC", "-fopenmp", "-ffp-contract=off",
                         "-I" + JSON_INC, "-I" + CUDA_INC, "-c", src, "-o", obj])
    with ThreadPoolExecutor(max_workers=8) as ex:
        for r in ex.map(_run, jobs):
            if verbose:
                sys.stderr.write(r.stderr)
    if force or jobs or not os.path.exists(out):
        _run([NVCC, *ARCH, "-shared", "-o", out, *objs, "-lgomp", "-lcudart", "-lcublas", "-lcusolver"])
    return out


def build_variant(name: str, defines, fast_only: bool = True) -> str:
    """variants/<name>/liblithogpu.so with extra -D flags (A/B timing).
    fast_only: the -D flags only reach the fp32 fast-path kernels
    (fast_rows.cu / fast_cols.cu); the other objects come from the main
    build (built first)."""
    import shutil
    d = os.path.join(ROOT, "variants", name)
    objdir = os.path.join(d, "obj")
    if fast_only:
        build()
        os.makedirs(objdir, exist_ok=True)
        for src in CU_SOURCES + CPP_SOURCES:
            if src in ("csrc/fast_rows.cu", "csrc/fast_cols.cu"):
                continue
            o = os.path.basename(src) + ".o"
            shutil.copy2(os.path.join(OBJ, o), os.path.join(objdir, o))
    return build(out=os.path.join(d, "liblithogpu.so"), defines=defines, objdir=objdir)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

"""Build the sm_100a extension in-tree: paper_2510_05254_b200/libndgx.so.

    python -m paper_2510_05254_b200.build [--force]

nvcc cross-compiles for sm_100a without a GPU.  Each translation unit is
compiled in parallel; the result is a self-contained shared library (static
cudart) exporting the C ABI declared in include/ndgx.h.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libndgx.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
         "-I", INCLUDE, "-I", CSRC]

# (source, object name, extra defines): the stage kernels are instantiated
# once per (dim, order, arithmetic) so the objects compile in parallel
SOURCES = [("ndgx_solver.cu", "ndgx_solver", []), ("ndgx_registry.cu", "ndgx_registry", []),
           ("ndgx_setup.cpp", "ndgx_setup", []), ("ndgx_nccl.cpp", "ndgx_nccl", [])] + [
    ("ndgx_inst.cu", f"ndgx_inst_d{d}_o{n}_e{e}",
     [f"-DNDGX_DIM={d}", f"-DNDGX_ORDER={n}", f"-DNDGX_EXACT={e}"])
    for d in (1, 2, 3) for n in range(2, 9) for e in (0, 1)]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src, os.path.join(INCLUDE, "ndgx.h")] + [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(item) -> str:
    src, name, defs = item
    obj = os.path.join(BUILD, name + ".o")
    path = os.path.join(CSRC, src)
    if _stale(obj, path):
        cmd = [NVCC] + ARCH + FLAGS + defs + ["-c", path, "-o", obj]
        if src.endswith(".cpp"):
            cxx = os.environ.get("CXX", shutil.which("g++") or "g++")
            cuda_inc = os.path.join(os.path.dirname(os.path.dirname(os.path.realpath(NVCC))), "include")
            cmd = [cxx, "-O2", "-fPIC", "-ffp-contract=off", "-std=c++17", "-I", INCLUDE, "-I", CSRC, "-I", cuda_inc,
                   "-c", path, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    if force:
        for f in os.listdir(BUILD):
            os.remove(os.path.join(BUILD, f))
    # the heaviest objects (3D and high orders) first
    order = sorted(SOURCES, key=lambda it: -sum(int(d.split("=")[1]) for d in it[2][:2]) if it[2] else 0)
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        done = dict(zip([it[1] for it in order], ex.map(_compile, order)))
    objs = [done[it[1]] for it in SOURCES]
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)

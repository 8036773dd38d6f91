"""Build the sm_100a extension in-tree: paper_2506_12204_b200/_lib/libsemsched_b200.so.

    python -m paper_2506_12204_b200.build

nvcc cross-compiles without a GPU. ``-fmad=false`` keeps the reference's
float64 chains unfused (bit-exact f_t, clocks and eviction costs).
"""

from __future__ import annotations

import os
import subprocess
import sys
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libsemsched_b200.so")
SOURCES = ["ss_kernel.cu", "ss_prepass.cu", "ss_epilogue.cu", "ss_step.cu", "ss_audit.cu", "ss_api.cu", "ss_tracegen.cpp", "ss_tracegen_dev.cu"]
HEADERS = ["ss_kernel.cuh", "ss_common.cuh", "ss_costs.cuh", "../../include/semsched_b200.h",
           "../../include/semsched_tracegen.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    """``defines``/``out`` build an experimental variant (e.g. SS_MINB=6)."""
    lib = out or LIB
    if not force and not _stale() and out is None:
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = LIBDIR if out is None else tempfile.mkdtemp(prefix="ss_build_")  # variants build in parallel
    def compile_one(src):
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        if src.endswith(".cpp"):
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-ffp-contract=off", "-pthread",
                   "-c", os.path.join(CSRC, src), "-o", obj]
        else:
            cmd = ([nvcc()] + NVCC_FLAGS + ["-Xptxas", "-v"] * verbose + [f"-D{d}" for d in defines]
                   + ["-c", os.path.join(CSRC, src), "-o", obj])
        subprocess.run(cmd, check=True)
        return obj

    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    tmp = lib + ".tmp"
    subprocess.run([nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs, check=True)
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv or bool(defs), verbose="-v" in sys.argv, defines=defs,
                out=outs[0] if outs else None))

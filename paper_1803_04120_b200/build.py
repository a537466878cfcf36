"""Build libsj.so in-tree for sm_100a (B200).  No JIT, no torch extension: plain nvcc.

    python -m paper_1803_04120_b200.build [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libsj.so")
SOURCES = ["api.cu", "context.cu", "index_build.cu", "radix_sort.cu", "join.cu", "extras.cu", "diag.cu",
           "refine_d2.cu", "refine_d3.cu", "refine_d4.cu", "refine_d5.cu", "refine_d6.cu", "dbscan.cu", "variants.cu"]
HEADERS = ["sj_common.cuh", "refine.cuh", "refine_launch.cuh", "scan.cuh"]

OBJDIR = os.path.join(ROOT, "build", "obj")
NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "--fmad=false",              # no FMA contraction anywhere (reading R1); refine also uses _rn intrinsics
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
    f"-I{INCLUDE}",
]
LINK_FLAGS = ["-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _deps_mtime() -> float:
    deps = [os.path.join(CSRC, f) for f in HEADERS] + [os.path.join(INCLUDE, "sj.h"), os.path.abspath(__file__)]
    return max(os.path.getmtime(p) for p in deps)


def _obj(src: str) -> str:
    return os.path.join(OBJDIR, os.path.splitext(src)[0] + ".o")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return _deps_mtime() > t or any(os.path.getmtime(os.path.join(CSRC, f)) > t for f in SOURCES)


def build(force: bool = False, verbose: bool = False) -> str:
    """nvcc -c every translation unit (in parallel, only the stale ones), then link libsj.so."""
    if not force and not _stale():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    dep_t = _deps_mtime()

    def compile_one(src):
        o = _obj(src)
        path = os.path.join(CSRC, src)
        if not force and os.path.exists(o) and os.path.getmtime(o) >= max(dep_t, os.path.getmtime(path)):
            return None
        tmp = o + f".tmp{os.getpid()}"
        cmd = [nvcc(), *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), "-c", path, "-o", tmp]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            return f"{src}:\n{r.stdout}{r.stderr}"
        if verbose:
            sys.stderr.write(r.stderr)
        os.replace(tmp, o)
        return None

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        errs = [e for e in ex.map(compile_one, SOURCES) if e]
    if errs:
        sys.stderr.write("\n".join(errs))
        raise RuntimeError("nvcc failed building libsj.so")
    tmp = LIB + f".tmp{os.getpid()}"
    r = subprocess.run([nvcc(), *LINK_FLAGS, *[_obj(f) for f in SOURCES], "-o", tmp], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libsj.so")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose="--verbose" in sys.argv))

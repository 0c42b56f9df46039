"""Build libtw_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2008_13006_b200.build        (or __graft_entry__.build())

`-gencode arch=compute_100a,code=sm_100a` (not -arch=sm_100a, which also
emits compute_100 PTX that ptxas rejects for tcgen05).  -lineinfo keeps the
ncu source page mapped.  The CUDA runtime is linked statically; the driver
entry point for cuTensorMapEncodeTiled is fetched at run time, so the .so
loads on a CPU-only box (compute calls then fail with TW_ERR_CUDA).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libtw_b200.so")

SOURCES = ["tw_pack.cpp", "tw_schedule.cpp", "tw_capi.cu", "tw_gemm_sm100.cu", "tw_aux.cu"]
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, ptxas_verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    cc = nvcc()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(INCLUDE, "tw_b200.h"))
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC]
    # (experiments) extra nvcc flags, e.g. -DTW_K2_STAGES=2; clear _build/ to rebuild
    common += os.environ.get("TW_B200_NVCC_FLAGS", "").split()
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if not _stale(obj, [path, *headers, __file__]):
            continue
        cmd = [cc, *common, *GENCODE, "-lineinfo", "-c", path, "-o", obj]
        if ptxas_verbose and src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    if _stale(LIB, objs):
        tmp = LIB + ".tmp"
        cmd = [cc, *GENCODE, "-shared", "-cudart", "static", "-o", tmp, *objs]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, ptxas_verbose="-v" in sys.argv))

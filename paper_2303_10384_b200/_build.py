"""Builds the sm_100a C-ABI library in-tree: paper_2303_10384_b200/lib/librnnt_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, static cudart, one object per kernel file,
linked with -shared.  Cross-compiles without a GPU.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB_DIR = os.path.join(PKG, "lib")
BUILD_PATH = os.path.join(LIB_DIR, "librnnt_b200.so")
# RNNT_B200_LIB overrides the library the binding loads (A/B timing of kernel variants on one box).
LIB_PATH = os.environ.get("RNNT_B200_LIB") or BUILD_PATH
OBJ_DIR = os.path.join(PKG, "lib", "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                     "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(BUILD_PATH):
        return True
    t = os.path.getmtime(BUILD_PATH)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return BUILD_PATH
    os.makedirs(OBJ_DIR, exist_ok=True)
    cc = nvcc()

    def compile_one(src):
        obj = os.path.join(OBJ_DIR, os.path.basename(src)[:-3] + ".o")
        r = subprocess.run([cc, *NVCC_FLAGS, "-c", src, "-o", obj], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, sources()))
    if verbose:
        for _, log in results:
            print(log)
    tmp = BUILD_PATH + f".tmp{os.getpid()}"
    # No library GEMMs: every kernel on the path is this library's own (libcuda is reached through the runtime's
    # driver entry points, e.g. cuTensorMapEncodeTiled).
    r = subprocess.run([cc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *[o for o, _ in results]],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, BUILD_PATH)
    return BUILD_PATH


if __name__ == "__main__":
    print(build(force=True, verbose=True))

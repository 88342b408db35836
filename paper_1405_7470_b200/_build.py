"""Build the in-tree CUDA library paper_1405_7470_b200/liblpy.so for sm_100a.

nvcc cross-compiles here without a GPU.  The explicit `-gencode
arch=compute_100a,code=sm_100a` form is required: plain -arch=sm_100a does not
assemble tcgen05.  cudart is linked statically so the .so
does not depend on torch's bundled runtime version; the driver API
(cuTensorMapEncodeTiled) is reached through cudaGetDriverEntryPoint, so no
-lcuda is needed at link time.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "liblpy.so")
PROBE_LIB = os.path.join(PKG, "liblpy_probe.so")   # hardware probes (tests/diagnostics only)

SOURCES = ["lpy_api.cu", "gemm_ffma.cu", "gemm_3xtf32.cu", "repack.cu"]
PROBE_SOURCES = ["probe_tcgen05.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{INCLUDE}",
                     "-Xptxas", "-v"]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found: cannot build the sm_100a library")
    return path


def _deps_mtime() -> float:
    files = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str, force: bool) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.splitext(src)[0] + ".o")
    srcp = os.path.join(CSRC, src)
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(srcp),
                                                                          _deps_mtime()):
        return obj, ""
    r = subprocess.run([nvcc(), *NVCC_FLAGS, "-c", srcp, "-o", obj], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every CUDA source and link liblpy.so; returns the library path."""
    os.makedirs(BUILD, exist_ok=True)
    allsrc = SOURCES + PROBE_SOURCES
    with cf.ThreadPoolExecutor(max_workers=min(8, len(allsrc))) as ex:
        results = dict(zip(allsrc, ex.map(lambda s: _compile(s, force), allsrc)))
    if verbose:
        for _, log in results.values():
            if log:
                print(log)
    for lib, srcs in ((LIB, SOURCES), (PROBE_LIB, PROBE_SOURCES)):
        objs = [results[s][0] for s in srcs]
        if force or not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs):
            tmp = lib + f".tmp{os.getpid()}"
            r = subprocess.run([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs],
                               capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
            os.replace(tmp, lib)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose=True))

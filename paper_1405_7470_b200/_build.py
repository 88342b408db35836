"""Build the in-tree CUDA libraries for sm_100a.

  liblpy.so        the product: C-ABI front end + FFMA and 3xTF32 kernels
  liblpy_probe.so  hardware probes (tcgen05 numerics, MMA / FFMA rates) for tests
  liblpy_trace.so  diagnostics: the product built with -DLPY_TRACE (per-CTA cycle
                   counters in the 3xTF32 kernel); never loaded by the product path
  liblpy_mutant.so the product with -DLPY_MUTATE_STAGE_RACE: each kernel's stage
                   hand-off broken (FFMA consumers release a stage before reading
                   it, the 3xTF32 split transform marks a stage ready before
                   writing its small parts) -- the race
                   detector tests must FAIL on it (tests/test_mutation_gpu.py);
                   never loaded by the product path

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
PROBE_LIB = os.path.join(PKG, "liblpy_probe.so")
TRACE_LIB = os.path.join(PKG, "liblpy_trace.so")
MUTANT_LIB = os.path.join(PKG, "liblpy_mutant.so")

SOURCES = ["lpy_api.cu", "gemm_ffma.cu", "gemm_3xtf32.cu", "repack.cu", "saxpy.cu", "coulomb.cu", "kgate.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{INCLUDE}",
                     "-Xptxas", "-v"]

# (object name, source, extra flags)
OBJECTS = [(os.path.splitext(s)[0], s, []) for s in SOURCES] + [
    ("probe_tcgen05", "probe_tcgen05.cu", []),
    ("gemm_3xtf32_trace", "gemm_3xtf32.cu", ["-DLPY_TRACE"]),
    ("gemm_ffma_mutant", "gemm_ffma.cu", ["-DLPY_MUTATE_STAGE_RACE"]),
    ("gemm_3xtf32_mutant", "gemm_3xtf32.cu", ["-DLPY_MUTATE_STAGE_RACE"]),
]
LIBS = [
    (LIB, [os.path.splitext(s)[0] for s in SOURCES]),
    (PROBE_LIB, ["probe_tcgen05"]),
    (TRACE_LIB, ["lpy_api", "gemm_ffma", "gemm_3xtf32_trace", "repack", "saxpy", "coulomb", "kgate"]),
    (MUTANT_LIB, ["lpy_api", "gemm_ffma_mutant", "gemm_3xtf32_mutant", "repack", "saxpy", "coulomb", "kgate"]),
]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found: cannot build the sm_100a library")
    return path


def _deps_mtime() -> float:
    files = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))
    return max(os.path.getmtime(f) for f in files)


def _compile(name: str, src: str, extra: list[str], force: bool) -> tuple[str, str]:
    obj = os.path.join(BUILD, name + ".o")
    srcp = os.path.join(CSRC, src)
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(srcp),
                                                                          _deps_mtime()):
        return obj, ""
    r = subprocess.run([nvcc(), *NVCC_FLAGS, *extra, "-c", srcp, "-o", obj], capture_output=True,
                       text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every CUDA source and link the libraries; returns liblpy.so's path."""
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(OBJECTS))) as ex:
        results = dict(zip([o[0] for o in OBJECTS],
                           ex.map(lambda o: _compile(o[0], o[1], o[2], force), OBJECTS)))
    if verbose:
        for _, log in results.values():
            if log:
                print(log)
    for lib, names in LIBS:
        objs = [results[n][0] for n in names]
        if force or not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs):
            tmp = lib + f".tmp{os.getpid()}"
            r = subprocess.run([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs],
                               capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
            os.replace(tmp, lib)
    return LIB


def build_variant(name: str, flags: list[str]) -> str:
    """Experimental copy of the product library compiled with extra nvcc flags
    (e.g. -DLPY_MMA_ORDER_B) as liblpy_<name>.so, for A/B timing
    (scripts/ab_lib.py).  Never loaded by the product path."""
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(BUILD, f"{os.path.splitext(src)[0]}_{name}.o")
        r = subprocess.run([nvcc(), *NVCC_FLAGS, *flags, "-c", os.path.join(CSRC, src), "-o", obj],
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        objs.append(obj)
    lib = os.path.join(PKG, f"liblpy_{name}.so")
    r = subprocess.run([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", lib, *objs],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return lib


if __name__ == "__main__":
    import sys
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":
        print(build_variant(sys.argv[2], sys.argv[3:]))
    else:
        print(build(force="--force" in sys.argv, verbose=True))

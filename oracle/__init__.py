"""ORACLE -- TEST INFRASTRUCTURE ONLY.

ctypes loader for oracle/oracle.c, the plain float64 CPU triple loop that
defines what the CUDA path must compute (section 2.1:
``sum(k, a[i,k]*b[k,j])``).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs may import this package;
the product package paper_1405_7470_b200 never does (tests/test_isolation.py
checks that).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liblpy_oracle.so")
_lock = threading.Lock()
_lib = None

ROW_MAJOR = 0
COL_MAJOR = 1


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (no fast-math, no FP contraction, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.run(["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
                        "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"], check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            i64, i32, fp, dp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p
            lib.lpy_oracle_gemm_rows_f64.argtypes = [i64, i64, i64, fp, i64, i32, fp, i64, i32,
                                                     i64, i64, dp, dp, i32]
            lib.lpy_oracle_gemm_rows_f64.restype = i32
            lib.lpy_oracle_gemm_elems_f64.argtypes = [i64, i64, i64, fp, i64, i32, fp, i64, i32,
                                                      i64, fp, fp, dp, dp, i32]
            lib.lpy_oracle_gemm_elems_f64.restype = i32
            lib.lpy_oracle_saxpy_f64.argtypes = [i64, ctypes.c_float, fp, i64, fp, i64, dp, i32]
            lib.lpy_oracle_saxpy_f64.restype = i32
            lib.lpy_oracle_coulomb_f64.argtypes = [i64, fp, i64, i64, fp, i64, fp, dp, dp, i32]
            lib.lpy_oracle_coulomb_f64.restype = i32
            lib.lpy_oracle_max_threads.argtypes = []
            lib.lpy_oracle_max_threads.restype = i32
            _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a.size else None


def _check_buf(buf: np.ndarray):
    if buf.dtype != np.float32 or not buf.flags.c_contiguous:
        raise TypeError("oracle inputs are contiguous float32 buffers")


def gemm_rows(M, N, K, A, lda, la, B, ldb, lb, row0=0, row1=None, nthreads=0):
    """Rows [row0, row1) of C = A*B and D = |A|*|B| in float64 (packed row-major)."""
    row1 = M if row1 is None else row1
    _check_buf(A)
    _check_buf(B)
    C = np.empty((row1 - row0, N), dtype=np.float64)
    D = np.empty((row1 - row0, N), dtype=np.float64)
    rc = _load().lpy_oracle_gemm_rows_f64(M, N, K, _ptr(A), lda, la, _ptr(B), ldb, lb,
                                           row0, row1, _ptr(C), _ptr(D), int(nthreads))
    if rc != 0:
        raise ValueError("oracle rejected its arguments")
    return C, D


def gemm(M, N, K, A, lda, la, B, ldb, lb, nthreads=0):
    """Full C = A*B and D = |A|*|B| in float64."""
    return gemm_rows(M, N, K, A, lda, la, B, ldb, lb, 0, M, nthreads)


def gemm_elems(M, N, K, A, lda, la, B, ldb, lb, ii, jj, nthreads=0):
    """C and D at the (ii[e], jj[e]) pairs only (same k order as `gemm`)."""
    _check_buf(A)
    _check_buf(B)
    ii = np.ascontiguousarray(ii, dtype=np.int64)
    jj = np.ascontiguousarray(jj, dtype=np.int64)
    C = np.empty(ii.shape[0], dtype=np.float64)
    D = np.empty(ii.shape[0], dtype=np.float64)
    rc = _load().lpy_oracle_gemm_elems_f64(M, N, K, _ptr(A), lda, la, _ptr(B), ldb, lb,
                                            ii.shape[0], _ptr(ii), _ptr(jj), _ptr(C), _ptr(D),
                                            int(nthreads))
    if rc != 0:
        raise ValueError("oracle rejected its arguments")
    return C, D


def saxpy(n, alpha, x, incx, y, incy, nthreads=0):
    """float64 values of alpha*x_i + y_i, i < n (Table 1 saxpy); x, y
    contiguous float32 buffers holding the strided vectors (only read)."""
    _check_buf(x)
    _check_buf(y)
    if n > 0 and (x.size < (n - 1) * incx + 1 or y.size < (n - 1) * incy + 1):
        raise ValueError("buffer shorter than the strided vector")
    out = np.empty(max(n, 0), dtype=np.float64)
    rc = _load().lpy_oracle_saxpy_f64(n, float(alpha), _ptr(x), incx, _ptr(y), incy, _ptr(out),
                                       int(nthreads))
    if rc != 0:
        raise ValueError("oracle rejected its arguments")
    return out


def saxpy_error_ulps(y32, ref64):
    """max |y - ref| in units of half an fp32 ulp of ref (<= 1 means y is the
    round-to-nearest of ref up to ref's own 2^-53 relative error).  Inputs are
    normal numbers or zeros (reading S1)."""
    y = np.asarray(y32, dtype=np.float64)
    ref = np.asarray(ref64, dtype=np.float64)
    if y.size == 0:
        return 0.0
    # half-ulp of the fp32 binade containing |ref|: 2^(floor(log2|ref|) - 24)
    mag = np.abs(ref)
    e = np.where(mag > 0, np.floor(np.log2(np.where(mag > 0, mag, 1.0))), -126.0)
    e = np.maximum(e, -126.0)                                    # subnormal spacing floor
    half = np.ldexp(1.0, (e - 24).astype(np.int64))          # 2^-150 at and below the subnormals
    # allow ref's own float64 rounding (<= 2^-53 |ref|)
    r = np.abs(y - ref) / (half + np.ldexp(mag, -52))
    r = np.where(np.isnan(y), np.inf, r)
    return float(r.max())


def coulomb(nt, targets, ldt, ns, sources, lds, q, nthreads=0):
    """float64 potentials phi[i] = sum_{j: r_ij != 0} q_j / r_ij and the parity
    normaliser D[i] = sum_j |q_j| / r_ij (Table 1's 3D Coulomb row).
    targets / sources: flat float32 buffers, point i at [i*ld : i*ld+3]."""
    for b in (targets, sources, q):
        _check_buf(b)
    if nt > 0 and targets.size < (nt - 1) * ldt + 3:
        raise ValueError("targets buffer too short")
    if ns > 0 and (sources.size < (ns - 1) * lds + 3 or q.size < ns):
        raise ValueError("sources / charges buffer too short")
    phi = np.empty(max(nt, 0), dtype=np.float64)
    D = np.empty(max(nt, 0), dtype=np.float64)
    rc = _load().lpy_oracle_coulomb_f64(nt, _ptr(targets), ldt, ns, _ptr(sources), lds, _ptr(q),
                                         _ptr(phi), _ptr(D), int(nthreads))
    if rc != 0:
        raise ValueError("oracle rejected its arguments")
    return phi, D


def max_threads() -> int:
    return int(_load().lpy_oracle_max_threads())


def normalized_error(C, Cref, D) -> float:
    """max_{ij} |C - Cref| / D  (north_star parity metric; reading A1:
    where D == 0, Cref is exactly 0 and C must be exactly +-0, else the error
    is reported as inf)."""
    C = np.asarray(C, dtype=np.float64)
    diff = np.abs(C - Cref)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(D > 0, diff / np.where(D > 0, D, 1.0), np.where(diff == 0, 0.0, np.inf))
    r = np.where(np.isnan(C), np.inf, r)
    return float(r.max()) if r.size else 0.0

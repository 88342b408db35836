"""paper_1405_7470_b200 -- B200-native fp32 GEMM after Loo.py (arXiv:1405.7470).

Thin Python binding over the C-ABI library ``liblpy.so`` (include/lpy.h).
Argument marshalling only: every step of the product runs in the library's
sm_100a kernels.  There is no CPU fallback -- if the library is missing or the
device is not a B200 the calls fail loudly.

Two layers:
  * ``lpy_gemm_f32``, ``lpy_gemm_f32_ex``, ``lpy_gemm_f32_host``,
    ``lpy_select_path``, ``lpy_status_string``, ``lpy_last_cuda_error``,
    ``lpy_version``: same names and arguments as the C functions (pointers as
    ints, stream as int/None), returning the raw status.
  * ``gemm(A, B, out=None, path="auto")`` on torch CUDA tensors, inferring
    M, N, K from shapes and layout/ld from strides (the paper's size inference,
    P:366-368, and stride dim_tags), raising ``LpyError``.
"""
from __future__ import annotations

import ctypes
import os
import threading

__all__ = [
    "ROW_MAJOR", "COL_MAJOR", "PATH_AUTO", "PATH_FFMA", "PATH_3XTF32", "PATHS", "LpyError",
    "GemmOpts", "library_path", "load_library", "lpy_gemm_f32", "lpy_gemm_f32_ex",
    "lpy_gemm_f32_host", "lpy_select_path", "lpy_status_string", "lpy_last_cuda_error",
    "lpy_version", "gemm", "operand_layout", "gemm_host", "lpy_saxpy_f32", "lpy_saxpy_f32_host",
    "saxpy", "saxpy_host", "lpy_coulomb_f32", "lpy_coulomb_f32_host", "coulomb", "coulomb_host",
    "KGate", "lpy_gemm_f32_gated", "lpy_kgate_signal", "kgate_signal",
]

ROW_MAJOR = 0
COL_MAJOR = 1
PATH_AUTO = 0
PATH_FFMA = 1
PATH_3XTF32 = 2
PATHS = {"auto": PATH_AUTO, "ffma": PATH_FFMA, "3xtf32": PATH_3XTF32}

_PKG = os.path.dirname(os.path.abspath(__file__))
_lock = threading.Lock()
_lib = None


def library_path() -> str:
    return os.path.join(_PKG, "liblpy.so")


class GemmOpts(ctypes.Structure):
    _fields_ = [("num_ctas", ctypes.c_int32), ("raster_group", ctypes.c_int32),
                ("promote_kblocks", ctypes.c_int32), ("tile_n", ctypes.c_int32),
                ("plan_sms", ctypes.c_int32), ("reserved", ctypes.c_int32 * 3)]


class KGate(ctypes.Structure):
    """lpy_kgate: arrival flags of a product whose operands arrive in chunks of K."""
    _fields_ = [("flags", ctypes.c_void_p), ("chunk_k", ctypes.c_int64), ("epoch", ctypes.c_uint32),
                ("timeout_ms", ctypes.c_uint32)]


class LpyError(RuntimeError):
    def __init__(self, status: int, where: str = ""):
        self.status = status
        msg = lpy_status_string(status)
        if status == 8:
            msg += f" (cudaError {lpy_last_cuda_error()})"
        super().__init__(f"{where}: {msg}" if where else msg)


def load_library():
    """Load liblpy.so (built by __graft_entry__.build()); raise if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is not built; run `python -c 'import __graft_entry__ as g; "
                               f"g.build()'` (no CPU fallback exists)")
        lib = ctypes.CDLL(path)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        gemm_args = [i64, i64, i64, vp, i64, i32, vp, i64, i32, vp, i64, i32, vp]
        lib.lpy_gemm_f32.argtypes = gemm_args
        lib.lpy_gemm_f32.restype = i32
        lib.lpy_gemm_f32_ex.argtypes = gemm_args + [i32, ctypes.POINTER(GemmOpts)]
        lib.lpy_gemm_f32_ex.restype = i32
        lib.lpy_gemm_f32_gated.argtypes = gemm_args + [i32, ctypes.POINTER(GemmOpts), ctypes.POINTER(KGate)]
        lib.lpy_gemm_f32_gated.restype = i32
        lib.lpy_kgate_signal.argtypes = [vp, ctypes.c_uint32, vp]
        lib.lpy_kgate_signal.restype = i32
        lib.lpy_gemm_f32_host.argtypes = gemm_args + [i32]
        lib.lpy_gemm_f32_host.restype = i32
        lib.lpy_select_path.argtypes = [i64, i64, i64, i32, ctypes.POINTER(i32)]
        lib.lpy_select_path.restype = i32
        lib.lpy_status_string.argtypes = [i32]
        lib.lpy_status_string.restype = ctypes.c_char_p
        lib.lpy_last_cuda_error.argtypes = []
        lib.lpy_last_cuda_error.restype = i32
        saxpy_args = [i64, ctypes.c_float, vp, i64, vp, i64, vp]
        lib.lpy_saxpy_f32.argtypes = saxpy_args
        lib.lpy_saxpy_f32.restype = i32
        lib.lpy_saxpy_f32_host.argtypes = saxpy_args
        lib.lpy_saxpy_f32_host.restype = i32
        coul_args = [i64, vp, i64, i64, vp, i64, vp, vp, vp]
        lib.lpy_coulomb_f32.argtypes = coul_args
        lib.lpy_coulomb_f32.restype = i32
        lib.lpy_coulomb_f32_host.argtypes = coul_args
        lib.lpy_coulomb_f32_host.restype = i32
        lib.lpy_version.argtypes = []
        lib.lpy_version.restype = i32
        _lib = lib
        return lib


# ----------------------------------------------------------------- C mirror
def lpy_gemm_f32(M, N, K, A, lda, layout_a, B, ldb, layout_b, C, ldc, layout_c, stream=None) -> int:
    return load_library().lpy_gemm_f32(M, N, K, A, lda, layout_a, B, ldb, layout_b, C, ldc, layout_c,
                                       stream)


def lpy_gemm_f32_ex(M, N, K, A, lda, layout_a, B, ldb, layout_b, C, ldc, layout_c, stream=None,
                    path=PATH_AUTO, opts: GemmOpts | None = None) -> int:
    return load_library().lpy_gemm_f32_ex(M, N, K, A, lda, layout_a, B, ldb, layout_b, C, ldc,
                                          layout_c, stream, path,
                                          ctypes.byref(opts) if opts is not None else None)


def lpy_gemm_f32_gated(M, N, K, A, lda, layout_a, B, ldb, layout_b, C, ldc, layout_c, stream=None,
                       path=PATH_AUTO, opts: GemmOpts | None = None, gate: KGate | None = None) -> int:
    return load_library().lpy_gemm_f32_gated(M, N, K, A, lda, layout_a, B, ldb, layout_b, C, ldc,
                                             layout_c, stream, path,
                                             ctypes.byref(opts) if opts is not None else None,
                                             ctypes.byref(gate) if gate is not None else None)


def lpy_kgate_signal(flag, value, stream=None) -> int:
    return load_library().lpy_kgate_signal(flag, value & 0xFFFFFFFF, stream)


def lpy_gemm_f32_host(M, N, K, A, lda, layout_a, B, ldb, layout_b, C, ldc, layout_c, stream=None,
                      path=PATH_AUTO) -> int:
    return load_library().lpy_gemm_f32_host(M, N, K, A, lda, layout_a, B, ldb, layout_b, C, ldc,
                                            layout_c, stream, path)


def lpy_select_path(M, N, K, requested=PATH_AUTO) -> tuple[int, int]:
    out = ctypes.c_int(0)
    st = load_library().lpy_select_path(M, N, K, requested, ctypes.byref(out))
    return st, out.value


def lpy_saxpy_f32(n, alpha, x, incx, y, incy, stream=None) -> int:
    return load_library().lpy_saxpy_f32(n, alpha, x, incx, y, incy, stream)


def lpy_saxpy_f32_host(n, alpha, x, incx, y, incy, stream=None) -> int:
    return load_library().lpy_saxpy_f32_host(n, alpha, x, incx, y, incy, stream)


def lpy_coulomb_f32(nt, t, ldt, ns, s, lds, q, phi, stream=None) -> int:
    return load_library().lpy_coulomb_f32(nt, t, ldt, ns, s, lds, q, phi, stream)


def lpy_coulomb_f32_host(nt, t, ldt, ns, s, lds, q, phi, stream=None) -> int:
    return load_library().lpy_coulomb_f32_host(nt, t, ldt, ns, s, lds, q, phi, stream)


def lpy_status_string(status: int) -> str:
    return load_library().lpy_status_string(status).decode()


def lpy_last_cuda_error() -> int:
    return load_library().lpy_last_cuda_error()


def lpy_version() -> int:
    return load_library().lpy_version()


# ----------------------------------------------------------------- torch layer
def operand_layout(x):
    """(layout, ld) of a 2-D strided tensor, or None if it is neither row- nor
    column-major (then the caller must make it contiguous)."""
    rows, cols = x.shape
    s0, s1 = x.stride()
    if (s1 == 1 or cols <= 1) and s0 >= max(1, cols):
        return ROW_MAJOR, s0
    if (s0 == 1 or rows <= 1) and s1 >= max(1, rows):
        return COL_MAJOR, s1
    if rows <= 1 and cols <= 1:
        return ROW_MAJOR, 1
    return None


def _stream_handle(stream, device_index=None):
    """cudaStream_t of `stream` (a torch.cuda.Stream or a raw handle), or of
    the current stream of `device_index` (default: the current device)."""
    import torch
    if stream is None:
        if device_index is None:
            device_index = torch.cuda.current_device()
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)   # no Stream object: ~1 us cheaper
        return raw(device_index) if raw is not None else torch.cuda.current_stream(device_index).cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _one_device(*tensors):
    """The single CUDA device all `tensors` live on (the C ABI works on the
    current device, so calls run under a guard for it); raises otherwise."""
    dev = tensors[0].device
    if dev.type != "cuda" or any(t.device != dev for t in tensors[1:]):
        raise ValueError(f"all operands must be on one CUDA device, got {sorted({str(t.device) for t in tensors})}")
    return dev


def _on_device(tensors, stream, call):
    """call(stream handle) with the tensors' device current: the guard is only
    entered when that device is not already current (it costs microseconds)."""
    import torch
    idx = _one_device(*tensors).index
    if idx is None or idx == torch.cuda.current_device():
        return call(_stream_handle(stream, idx))
    with torch.cuda.device(idx):
        return call(_stream_handle(stream, idx))


def _path_id(path) -> int:
    return PATHS[path] if isinstance(path, str) else int(path)


def gemm(A, B, out=None, path="auto", stream=None, opts: GemmOpts | None = None, gate: KGate | None = None):
    """C = A @ B for fp32 CUDA tensors through lpy_gemm_f32_ex (or, with a
    `gate`, lpy_gemm_f32_gated: operands read only as their K chunks are
    flagged ready).  `out` may be row- or column-major (any ld); it is
    overwritten."""
    import torch
    if A.dtype != torch.float32 or B.dtype != torch.float32:
        raise TypeError("lpy.gemm is fp32 in, fp32 out (PAPER.md P:362-365)")
    if A.dim() != 2 or B.dim() != 2 or A.shape[1] != B.shape[0]:
        raise ValueError(f"shape mismatch {tuple(A.shape)} @ {tuple(B.shape)}")
    if not (A.is_cuda and B.is_cuda):
        raise ValueError("device tensors required (use gemm_host for host buffers)")
    M, K = A.shape
    N = B.shape[1]
    la = operand_layout(A)
    if la is None:
        A = A.contiguous()
        la = operand_layout(A)
    lb = operand_layout(B)
    if lb is None:
        B = B.contiguous()
        lb = operand_layout(B)
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=A.device)
    if out.shape != (M, N) or out.dtype != torch.float32:
        raise ValueError("out must be an fp32 M x N tensor")
    lc = operand_layout(out)
    if lc is None:
        raise ValueError("out must be row- or column-major")
    lib = _lib or load_library()
    po = ctypes.byref(opts) if opts is not None else None
    if gate is not None:
        pg = ctypes.byref(gate)
        st = _on_device((A, B, out), stream, lambda sh: lib.lpy_gemm_f32_gated(
            M, N, K, A.data_ptr(), la[1], la[0], B.data_ptr(), lb[1], lb[0], out.data_ptr(), lc[1], lc[0], sh,
            _path_id(path), po, pg))
        if st != 0:
            raise LpyError(st, "lpy_gemm_f32_gated")
        return out
    st = _on_device((A, B, out), stream, lambda sh: lib.lpy_gemm_f32_ex(
        M, N, K, A.data_ptr(), la[1], la[0], B.data_ptr(), lb[1], lb[0], out.data_ptr(), lc[1], lc[0], sh,
        _path_id(path), po))
    if st != 0:
        raise LpyError(st, "lpy_gemm_f32_ex")
    return out


def kgate_signal(flags, index, value, stream=None):
    """flags[index] := value (uint32, release) once `stream`'s earlier work is
    done, through lpy_kgate_signal.  `flags` is a CUDA int32 tensor (the flag
    words; torch has no uint32 arithmetic, the bits are the same)."""
    import torch
    if flags.dtype != torch.int32 or not flags.is_cuda or flags.dim() != 1 or not 0 <= index < flags.shape[0]:
        raise ValueError("flags must be a 1-D int32 CUDA tensor and index within it")
    ptr = flags.data_ptr() + 4 * index
    st = _on_device((flags,), stream, lambda sh: lpy_kgate_signal(ptr, int(value), sh))
    if st != 0:
        raise LpyError(st, "lpy_kgate_signal")


def gemm_host(M, N, K, A, lda, la, B, ldb, lb, C, ldc, lc, path="auto", stream=None):
    """End-to-end product on host buffers (numpy arrays or CPU torch tensors,
    ideally pinned) through lpy_gemm_f32_host; synchronises before returning."""
    def ptr(x):
        if hasattr(x, "data_ptr"):
            return x.data_ptr()
        return x.ctypes.data
    st = lpy_gemm_f32_host(M, N, K, ptr(A), lda, la, ptr(B), ldb, lb, ptr(C), ldc, lc,
                           _stream_handle(stream) if stream is not None else None, _path_id(path))
    if st != 0:
        raise LpyError(st, "lpy_gemm_f32_host")
    return C


def _vec(v, name):
    import torch
    if v.dtype != torch.float32 or v.dim() != 1:
        raise TypeError(f"{name} must be a 1-D fp32 tensor")
    inc = v.stride(0) if v.shape[0] > 1 else 1
    if inc < 1:
        raise ValueError(f"{name} needs a positive stride")
    return inc


def saxpy(alpha, x, y, stream=None):
    """y := alpha * x + y in place on 1-D fp32 CUDA tensors (any positive
    stride) through lpy_saxpy_f32 -- Table 1's saxpy."""
    if x.shape != y.shape:
        raise ValueError("x and y must have the same length")
    if not (x.is_cuda and y.is_cuda):
        raise ValueError("device tensors required (use saxpy_host for host buffers)")
    import torch
    incx, incy = _vec(x, "x"), _vec(y, "y")
    st = _on_device((x, y), stream, lambda sh: lpy_saxpy_f32(x.shape[0], float(alpha), x.data_ptr(), incx,
                                                             y.data_ptr(), incy, sh))
    if st != 0:
        raise LpyError(st, "lpy_saxpy_f32")
    return y


def saxpy_host(alpha, x, y, stream=None):
    """End-to-end saxpy on host buffers (1-D fp32 CPU tensors, ideally pinned):
    copies in, computes, copies y back, synchronises (lpy_saxpy_f32_host)."""
    if x.shape != y.shape:
        raise ValueError("x and y must have the same length")
    incx, incy = _vec(x, "x"), _vec(y, "y")
    st = lpy_saxpy_f32_host(x.shape[0], float(alpha), x.data_ptr(), incx, y.data_ptr(), incy,
                            _stream_handle(stream) if stream is not None else None)
    if st != 0:
        raise LpyError(st, "lpy_saxpy_f32_host")
    return y


def _points(p, name, device=None):
    """Row stride (ELEMENTS) of an (n, >=3) fp32 point array with unit column
    stride, on `device` ("cuda" / "cpu") when given."""
    import torch
    if not isinstance(p, torch.Tensor) or p.dtype != torch.float32 or p.dim() != 2 or p.shape[1] < 3 or \
            (p.shape[0] >= 1 and p.stride(1) != 1):
        raise TypeError(f"{name} must be an (n, >=3) fp32 tensor with unit column stride")
    if device is not None and p.device.type != device:
        raise ValueError(f"{name} must be a {device} tensor")
    if p.shape[0] > 1 and p.stride(0) < 3:
        raise ValueError(f"{name}: rows overlap (row stride {p.stride(0)} < 3)")
    return p.stride(0) if p.shape[0] > 1 else max(3, p.shape[1])


def _vector_arg(v, name, n, device):
    """Check a contiguous (n,) fp32 tensor on `device` ("cuda" / "cpu")."""
    import torch
    if not isinstance(v, torch.Tensor) or v.dtype != torch.float32 or v.dim() != 1 or v.shape[0] != n or \
            (n > 1 and v.stride(0) != 1):
        raise TypeError(f"{name} must be a contiguous ({n},) fp32 tensor")
    if v.device.type != device:
        raise ValueError(f"{name} must be a {device} tensor")


def coulomb(targets, sources, charges, out=None, stream=None):
    """phi[i] = sum_{j: r_ij != 0} q_j / r_ij on CUDA tensors through
    lpy_coulomb_f32 (Table 1's 3D Coulomb potential).
    targets (nt, >=3), sources (ns, >=3): x, y, z in the first three columns;
    charges (ns,) contiguous; returns phi (nt,)."""
    import torch
    ldt, lds = _points(targets, "targets", "cuda"), _points(sources, "sources", "cuda")
    _vector_arg(charges, "charges", sources.shape[0], "cuda")
    nt = targets.shape[0]
    if out is None:
        out = torch.empty(nt, dtype=torch.float32, device=targets.device)
    _vector_arg(out, "out", nt, "cuda")
    st = _on_device((targets, sources, charges, out), stream, lambda sh: lpy_coulomb_f32(
        nt, targets.data_ptr(), ldt, sources.shape[0], sources.data_ptr(), lds, charges.data_ptr(),
        out.data_ptr(), sh))
    if st != 0:
        raise LpyError(st, "lpy_coulomb_f32")
    return out


def coulomb_host(targets, sources, charges, out, stream=None):
    """End-to-end Coulomb on host (CPU, ideally pinned) tensors; synchronises."""
    ldt, lds = _points(targets, "targets", "cpu"), _points(sources, "sources", "cpu")
    _vector_arg(charges, "charges", sources.shape[0], "cpu")
    _vector_arg(out, "out", targets.shape[0], "cpu")
    st = lpy_coulomb_f32_host(targets.shape[0], targets.data_ptr(), ldt, sources.shape[0], sources.data_ptr(),
                              lds, charges.data_ptr(), out.data_ptr(),
                              _stream_handle(stream) if stream is not None else None)
    if st != 0:
        raise LpyError(st, "lpy_coulomb_f32_host")
    return out

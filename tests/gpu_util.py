"""Helpers for the GPU parity tests: lay synthetic inputs out in any layout /
leading dimension, run the product through the C-ABI (lpy_gemm_f32_ex), and
compare against the float64 oracle on the same input bits."""
import numpy as np
import torch

import oracle
import paper_1405_7470_b200 as lpy
import synth

SENTINEL = np.float32(-31337.0)
TOL = 1e-5          # north_star: max |C - Cref| / sum_k |A_ik||B_kj| <= 1e-5


def device_buffer(host: np.ndarray, pad_floats: int = 0) -> torch.Tensor:
    """A device copy of a flat fp32 buffer, optionally offset by `pad_floats`
    elements (to make the base pointer deliberately not 16-byte aligned)."""
    t = torch.empty(host.size + pad_floats + 4, dtype=torch.float32, device="cuda")
    t[pad_floats:pad_floats + host.size].copy_(torch.from_numpy(host))
    return t[pad_floats:pad_floats + host.size]


def run_gemm(A, B, la=0, lb=0, lc=0, lda=None, ldb=None, ldc=None, path="ffma", opts=None,
             base_offset=0):
    """C = A*B via lpy_gemm_f32_ex with the given layouts/lds; returns
    (logical C as np.float32, whether C's padding survived untouched)."""
    M, K = A.shape
    N = B.shape[1]
    abuf, lda = synth.store(A, la, lda)
    bbuf, ldb = synth.store(B, lb, ldb)
    cbuf, ldc = synth.store(np.zeros((M, N), np.float32), lc, ldc, pad_value=np.nan)
    cbuf[:] = SENTINEL            # every element, padding included, starts as the sentinel
    dA = device_buffer(abuf, base_offset)
    dB = device_buffer(bbuf, base_offset)
    dC = device_buffer(cbuf, base_offset)
    st = lpy.lpy_gemm_f32_ex(M, N, K, dA.data_ptr() if abuf.size else 0, lda, la,
                             dB.data_ptr() if bbuf.size else 0, ldb, lb,
                             dC.data_ptr() if cbuf.size else 0, ldc, lc,
                             torch.cuda.current_stream().cuda_stream, lpy.PATHS[path], opts)
    if st != 0:
        raise lpy.LpyError(st, "lpy_gemm_f32_ex")
    torch.cuda.synchronize()
    out = dC.cpu().numpy()
    C = synth.load_logical(out, M, N, lc, ldc)
    mask = np.ones(out.size, dtype=bool)
    if M and N:
        if lc == synth.ROW_MAJOR:
            idx = np.arange(M)[:, None] * ldc + np.arange(N)[None, :]
        else:
            idx = np.arange(M)[:, None] + np.arange(N)[None, :] * ldc
        mask[idx.reshape(-1)] = False
    pad_ok = bool(np.all(out[mask] == SENTINEL))
    return C, pad_ok


def oracle_ref(A, B):
    M, K = A.shape
    N = B.shape[1]
    return oracle.gemm(M, N, K, np.ascontiguousarray(A).reshape(-1), max(1, K), 0,
                       np.ascontiguousarray(B).reshape(-1), max(1, N), 0)


def check(C, A, B, exact=False, tol=TOL):
    Cref, D = oracle_ref(A, B)
    if exact:
        assert np.array_equal(C.astype(np.float64), Cref), "integer-valued product not exact"
        return 0.0
    err = oracle.normalized_error(C, Cref, D)
    assert err <= tol, f"normalized error {err:.3e} > {tol}"
    return err

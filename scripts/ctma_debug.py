#!/usr/bin/env python
"""(Rejected TMA-store epilogue, profiles/r02_tf32_tma_store_rejected.txt.) Which shapes / lds make a
TMA-store epilogue write outside the logical C?
(Found: a bulk tensor store clips a row at 16-byte granularity, so it is used only for N % 4 == 0.)
Runs tests/test_parity_gpu.py::test_tiny_and_edge_shapes_all_layouts's row-major cases and prints
where the sentinel was overwritten."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import synth
import paper_1405_7470_b200 as lpy
from gpu_util import SENTINEL, device_buffer

EDGE = [1, 2, 3, 7, 8, 9, 15, 16, 17, 31, 32, 33, 127, 128, 129, 255, 256, 257]
rng = np.random.default_rng(0)
shapes = [(1, 1, 1), (3, 5, 7), (129, 257, 33), (128, 128, 32)] + [tuple(int(x) for x in rng.choice(EDGE, 3)) for _ in range(8)]
bad = 0
for (M, N, K) in shapes:
    for pad in (0, 3, 4):
        A = synth.matrix(M, K, seed=1, matrix_id=synth.MATRIX_A)
        B = synth.matrix(K, N, seed=1, matrix_id=synth.MATRIX_B)
        abuf, lda = synth.store(A, 0, synth.min_ld(M, K, 0) + pad)
        bbuf, ldb = synth.store(B, 0, synth.min_ld(K, N, 0) + pad)
        cbuf, ldc = synth.store(np.zeros((M, N), np.float32), 0, synth.min_ld(M, N, 0) + pad, pad_value=np.nan)
        cbuf[:] = SENTINEL
        dA, dB, dC = device_buffer(abuf), device_buffer(bbuf), device_buffer(cbuf)
        st = lpy.lpy_gemm_f32_ex(M, N, K, dA.data_ptr(), lda, 0, dB.data_ptr(), ldb, 0, dC.data_ptr(), ldc, 0,
                                 torch.cuda.current_stream().cuda_stream, lpy.PATHS["3xtf32"], None)
        torch.cuda.synchronize()
        out = dC.cpu().numpy()
        rows, cols = np.divmod(np.arange(out.size), ldc)
        outside = (cols >= N) | (rows >= M)
        hit = np.nonzero(outside & (out != SENTINEL))[0]
        if hit.size:
            bad += 1
            r, c = rows[hit], cols[hit]
            print(f"M={M} N={N} K={K} ldc={ldc} buf={out.size} ptr%128={dC.data_ptr() % 128}: {hit.size} outside writes, "
                  f"rows {r.min()}..{r.max()} cols {c.min()}..{c.max()} first vals {out[hit[:4]]}", flush=True)
print("bad", bad)

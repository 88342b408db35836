#!/usr/bin/env python
"""Repeatability stress for split-K products: the same product many times at
several grids, counting results that differ from the first (diagnostics)."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402
import synth  # noqa: E402
from gpu_util import run_gemm  # noqa: E402

path = sys.argv[1] if len(sys.argv) > 1 else "ffma"
M, N, K = (int(x) for x in (sys.argv[2:5] if len(sys.argv) > 4 else (2560, 2304, 1024)))
tile_n = int(sys.argv[5]) if len(sys.argv) > 5 else 0
if len(sys.argv) > 6:                      # alternative library build
    lpy.library_path = (lambda p: (lambda: p))(os.path.abspath(sys.argv[6]))
A = synth.matrix(M, K, seed=21, matrix_id=0)
B = synth.matrix(K, N, seed=21, matrix_id=1)
ref = None
bad = {}
for it in range(12):
    for ctas in (0, 148, 74, 32):
        o = lpy.GemmOpts()
        o.num_ctas = ctas
        o.tile_n = tile_n
        C, _ = run_gemm(A, B, path=path, opts=o)
        if ref is None:
            ref = C
            continue
        d = C != ref
        if d.any():
            idx = np.argwhere(d)
            rel = float(np.max(np.abs(C[d].astype(np.float64) - ref[d]) / (np.abs(ref[d]) + 1e-30)))
            bad.setdefault(ctas, []).append((it, int(d.sum()), f"maxrel {rel:.2e}",
                                             sorted(set((idx[:, 0] % 128).tolist()))[:8],
                                             sorted(set((idx[:, 1] % 256).tolist()))[:8]))
print(path, M, N, K, "tile_n", tile_n, "mismatching runs:", {k: len(v) for k, v in bad.items()})
for k, v in bad.items():
    print(k, v[:4])

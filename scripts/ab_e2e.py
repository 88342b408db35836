#!/usr/bin/env python
"""Interleaved A/B of library builds on the end-to-end host entry
(lpy_gemm_f32_host, pinned host buffers, n = 8192): ms per product."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

n, libs = int(sys.argv[1]), sys.argv[2:]
A = torch.randn(n, n).pin_memory()
B = torch.randn(n, n).pin_memory()
C = torch.empty(n, n).pin_memory()
res = {}
for rnd in range(3):
    for lib in libs:
        lpy._lib = None
        lpy.library_path = (lambda p: (lambda: p))(os.path.abspath(lib))
        lpy.load_library()
        lpy.gemm_host(n, n, n, A, n, 0, B, n, 0, C, n, 0, path="3xtf32")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            lpy.gemm_host(n, n, n, A, n, 0, B, n, 0, C, n, 0, path="3xtf32")
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(lib, []).append(e0.elapsed_time(e1) / 5)
for lib, v in res.items():
    print(f"{os.path.basename(lib):20s} n={n}: median {statistics.median(v):7.3f} ms  ({', '.join(f'{x:.2f}' for x in v)})")

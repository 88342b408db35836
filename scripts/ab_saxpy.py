#!/usr/bin/env python
"""Interleaved A/B of library builds on saxpy (n = 2^28): GB/s per build."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

n = int(sys.argv[1])
libs = sys.argv[2:]
x = torch.rand(n, device="cuda")
y = torch.rand(n, device="cuda")
res = {}
for rnd in range(3):
    for lib in libs:
        lpy._lib = None
        lpy.library_path = (lambda p: (lambda: p))(os.path.abspath(lib))
        lpy.load_library()
        for _ in range(3):
            lpy.saxpy(1e-3, x, y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            lpy.saxpy(1e-3, x, y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        res.setdefault(lib, []).append(12.0 * n / ms / 1e6)
for lib, v in res.items():
    print(f"{os.path.basename(lib):26s} n={n}: median {statistics.median(v):8.1f} GB/s  ({', '.join(f'{a:.0f}' for a in v)})")

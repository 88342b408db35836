#!/usr/bin/env python
"""A/B timing of library builds: for each .so given, time C = A*B at n on a
path (row-major, device-resident inputs, CUDA events, median of rounds) and
check a sample of the result against the default library's.

usage: python scripts/ab_lib.py <path> <n> lib1.so [lib2.so ...]
env LA / LB = row|col pick the A / B layouts (default row).
"""
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

path, n, libs = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
A = torch.randn(n, n, device="cuda")
B = torch.randn(n, n, device="cuda")
if os.environ.get("LA", "row") == "col":
    A = A.t().contiguous().t()
if os.environ.get("LB", "row") == "col":
    B = B.t().contiguous().t()
results = {}
for rnd in range(int(os.environ.get("ROUNDS", "3"))):
    for lib in libs:
        lpy._lib = None
        lpy.library_path = (lambda p: (lambda: p))(os.path.abspath(lib))
        lpy.load_library()
        C = torch.empty(n, n, device="cuda")
        for _ in range(3):
            lpy.gemm(A, B, out=C, path=path)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            lpy.gemm(A, B, out=C, path=path)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        results.setdefault(lib, []).append(2 * n ** 3 / ms / 1e9)
        if rnd == 0:
            ref = (A[:64].double() @ B.double())
            err = ((C[:64].double() - ref).abs() / (A[:64].abs().double() @ B.abs().double())).max().item()
            print(f"{os.path.basename(lib)}: sample normalised error {err:.2e}")
for lib, v in results.items():
    print(f"{os.path.basename(lib):28s} {path} n={n}: median {statistics.median(v):8.1f} TFLOP/s  ({', '.join(f'{x:.1f}' for x in v)})")

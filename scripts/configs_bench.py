#!/usr/bin/env python
"""Time every BASELINE.json config on both paths (device-resident inputs,
CUDA events, L2 flushed between iterations for the small configs whose
working set fits in L2) and print a table: the per-config numbers behind
DESIGN.md's results section.  The headline bench line stays bench.py's."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

CONFIGS = [
    ("cfg1 n=128 row-major", 128, 128, 128, 0, 0, 0),
    ("cfg2 n=1024 A row B row", 1024, 1024, 1024, 0, 0, 0),
    ("cfg2 n=1024 A row B col", 1024, 1024, 1024, 0, 1, 0),
    ("cfg2 n=1024 A col B row", 1024, 1024, 1024, 1, 0, 0),
    ("cfg2 n=1024 A col B col", 1024, 1024, 1024, 1, 1, 0),
    ("cfg3 n=4096 row-major", 4096, 4096, 4096, 0, 0, 0),
    ("cfg4 n=8192 row-major", 8192, 8192, 8192, 0, 0, 0),
    ("cfg5 1000x3000x777 B col, ld=777 (repack)", 1000, 3000, 777, 0, 1, 777),
    ("cfg5 1000x3000x777 B col, ld=780", 1000, 3000, 777, 0, 1, 780),
]
flush = torch.empty(256 * 2 ** 20 // 4, device="cuda")   # 256 MB > L2


def operand(rows, cols, layout, ld):
    if layout == 0:
        ld = ld or cols
        return torch.randn(rows, ld, device="cuda")[:, :cols]
    ld = ld or rows
    return torch.randn(cols, ld, device="cuda")[:, :rows].t()


print(f"{'config':44s} {'path':7s} {'ms':>9s} {'TFLOP/s':>9s}")
for name, M, N, K, la, lb, ld in CONFIGS:
    A = operand(M, K, la, ld if la == 0 else 0)
    B = operand(K, N, lb, ld if lb == 1 else 0)
    C = torch.empty(M, N, device="cuda")
    small = 4 * (M * K + K * N + M * N) < 64 * 2 ** 20
    for path in ("ffma", "3xtf32"):
        for _ in range(3):
            lpy.gemm(A, B, out=C, path=path)
        reps = 20 if M * N * K < 2 ** 33 else 5
        tot = 0.0
        for _ in range(reps):
            if small:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lpy.gemm(A, B, out=C, path=path)
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        ms = tot / reps
        print(f"{name:44s} {path:7s} {ms:9.4f} {2 * M * N * K / ms / 1e9:9.2f}", flush=True)

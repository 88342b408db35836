#!/usr/bin/env python
"""Time both paths at n (default 8192) for all four A/B layout combinations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = torch.randn(n, n, device="cuda")
B = torch.randn(n, n, device="cuda")
for path in ("3xtf32", "ffma"):
    for la in ("row", "col"):
        for lb in ("row", "col"):
            a = A if la == "row" else A.t().contiguous().t()
            b = B if lb == "row" else B.t().contiguous().t()
            C = torch.empty(n, n, device="cuda")
            for _ in range(3):
                lpy.gemm(a, b, out=C, path=path)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                lpy.gemm(a, b, out=C, path=path)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            print(f"{path:7s} A {la} B {lb}: {ms:.3f} ms  {2 * n ** 3 / ms / 1e9:.1f} TFLOP/s")

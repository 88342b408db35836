#!/usr/bin/env python
"""Run C = A*B a few times for one (path, n, A layout, B layout) -- a target
for ncu captures of a single kernel variant.
usage: python scripts/one_gemm.py <path> <n> <la row|col> <lb row|col> [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

path, n, la, lb = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 4
A = torch.randn(n, n, device="cuda")
B = torch.randn(n, n, device="cuda")
a = A if la == "row" else A.t().contiguous().t()
b = B if lb == "row" else B.t().contiguous().t()
C = torch.empty(n, n, device="cuda")
for _ in range(reps):
    lpy.gemm(a, b, out=C, path=path)
torch.cuda.synchronize()
print("ok")

#!/usr/bin/env python
"""Run C = A*B a few times for one (path, M, N, K, A layout, B layout, ld pad):
a target for ncu captures of one configuration (e.g. BASELINE config 5:
1000 3000 777 row col 0).
usage: python scripts/cfg_gemm.py <path> M N K <row|col> <row|col> [ld_pad] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

path = sys.argv[1]
M, N, K = (int(x) for x in sys.argv[2:5])
la, lb = sys.argv[5], sys.argv[6]
pad = int(sys.argv[7]) if len(sys.argv) > 7 else 0
reps = int(sys.argv[8]) if len(sys.argv) > 8 else 4


def operand(rows, cols, layout):
    if layout == "row":
        return torch.randn(rows, cols + pad, device="cuda")[:, :cols]
    return torch.randn(cols, rows + pad, device="cuda")[:, :rows].t()


a, b = operand(M, K, la), operand(K, N, lb)
C = torch.empty(M, N, device="cuda")
for _ in range(reps):
    lpy.gemm(a, b, out=C, path=path)
torch.cuda.synchronize()
print("ok")

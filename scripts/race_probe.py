#!/usr/bin/env python
"""Diagnose split-K FFMA nondeterminism: repeat one product, compare each run
with an fp64 reference, histogram where the wrong elements sit in the tile."""
import os
import sys
from collections import Counter

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

M, N, K, tn = (int(x) for x in sys.argv[1:5])
if len(sys.argv) > 5:                      # alternative library build
    lpy.library_path = (lambda p: (lambda: p))(os.path.abspath(sys.argv[5]))
torch.manual_seed(0)
A = torch.randn(M, K, device="cuda")
B = torch.randn(K, N, device="cuda")
ref = (A.double() @ B.double())
D = (A.abs().double() @ B.abs().double())
cols, rows, wrong_runs = Counter(), Counter(), 0
for it in range(8):
    o = lpy.GemmOpts(); o.tile_n = tn
    C = lpy.gemm(A, B, path="ffma", opts=o)
    err = ((C.double() - ref).abs() / D)
    bad = torch.nonzero(err > 1e-5).cpu().numpy()
    if len(bad):
        wrong_runs += 1
        cols.update((bad[:, 1] % tn).tolist())
        rows.update((bad[:, 0] % 128).tolist())
print(f"{M}x{N}x{K} tile_n={tn}: {wrong_runs}/8 runs with errors > 1e-5")
print("cols:", sorted(cols.keys()))
print("rows:", sorted(rows.keys()))

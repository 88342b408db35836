#!/usr/bin/env python
"""C = A*B (row-major, uniform[-1,1)) a few times through a given library build -- an ncu target
for A/B builds.  usage: python scripts/lib_gemm.py <lib.so> <path> M N K [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1405_7470_b200 as lpy
lib, path = sys.argv[1], sys.argv[2]
M, N, K = (int(x) for x in sys.argv[3:6])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
lpy.library_path = lambda: os.path.abspath(lib)
a = torch.rand(M, K, device="cuda") * 2 - 1
b = torch.rand(K, N, device="cuda") * 2 - 1
C = torch.empty(M, N, device="cuda")
for _ in range(reps):
    lpy.gemm(a, b, out=C, path=path)
torch.cuda.synchronize()

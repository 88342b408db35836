#!/usr/bin/env python
"""Race detector over a library build (tests/test_mutation_gpu.py's DETECTOR,
more repetitions): python scripts/race_lib.py <lib.so|product> <path> <reps> "M,N,K;..." """
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1405_7470_b200 as lpy
lib, path, reps, shapes = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
if lib != "product":
    lpy.library_path = lambda: os.path.abspath(lib)
bad = 0
for spec in shapes.split(";"):
    M, N, K = (int(x) for x in spec.split(","))
    for la in ("row", "col"):
        for lb in ("row", "col"):
            g = torch.Generator(device="cuda")
            g.manual_seed(M + K)
            A = torch.rand(M, K, device="cuda", generator=g) * 2 - 1
            B = torch.rand(K, N, device="cuda", generator=g) * 2 - 1
            if la == "col":
                A = A.t().contiguous().t()
            if lb == "col":
                B = B.t().contiguous().t()
            ref = A.double() @ B.double()
            D = A.abs().double() @ B.abs().double()
            first, worst, same = None, 0.0, True
            for _ in range(reps):
                C = lpy.gemm(A, B, path=path)
                worst = max(worst, ((C.double() - ref).abs() / D).max().item())
                if first is None:
                    first = C.clone()
                else:
                    same = same and torch.equal(C, first)
            ok = worst <= 1e-5 and same
            bad += not ok
            print(f"{spec} {la}/{lb}: {'PASS' if ok else 'FAIL'} max_err={worst:.3e} repeatable={same}", flush=True)
print("RACE", "FAIL" if bad else "PASS")

#!/usr/bin/env python
"""Device time per product for a list of shapes on one path (row-major,
device-resident inputs, 3 warm-up calls, CUDA events around `reps`
back-to-back calls, median of 3 rounds).  Environment switches of the library
(e.g. LPY_TF32_STREAMK=0) apply, so A/B runs are two invocations.

usage: [PLAN_SMS=n] python scripts/shapes_time.py <path> M,N,K [M,N,K ...]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

path = sys.argv[1]
tag = os.environ.get("TAG", "")
opts = None
if os.environ.get("PLAN_SMS"):          # plan for fewer SMs (the row-panel product beside its broadcast)
    opts = lpy.GemmOpts()
    opts.plan_sms = int(os.environ["PLAN_SMS"])
for spec in sys.argv[2:]:
    M, N, K = (int(x) for x in spec.split(","))
    A = torch.rand(M, K, device="cuda") * 2 - 1
    B = torch.rand(K, N, device="cuda") * 2 - 1
    C = torch.empty(M, N, device="cuda")
    reps = max(3, min(50, int(2e12 / (2.0 * M * N * K) * 10)))
    for _ in range(3):
        lpy.gemm(A, B, out=C, path=path, opts=opts)
    torch.cuda.synchronize()
    res = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            lpy.gemm(A, B, out=C, path=path, opts=opts)
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / reps)
    ms = statistics.median(res)
    ref = A[:32].double() @ B.double()
    err = ((C[:32].double() - ref).abs() / (A[:32].abs().double() @ B.abs().double())).max().item()
    print(f"{tag:10s} {path} {M}x{N}x{K}: {ms:.4f} ms  {2.0 * M * N * K / ms / 1e9:.1f} TFLOP/s  "
          f"(rounds {', '.join(f'{x:.4f}' for x in res)}; err {err:.1e})", flush=True)

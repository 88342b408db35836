#!/usr/bin/env python
"""FFMA tile width A/B on the under-filled configs: opts.tile_n 0 (auto) / 128 /
256, CUDA-graph replay of 20 calls, median of 5 interleaved rounds."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1405_7470_b200 as lpy

CASES = [("cfg2 n1024 rr", 1024, 1024, 1024, "row", "row"), ("cfg2 n1024 cc", 1024, 1024, 1024, "col", "col"),
         ("cfg5", 1000, 3000, 780, "row", "col"), ("n2048", 2048, 2048, 2048, "row", "row")]
graphs = {}
for name, M, N, K, la, lb in CASES:
    a = torch.rand(M, K, device="cuda") * 2 - 1 if la == "row" else (torch.rand(K, M, device="cuda") * 2 - 1).t()
    b = torch.rand(K, N, device="cuda") * 2 - 1 if lb == "row" else (torch.rand(N, K, device="cuda") * 2 - 1).t()
    C = torch.empty(M, N, device="cuda")
    for tn in (0, 128, 256):
        o = lpy.GemmOpts()
        o.tile_n = tn
        for _ in range(3):
            lpy.gemm(a, b, out=C, path="ffma", opts=o)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                lpy.gemm(a, b, out=C, path="ffma", opts=o)
        graphs[(name, tn)] = (g, 2.0 * M * N * K, (a, b, C))   # keep the captured tensors alive
res = {}
for _ in range(5):
    for key, (g, fl, _) in graphs.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(key, []).append(e0.elapsed_time(e1) / 20 * 1e3)
for key, (g, fl, _) in graphs.items():
    us = statistics.median(res[key])
    print(f"{key[0]:16s} tile_n={key[1]:3d}: {us:8.2f} us {fl / us / 1e6:6.2f} TFLOP/s")

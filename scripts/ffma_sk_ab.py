#!/usr/bin/env python
"""FFMA stream-K A/B on the under-filled configs: device time per call from
CUDA-graph replay of 20 calls (launch gaps excluded), median of 5, plus a parity
check against float64 torch on sampled rows.  Run once per LPY_FFMA_STREAMK
setting (0 = split-K / cluster split, 2 = stream-K forced, 1 = auto).
usage: TAG=x python scripts/ffma_sk_ab.py"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1405_7470_b200 as lpy

tag = os.environ.get("TAG", os.environ.get("LPY_FFMA_STREAMK", "1"))
PATH = os.environ.get("LPY_PATH", "ffma")
CASES = [("cfg2 n1024 rr", 1024, 1024, 1024, "row", "row", 0), ("cfg2 n1024 rc", 1024, 1024, 1024, "row", "col", 0),
         ("cfg2 n1024 cr", 1024, 1024, 1024, "col", "row", 0), ("cfg2 n1024 cc", 1024, 1024, 1024, "col", "col", 0),
         ("cfg5 ld777", 1000, 3000, 777, "row", "col", 0), ("cfg5 ld780", 1000, 3000, 777, "row", "col", 3),
         ("n2048", 2048, 2048, 2048, "row", "row", 0), ("n4096", 4096, 4096, 4096, "row", "row", 0),
         ("2048x2048x8192", 2048, 2048, 8192, "row", "row", 0)]


def operand(rows, cols, layout, pad):
    if layout == "row":
        return torch.rand(rows, cols + pad, device="cuda")[:, :cols] * 2 - 1
    return (torch.rand(cols, rows + pad, device="cuda")[:, :rows] * 2 - 1).t()


for name, M, N, K, la, lb, pad in CASES:
    a, b = operand(M, K, la, pad), operand(K, N, lb, pad)
    C = torch.empty(M, N, device="cuda")
    for _ in range(3):
        lpy.gemm(a, b, out=C, path=PATH)
    torch.cuda.synchronize()
    ref = a[:64].double() @ b.double()
    err = ((C[:64].double() - ref).abs() / (a[:64].abs().double() @ b.abs().double())).max().item()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            lpy.gemm(a, b, out=C, path=PATH)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 20 * 1e3)
    us = statistics.median(ts)
    print(f"{tag:6s} {name:18s} {us:9.2f} us  {2.0 * M * N * K / us / 1e6:7.2f} TFLOP/s  err {err:.1e}", flush=True)

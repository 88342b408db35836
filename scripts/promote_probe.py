#!/usr/bin/env python
"""Does the TMEM partial drain (promotion every `promote` k-blocks) slow the narrow 3xTF32 tiles?
CUDA-graph replay of products at promote_kblocks 4 / 8 / 16, interleaved rounds."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1405_7470_b200 as lpy
shapes = [(1024, 1024, 1024), (1000, 3000, 780), (2048, 1024, 2048), (8192, 8192, 8192)]
res = {}
graphs = {}
for (M, N, K) in shapes:
    a = torch.rand(M, K, device="cuda") * 2 - 1
    b = torch.rand(K, N, device="cuda") * 2 - 1
    c = torch.empty(M, N, device="cuda")
    reps = 20 if M * N * K < 2e10 else 2
    for pr in (4, 8, 16):
        o = lpy.GemmOpts()
        o.promote_kblocks = pr
        for _ in range(2):
            lpy.gemm(a, b, out=c, path="3xtf32", opts=o)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                lpy.gemm(a, b, out=c, path="3xtf32", opts=o)
        graphs[(M, N, K, pr)] = (g, reps, (a, b, c))
for rnd in range(5):
    for key, (g, reps, _) in graphs.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        res.setdefault(key, []).append(e0.elapsed_time(e1) / reps * 1e3)
for key, v in res.items():
    print(f"{key[0]}x{key[1]}x{key[2]} promote={key[3]:2d}: {statistics.median(v):9.2f} us", flush=True)

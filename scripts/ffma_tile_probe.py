#!/usr/bin/env python
"""Tile width on the under-filled / mid-size configs: opts.tile_n 128 vs 256 (and 192 on the 3xTF32
path: PATH=3xtf32) vs the launcher's choice (0), CUDA-graph replay, interleaved rounds; sampled parity
against float64.  CASES=wide: the mid-size shape list."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1405_7470_b200 as lpy
cases = [(1024, 1024, 1024, "row", "row"), (1024, 1024, 1024, "col", "row"), (1000, 3000, 780, "row", "col"),
         (1000, 3000, 780, "col", "row"), (2048, 2048, 2048, "row", "row"), (512, 512, 512, "row", "row"),
         (1000, 3000, 777, "row", "col")]
if os.environ.get("CASES") == "wide":
    cases = [(2048, 2048, 8192, "row", "row"), (4096, 4096, 1024, "row", "row"), (4096, 4096, 4096, "row", "row"),
             (3000, 5000, 1000, "row", "row"), (1024, 8192, 8192, "row", "row"), (2048, 4096, 2048, "row", "row"),
             (1536, 2048, 2048, "row", "row")]
PATH = os.environ.get("PATH_", "ffma")
WIDTHS = (0, 128, 256) if PATH == "ffma" else (0, 128, 192, 256)
graphs = {}
for (M, N, K, la, lb) in cases:
    a = torch.rand(M, K, device="cuda") * 2 - 1 if la == "row" else (torch.rand(K, M, device="cuda") * 2 - 1).t()
    b = torch.rand(K, N, device="cuda") * 2 - 1 if lb == "row" else (torch.rand(N, K, device="cuda") * 2 - 1).t()
    c = torch.empty(M, N, device="cuda")
    ref = a[:16].double() @ b.double()
    D = a[:16].abs().double() @ b.abs().double()
    for tn in WIDTHS:
        o = lpy.GemmOpts()
        o.tile_n = tn
        for _ in range(2):
            lpy.gemm(a, b, out=c, path=PATH, opts=o)
        torch.cuda.synchronize()
        err = ((c[:16].double() - ref).abs() / D).max().item()
        reps = 20 if M * N * K < 1e10 else 4
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                lpy.gemm(a, b, out=c, path=PATH, opts=o)
        graphs[(M, N, K, la, lb, tn)] = (g, err, (a, b, c), reps)
res = {}
for rnd in range(5):
    for key, (g, err, _, reps) in graphs.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        res.setdefault(key, []).append(e0.elapsed_time(e1) / reps * 1e3)
for key, v in res.items():
    print(f"{key[0]}x{key[1]}x{key[2]} {key[3]}/{key[4]} tile_n={key[5]:3d}: {statistics.median(v):8.2f} us  err {graphs[key][1]:.1e}", flush=True)

#!/usr/bin/env python
"""Small BASELINE configs (1, 2, 5): where does a call's time go?

For each config and path:
  eager_us  - events around one lpy.gemm call after an L2 flush (what
              scripts/configs_bench.py reports: includes the host's enqueue
              latency, since the GPU idles until the launch arrives)
  host_us   - host cost of one lpy.gemm call (Python binding + C front end +
              launch), from perf_counter over 400 calls with no sync
  graph_us  - device time per call from a CUDA graph of 50 captured calls
              replayed back to back (no host in the loop; inputs L2-warm)
and checks that the graph's result is bitwise equal to the eager one."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

CONFIGS = [
    ("cfg1 n=128", 128, 128, 128, 0, 0, 0),
    ("cfg2 n=1024 A row B row", 1024, 1024, 1024, 0, 0, 0),
    ("cfg2 n=1024 A row B col", 1024, 1024, 1024, 0, 1, 0),
    ("cfg2 n=1024 A col B row", 1024, 1024, 1024, 1, 0, 0),
    ("cfg2 n=1024 A col B col", 1024, 1024, 1024, 1, 1, 0),
    ("cfg5 1000x3000x777 ld=777 (repack)", 1000, 3000, 777, 0, 1, 777),
    ("cfg5 1000x3000x777 ld=780", 1000, 3000, 777, 0, 1, 780),
    ("n=512", 512, 512, 512, 0, 0, 0),
    ("n=2048", 2048, 2048, 2048, 0, 0, 0),
    ("2048x2048x8192", 2048, 2048, 8192, 0, 0, 0),
]
paths = sys.argv[1].split(",") if len(sys.argv) > 1 else ["ffma", "3xtf32"]
if os.environ.get("SHAPES"):   # comma-separated substrings of config names to keep
    keep = os.environ["SHAPES"].split(",")
    CONFIGS = [c for c in CONFIGS if any(k in c[0] for k in keep)]
flush = torch.empty(256 * 2 ** 20 // 4, device="cuda")


def operand(rows, cols, layout, ld):
    if layout == 0:
        ld = ld or cols
        return torch.randn(rows, ld, device="cuda")[:, :cols]
    ld = ld or rows
    return torch.randn(cols, ld, device="cuda")[:, :rows].t()


print(f"{'config':36s} {'path':7s} {'eager_us':>9s} {'host_us':>8s} {'graph_us':>9s} {'TFLOP/s(graph)':>15s} bitwise")
for name, M, N, K, la, lb, ld in CONFIGS:
    torch.manual_seed(0)
    A = operand(M, K, la, ld if la == 0 else 0)
    B = operand(K, N, lb, ld if lb == 1 else 0)
    C = torch.empty(M, N, device="cuda")
    for path in paths:
        f = lambda: lpy.gemm(A, B, out=C, path=path)
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        ref = C.clone()
        tot = 0.0
        for _ in range(30):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        eager = 1e3 * tot / 30
        # host enqueue cost (the queue absorbs 400 small launches)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(400):
            f()
        host = 1e6 * (time.perf_counter() - t0) / 400
        torch.cuda.synchronize()
        # graph of 50 calls
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            C.zero_()
            with torch.cuda.graph(g, stream=s):
                for _ in range(50):
                    f()
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
        torch.cuda.synchronize()
        same = bool(torch.equal(C, ref))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        gus = 1e3 * e0.elapsed_time(e1) / 200
        print(f"{name:36s} {path:7s} {eager:9.2f} {host:8.2f} {gus:9.2f} {2 * M * N * K / gus / 1e6:15.2f} {same}",
              flush=True)
        del g

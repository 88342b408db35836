#!/usr/bin/env python
"""GEMM side of the multi-GPU step on one GPU: rank 0's row panel of an
n x n x n product split over G ranks (rows = n/G), B in `chunks` column blocks,
block products on S streams with grids sized to their tiles (dist.chunk_grid)
-- vs the same panel as one product.  No broadcast (1 GPU); this isolates what
chunking costs the products.  usage: panel_probe.py [n] [G] [path]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402
from paper_1405_7470_b200.dist import chunk_bounds, chunk_grid, chunk_tile_n, rowpanel_gemm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
path = sys.argv[3] if len(sys.argv) > 3 else "3xtf32"
rows = n // G
sms = torch.cuda.get_device_properties(0).multi_processor_count
A = torch.randn(rows, n, device="cuda")
Bfull = torch.randn(n, n, device="cuda")
C = torch.empty(rows, n, device="cuda")


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


flops = 2.0 * rows * n * n
ms = timeit(lambda: lpy.gemm(A, Bfull, out=C, path=path))
print(f"n={n} G={G} rows={rows} {path}: one product {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s")
for chunks in (2, 4, 8):
    bounds = chunk_bounds(n, chunks)
    blocks = [Bfull[:, c0:c1].contiguous() for c0, c1 in bounds]
    for nstreams in (1, 2, 4, 8):
        if nstreams > chunks:
            continue
        streams = [torch.cuda.Stream() for _ in range(nstreams)]

        def gemm_fn(a, b, c):
            o = lpy.GemmOpts()
            o.num_ctas = chunk_grid(a.shape[0], b.shape[1], sms, path)
            o.tile_n = chunk_tile_n(path)
            lpy.gemm(a, b, out=c, path=path, opts=o)

        def step():
            # single-process: no broadcast; the stream / event orchestration only
            import torch.distributed as dist  # noqa: F401
            rowpanel_gemm(A, blocks, C, bounds, gemm_fn=gemm_fn, compute_streams=streams, broadcast=False)

        ms = timeit(step)
        print(f"  chunks={chunks} streams={nstreams}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s")

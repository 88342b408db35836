#!/usr/bin/env python
"""3xTF32 at n (default 8192): time per product for each raster group given on
the command line (opts.raster_group, in CTA-pair tile rows), back-to-back
median of 12 after warm-up.  Run once per LPY_L2HINT setting (read at load);
DRAM bytes per product come from an ncu pass over the same script.
usage: LPY_L2HINT=0|1|2 python scripts/l2_ab.py n group [group ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

n = int(sys.argv[1])
groups = [int(g) for g in sys.argv[2:]] or [0]
reps = int(os.environ.get("REPS", "12"))
A = torch.rand(n, n, device="cuda") * 2 - 1
B = torch.rand(n, n, device="cuda") * 2 - 1
C = torch.empty(n, n, device="cuda")
hint = os.environ.get("LPY_L2HINT", "0")
for g in groups:
    o = lpy.GemmOpts()
    o.raster_group = g
    for _ in range(3):
        lpy.gemm(A, B, out=C, path="3xtf32", opts=o)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lpy.gemm(A, B, out=C, path="3xtf32", opts=o)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"hint={hint} group={g}: {ms:.4f} ms  {2 * n ** 3 / ms / 1e9:.1f} TFLOP/s", flush=True)

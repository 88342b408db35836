#!/usr/bin/env python
"""How fast can 128 SMs write a 12 MB C from scratch (config 5's output)?  torch fill_ of
1000 x 3000 fp32 and of a 2.5x larger buffer, CUDA-graph replayed (ncu for the kernel time)."""
import torch
for n in (1000 * 3000, 1000 * 3000 * 4):
    x = torch.empty(n, device="cuda")
    for _ in range(3):
        x.fill_(1.0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            x.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(f"fill {n * 4 / 1e6:.1f} MB: {us:.2f} us/call  {n * 4 / us / 1e6:.2f} TB/s")

#!/usr/bin/env python
"""Interleaved A/B timing of library builds on the Coulomb self-potential
(N particles, default 2^16): usage ab_coulomb.py <N> lib1.so [lib2.so ...]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402
import synth  # noqa: E402

n, libs = int(sys.argv[1]), sys.argv[2:]
pos, q = synth.particles(n, 0)
P = torch.from_numpy(pos.reshape(n, 3)).cuda()
Q = torch.from_numpy(q).cuda()
res = {}
ref = None
for rnd in range(3):
    for lib in libs:
        lpy._lib = None
        lpy.library_path = (lambda p: (lambda: p))(os.path.abspath(lib))
        lpy.load_library()
        phi = torch.empty(n, device="cuda")
        for _ in range(3):
            lpy.coulomb(P, P, Q, out=phi)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            lpy.coulomb(P, P, Q, out=phi)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        res.setdefault(lib, []).append(n * n / ms / 1e9)
        if ref is None:
            ref = phi.clone()
        elif rnd == 0:
            d = ((phi - ref).abs().max() / ref.abs().max()).item()
            print(f"{os.path.basename(lib)}: max |diff| / max |phi| vs first lib {d:.2e}")
for lib, v in res.items():
    print(f"{os.path.basename(lib):24s} N={n}: median {statistics.median(v):8.3f} T pairs/s  ({', '.join(f'{x:.3f}' for x in v)})")

#!/usr/bin/env python
"""Fixed cost of a launch shaped like the GEMM kernels (threads, dynamic smem),
back to back and after an L2-flushing fill, vs an lpy GEMM at n=128."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

probe = ctypes.CDLL(os.path.join(ROOT, "paper_1405_7470_b200", "liblpy_probe.so"))
probe.lpy_probe_empty_launch.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p, ctypes.c_void_p]
out = torch.zeros(4, dtype=torch.int32, device="cuda")
flush = torch.empty(64 << 20, device="cuda")


def t(fn, reps=50, flush_between=False):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        if flush_between:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return 1e3 * tot / reps


for ctas, threads, smem in [(1, 128, 16), (1, 384, 16), (1, 384, 100 << 10), (1, 384, 197 << 10),
                            (148, 384, 197 << 10), (148, 384, 227 << 10)]:
    f = lambda: probe.lpy_probe_empty_launch(ctas, threads, smem, out.data_ptr(), None)
    print(f"empty ctas={ctas:3d} threads={threads} smem={smem >> 10:3d} KB: "
          f"{t(f):7.2f} us back-to-back, {t(f, flush_between=True):7.2f} us after flush")
for n in (128, 256, 512, 1024):
    A = torch.randn(n, n, device="cuda")
    B = torch.randn(n, n, device="cuda")
    C = torch.empty(n, n, device="cuda")
    for path in ("ffma", "3xtf32"):
        f = lambda: lpy.gemm(A, B, out=C, path=path)
        print(f"gemm {path:6s} n={n:5d}: {t(f):7.2f} us back-to-back, {t(f, flush_between=True):7.2f} us after flush")

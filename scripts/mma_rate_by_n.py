#!/usr/bin/env python
"""Cycles per kind::tf32 MMA (K=8) by tile width N, single CTA (M=128) and CTA pair (M=256), A K-major,
B K- or MN-major (liblpy_probe.so lpy_probe_umma_rate_fmt; full rate = N/2 cycles)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
P = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1405_7470_b200", "liblpy_probe.so"))
P.lpy_probe_umma_rate_fmt.argtypes = [ctypes.c_int] * 6 + [ctypes.c_void_p, ctypes.c_void_p]
cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
iters = 4000
for cg in (2,):
    for fb in (1,):
        for n in (128, 256):
            rc = P.lpy_probe_umma_rate_fmt(n, 0, fb, iters, 148, cg, cyc.data_ptr(), None)
            torch.cuda.synchronize()
            c = cyc.item() / iters
            print(f"cg={cg} fb={fb} N={n:3d}: {c:7.2f} cycles/MMA  ({n / 2 / c:.2f} of full rate)  rc={rc}", flush=True)

# commits after every `every` k-blocks of 6 MMAs (the 3xTF32 k-block), the issuer waiting on the commit `lag` commits
# back; pattern 0: six plain SS MMAs, 1: the kernel's (collector fill / lastuse + SS), 2: the same with the third MMA
# in TS form (A from TMEM)
P.lpy_probe_umma_rate_commit.argtypes = [ctypes.c_int] * 7 + [ctypes.c_void_p, ctypes.c_void_p]
iters = 6000
for pattern in (0, 1, 2):
    for n in (128, 192, 256):
        for every, lag in ((0, 0), (1, 0), (0, -2)):
            rc = P.lpy_probe_umma_rate_commit(n, iters, every, lag, pattern, 148, 2, cyc.data_ptr(), None)
            torch.cuda.synchronize()
            c = cyc.item() / iters
            print(f"pattern={pattern} cg=2 N={n:3d} every={every} lag={lag:2d}: {c:7.2f} cycles/MMA ({n / 2 / c:.2f} of full)  rc={rc}",
                  flush=True)

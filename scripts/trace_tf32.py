#!/usr/bin/env python
"""Where does the 3xTF32 kernel's time go?  Runs the diagnostics build
(liblpy_trace.so, -DLPY_TRACE) once at n and prints per-role cycle shares
averaged over CTAs: MMA thread waiting for transformed stages / for drained
TMEM buffers, producer waiting for free stages, transform warp waiting for TMA.

usage: python scripts/trace_tf32.py [n] [promote_kblocks]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

TRACE = os.path.join(ROOT, "paper_1405_7470_b200", "liblpy_trace.so")
lpy.library_path = lambda: TRACE
lib = lpy.load_library()
lib.lpy_trace_set_buffer.argtypes = [ctypes.c_void_p]

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
promote = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A = torch.randn(n, n, device="cuda")
B = torch.randn(n, n, device="cuda")
if os.environ.get("LA", "row") == "col":   # LA / LB = row|col: operand layouts
    A = A.t().contiguous().t()
if os.environ.get("LB", "row") == "col":
    B = B.t().contiguous().t()
opts = lpy.GemmOpts()
opts.promote_kblocks = promote
for _ in range(3):
    lpy.gemm(A, B, path="3xtf32", opts=opts)
sms = torch.cuda.get_device_properties(0).multi_processor_count
buf = torch.zeros(sms * 8, dtype=torch.int64, device="cuda")
lib.lpy_trace_set_buffer(buf.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
lpy.gemm(A, B, path="3xtf32", opts=opts)
e1.record()
torch.cuda.synchronize()
lib.lpy_trace_set_buffer(None)
t = buf.view(sms, 8).double()
lead = t[t[:, 0] > 0]
names = ["mma_total", "mma_wait_ready", "mma_wait_acce", "prod_wait_empty", "xform_wait_full",
         "epi_wait_accf", "xform_busy", "epi_busy"]
ms = e0.elapsed_time(e1)
print(f"n={n} promote={promote or 'default'}: {ms:.3f} ms, {2 * n ** 3 / ms / 1e9:.1f} GFLOP/s")
tot = lead[:, 0].mean().item()
print(f"MMA thread cycles (mean over {lead.shape[0]} leader CTAs): {tot:.3e}")
for i, nm in enumerate(names):
    col = (lead if i < 3 else t)[:, i]
    print(f"  {nm:18s} mean {col.mean().item():.3e} cycles  ({100 * col.mean().item() / tot:5.1f}% of MMA total)")

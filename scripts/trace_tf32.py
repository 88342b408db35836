#!/usr/bin/env python
"""Where does the 3xTF32 kernel's time go?  Runs the diagnostics build
(liblpy_trace.so, -DLPY_TRACE) once at n and prints per-role cycle shares
averaged over CTAs: MMA thread waiting for transformed stages / for drained
TMEM buffers, producer waiting for free stages, transform warp waiting for TMA.

usage: python scripts/trace_tf32.py [n | M,N,K] [promote_kblocks]
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

shape = sys.argv[1] if len(sys.argv) > 1 else "8192"
M, N, K = (int(x) for x in shape.split(",")) if "," in shape else (int(shape),) * 3
n = M
promote = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A = torch.randn(M, K, device="cuda")
B = torch.randn(K, N, device="cuda")
if os.environ.get("LA", "row") == "col":   # LA / LB = row|col: operand layouts
    A = A.t().contiguous().t()
if os.environ.get("LB", "row") == "col":
    B = B.t().contiguous().t()
opts = lpy.GemmOpts()
opts.promote_kblocks = promote
for _ in range(3):
    lpy.gemm(A, B, path="3xtf32", opts=opts)
sms = torch.cuda.get_device_properties(0).multi_processor_count
buf = torch.zeros(sms * 8 + 16 + 12 * sms, dtype=torch.int64, device="cuda")
lib.lpy_trace_set_buffer(buf.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
lpy.gemm(A, B, path="3xtf32", opts=opts)
e1.record()
torch.cuda.synchronize()
lib.lpy_trace_set_buffer(None)
grid = int(os.environ.get("GRID", "0")) or sms   # CTAs launched (timeline slots follow grid*8 counters)
tl = buf[grid * 8: grid * 8 + 13].cpu().tolist()
ev = ["entry", "setup synced", "first TMA issued", "first stage transformed-in (xform saw full)", "MMA saw first ready",
      "MMA last commit issued", "epilogue saw first accf", "epilogue done", "exit (after cluster sync+dealloc)",
      "epilogue: last TMEM partial read", "split: partial written", "split: fenced + barrier", "split: fix-up sum read"]
if tl[0]:
    print("CTA 0 timeline (us from entry):")
    for name, v in zip(ev, tl):
        print(f"  {name:44s} {(v - tl[0]) / 1e3 if v else float('nan'):8.2f}")
ce4 = buf[grid * 8 + 16: grid * 8 + 16 + 12 * grid].view(grid, 12).double()
ce = ce4[:, :2]
if ce[0, 0] > 0:
    t0 = ce[:, 0].min()
    st, en = (ce[:, 0] - t0) / 1e3, (ce[:, 1] - t0) / 1e3
    print(f"per-CTA (us from first entry): entry min/med/max {st.min():.2f}/{st.median():.2f}/{st.max():.2f}, "
          f"exit min/med/max {en.min():.2f}/{en.median():.2f}/{en.max():.2f}")
    order = torch.argsort(en)
    print("  slowest CTAs (id: entry-exit):", ", ".join(f"{int(i)}: {st[i]:.1f}-{en[i]:.1f}" for i in order[-6:]))
    fx = ce4[:, 2] > 0
    if fx.any():
        f0, f1 = (ce4[fx, 2] - t0) / 1e3, (ce4[fx, 3] - t0) / 1e3
        print(f"  fix-up CTAs: {int(fx.sum())}, start min/med/max {f0.min():.2f}/{f0.median():.2f}/{f0.max():.2f}, "
              f"loads done min/med/max {f1.min():.2f}/{f1.median():.2f}/{f1.max():.2f}, exit max {en[fx].max():.2f}")
    mm = ce4[:, 4] > 0
    if mm.any():
        m1 = (ce4[mm, 4] - t0) / 1e3
        print(f"  MMA loop done (leaders) min/med/max {m1.min():.2f}/{m1.median():.2f}/{m1.max():.2f}")
    lp = ce4[:, 5] > 0
    if lp.any():
        l1 = (ce4[lp, 5] - t0) / 1e3
        print(f"  last partial promoted min/med/max {l1.min():.2f}/{l1.median():.2f}/{l1.max():.2f}")
    wt = ce4[:, 7] > 0
    if wt.any():
        w7 = (ce4[wt, 7] - t0) / 1e3
        print(f"  fix-up: other pieces written min/med/max {w7.min():.2f}/{w7.median():.2f}/{w7.max():.2f}; "
              f"reads (loads done - written) med/max {((ce4[wt, 3] - ce4[wt, 7]) / 1e3).median():.2f}/"
              f"{((ce4[wt, 3] - ce4[wt, 7]) / 1e3).max():.2f}")
    wr = ce4[:, 8] > 0
    if wr.any():
        a8, a9 = (ce4[wr, 8] - t0) / 1e3, (ce4[wr, 9] - t0) / 1e3
        print(f"  writers: {int(wr.sum())}, ticket min/med/max {a8.min():.2f}/{a8.median():.2f}/{a8.max():.2f}, "
              f"write time med/max {(a9 - a8).median():.2f}/{(a9 - a8).max():.2f}")
    sk = ce4[:, 6] > 0
    if sk.any():
        s1 = (ce4[sk, 6] - t0) / 1e3
        print(f"  first split piece's first MMA (leaders) min/med/max {s1.min():.2f}/{s1.median():.2f}/{s1.max():.2f}")
t = buf[: grid * 8].view(grid, 8).double()
lead = t[t[:, 0] > 0]
names = ["mma_total", "mma_wait_ready", "mma_wait_acce", "prod_wait_empty", "xform_wait_full",
         "epi_wait_accf", "xform_busy", "epi_busy"]
ms = e0.elapsed_time(e1)
print(f"{M}x{N}x{K} promote={promote or 'default'}: {ms:.3f} ms, {2 * M * N * K / ms / 1e9:.1f} GFLOP/s")
tot = lead[:, 0].mean().item()
print(f"MMA thread cycles (mean over {lead.shape[0]} leader CTAs): {tot:.3e}")
for i, nm in enumerate(names):
    col = (lead if i < 3 else t)[:, i]
    print(f"  {nm:18s} mean {col.mean().item():.3e} cycles  ({100 * col.mean().item() / tot:5.1f}% of MMA total)")

#!/usr/bin/env python
"""Host cost of one GEMM call, layer by layer (n=128, queue absorbs the launches):
  ctypes no-op      lpy_version() through ctypes (the FFI floor)
  C ABI             lpy_gemm_f32_ex through ctypes with prebuilt arguments
                    (validation, descriptor encode, launch)
  lpy.gemm          the torch-facing binding (shape/stride inference, device
                    guard, current stream)
  torch.mm          cuBLAS through torch, for context."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1405_7470_b200 as lpy  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
A = torch.randn(n, n, device="cuda")
B = torch.randn(n, n, device="cuda")
C = torch.empty(n, n, device="cuda")
lib = lpy.load_library()
stream = torch.cuda.current_stream().cuda_stream
pa, pb, pc = A.data_ptr(), B.data_ptr(), C.data_ptr()


def per_call(fn, reps=300):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    dt = time.perf_counter() - t0
    torch.cuda.synchronize()
    return 1e6 * dt / reps


probe_path = os.path.join(ROOT, "paper_1405_7470_b200", "liblpy_probe.so")
rows = [("ctypes no-op (lpy_version)", lambda: lib.lpy_version()),
        ("C ABI M=0 (validation only)",
         lambda: lib.lpy_gemm_f32_ex(0, n, n, pa, n, 0, pb, n, 0, pc, n, 0, stream, 0, None)),
        ("C ABI K=0 (validation + memset)",
         lambda: lib.lpy_gemm_f32_ex(n, n, 0, pa, n, 0, pb, n, 0, pc, n, 0, stream, 0, None))]
if os.path.exists(probe_path):
    import ctypes
    probe = ctypes.CDLL(probe_path)
    probe.lpy_probe_empty_launch.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p, ctypes.c_void_p]
    flag = torch.zeros(4, dtype=torch.int32, device="cuda")
    rows.append(("empty kernel <<<148, 384, 197 KB>>>",
                 lambda: probe.lpy_probe_empty_launch(148, 384, 197 << 10, flag.data_ptr(), stream)))
for path in ("ffma", "3xtf32"):
    pid = lpy.PATHS[path]
    rows.append((f"C ABI lpy_gemm_f32_ex {path}",
                 lambda pid=pid: lib.lpy_gemm_f32_ex(n, n, n, pa, n, 0, pb, n, 0, pc, n, 0, stream, pid, None)))
    rows.append((f"lpy.gemm {path}", lambda path=path: lpy.gemm(A, B, out=C, path=path)))
rows.append(("torch.mm (cuBLAS)", lambda: torch.mm(A, B, out=C)))
for name, fn in rows:
    print(f"{name:36s} {per_call(fn):8.2f} us/call", flush=True)

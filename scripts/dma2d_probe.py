"""PCIe rates of 2-D copies: column blocks (w columns) of a pinned row-major
8192 x 8192 fp32 host matrix into packed device blocks (cudaMemcpy2DAsync),
vs one linear copy of the same bytes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from cuda.bindings import runtime as rt

n = 8192
H = torch.empty(n, n, dtype=torch.float32).pin_memory()
D = torch.empty(n * n, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
H2D = rt.cudaMemcpyKind.cudaMemcpyHostToDevice


def timed(fn, reps=3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms = timed(lambda: rt.cudaMemcpyAsync(D.data_ptr(), H.data_ptr(), 4 * n * n, H2D, s))
print(f"linear 268 MB: {ms:.3f} ms  {4 * n * n / ms / 1e6:.1f} GB/s")
for w in (4096, 2048, 1024, 512, 256, 128):
    def f():
        for c0 in range(0, n, w):
            rt.cudaMemcpy2DAsync(D.data_ptr() + 4 * n * c0, 4 * w, H.data_ptr() + 4 * c0, 4 * n, 4 * w, n, H2D, s)
    ms = timed(f)
    print(f"2-D column blocks w={w:5d} ({n // w} copies of {n} rows x {4 * w} B): {ms:.3f} ms  "
          f"{4 * n * n / ms / 1e6:.1f} GB/s")

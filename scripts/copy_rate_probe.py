"""Copy throughput of a few SMs, alone: thread copies (4 x 16 B in flight per
thread, 512 threads per CTA) vs TMA bulk copies (one thread, 6 x 32 KB in
flight per CTA), 268 MB device-to-device (diagnostics for the broadcast's SM
budget)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1405_7470_b200 as lpy
probe = ctypes.CDLL(os.path.join(os.path.dirname(lpy.library_path()), "liblpy_probe.so"))
for f in (probe.lpy_probe_persistent_copy, probe.lpy_probe_bulk_copy):
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_void_p]
n = 1 << 26
src = torch.rand(n, device="cuda")
dst = torch.empty(n, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for name, fn, arg in (("threads", probe.lpy_probe_persistent_copy, n), ("bulk", probe.lpy_probe_bulk_copy, 4 * n)):
    for ctas in (1, 2, 4, 8, 16, 32, 148):
        dst.zero_()
        fn(dst.data_ptr(), src.data_ptr(), arg, ctas, s)
        torch.cuda.synchronize()
        assert torch.equal(dst, src), (name, ctas)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            fn(dst.data_ptr(), src.data_ptr(), arg, ctas, s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{name:8s} ctas={ctas:4d}: {4 * n / ms / 1e6:8.1f} GB/s copied ({4 * n / ms / 1e6 / ctas:6.1f} per CTA)", flush=True)

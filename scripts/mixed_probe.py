#!/usr/bin/env python
"""Probe: B multicast on the 33 clusters of 4 that place (132 SMs) for C[:, :Nx], and the plain
pair kernel on the leftover 16 SMs (8 pairs, num_ctas=16) for C[:, Nx:], on two streams at once,
vs the default full-chip product and vs multicast alone.  CUDA-graph replay, interleaved rounds.
usage: python scripts/mixed_probe.py <product.so> <mc.so> n Nx[,Nx...]"""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1405_7470_b200 as lpy

L0, L1 = (ctypes.CDLL(os.path.abspath(x)) for x in sys.argv[1:3])
n = int(sys.argv[3])
nxs = [int(x) for x in sys.argv[4].split(",")]
i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
for L in (L0, L1):
    L.lpy_gemm_f32_ex.argtypes = [i64, i64, i64, vp, i64, i32, vp, i64, i32, vp, i64, i32, vp, i32, vp]
    L.lpy_gemm_f32_ex.restype = i32
A = torch.rand(n, n, device="cuda") * 2 - 1
B = torch.rand(n, n, device="cuda") * 2 - 1
C = torch.empty(n, n, device="cuda")


def call(L, cols0, cols1, stream, num_ctas=0):
    o = lpy.GemmOpts()
    o.num_ctas = num_ctas
    st = L.lpy_gemm_f32_ex(n, cols1 - cols0, n, A.data_ptr(), n, 0, B.data_ptr() + 4 * cols0, n, 0,
                           C.data_ptr() + 4 * cols0, n, 0, stream.cuda_stream, 2, ctypes.byref(o))
    assert st == 0, st


s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def variant(name):
    if name == "base":
        return lambda: call(L0, 0, n, s1)
    if name == "mc":
        return lambda: call(L1, 0, n, s1)
    nx = int(name[5:])

    def f():
        ev = torch.cuda.Event()
        ev.record(s1)
        s2.wait_event(ev)
        call(L1, 0, nx, s1)
        call(L0, nx, n, s2, num_ctas=16)
        ev2 = torch.cuda.Event()
        ev2.record(s2)
        s1.wait_event(ev2)
    return f


names = ["base", "mc"] + [f"mixed{nx}" for nx in nxs]
ref = (A[:64].double() @ B.double())
D = (A[:64].abs().double() @ B.abs().double())
graphs = {}
for nm in names:
    f = variant(nm)
    for _ in range(2):
        with torch.cuda.stream(s1):
            f()
    torch.cuda.synchronize()
    err = ((C[:64].double() - ref).abs() / D).max().item()
    g = torch.cuda.CUDAGraph()
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s1):
        for _ in range(3):
            f()
    graphs[nm] = (g, err)
torch.cuda.synchronize()
res = {nm: [] for nm in names}
for rnd in range(6):
    for nm in names[rnd % len(names):] + names[:rnd % len(names)]:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        with torch.cuda.stream(s1):
            graphs[nm][0].replay()
        e1.record(s1)
        torch.cuda.synchronize()
        res[nm].append(e0.elapsed_time(e1) / 3)
for nm in names:
    ms = statistics.median(res[nm])
    print(f"{nm:12s} {ms:8.3f} ms  {2 * n ** 3 / ms / 1e9:7.1f} TFLOP/s  err {graphs[nm][1]:.1e}  "
          f"({' '.join(f'{x:.3f}' for x in res[nm])})", flush=True)

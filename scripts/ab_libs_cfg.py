#!/usr/bin/env python
"""Interleaved A/B of library builds on a list of shapes (one path): CUDA-graph
replay of 20 calls per measurement, rounds interleaved over the libraries,
median per (library, shape); sampled parity vs float64 torch per library.
usage: python scripts/ab_libs_cfg.py <path> lib1.so lib2.so ...   (shapes: SHAPES env,
       "M,N,K,la,lb;..." default the FFMA under-filled configs + n=8192)"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1405_7470_b200 as lpy

path, libs = sys.argv[1], sys.argv[2:]
shapes = os.environ.get("SHAPES", "1024,1024,1024,row,row;1024,1024,1024,row,col;1000,3000,780,row,col;"
                                  "2048,2048,2048,row,row;8192,8192,8192,row,row")
cases = []
for spec in shapes.split(";"):
    M, N, K, la, lb = spec.split(",")
    M, N, K = int(M), int(N), int(K)
    a = torch.rand(M, K, device="cuda") * 2 - 1 if la == "row" else (torch.rand(K, M, device="cuda") * 2 - 1).t()
    b = torch.rand(K, N, device="cuda") * 2 - 1 if lb == "row" else (torch.rand(N, K, device="cuda") * 2 - 1).t()
    cases.append((spec, a, b, torch.empty(M, N, device="cuda")))


import ctypes
_libs = {}


def use(lib):
    """Bind `gemm` to lpy_gemm_f32_ex of this .so (raw ctypes: an older build may
    lack symbols the current binding expects)."""
    global gemm
    if lib not in _libs:
        L = ctypes.CDLL(os.path.abspath(lib))
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.lpy_gemm_f32_ex.argtypes = [i64, i64, i64, vp, i64, i32, vp, i64, i32, vp, i64, i32, vp, i32, vp]
        L.lpy_gemm_f32_ex.restype = i32
        _libs[lib] = L
    L = _libs[lib]
    pid = lpy.PATHS[path]

    def gemm(a, b, out):
        la, lb, lc = lpy.operand_layout(a), lpy.operand_layout(b), lpy.operand_layout(out)
        st = L.lpy_gemm_f32_ex(a.shape[0], b.shape[1], a.shape[1], a.data_ptr(), la[1], la[0], b.data_ptr(), lb[1],
                               lb[0], out.data_ptr(), lc[1], lc[0], torch.cuda.current_stream().cuda_stream, pid, None)
        assert st == 0, st


graphs = {}
for lib in libs:
    use(lib)
    for spec, a, b, C in cases:
        reps = 20 if a.shape[0] * b.shape[1] * a.shape[1] < 2e10 else 3
        for _ in range(3):
            gemm(a, b, C)
        torch.cuda.synchronize()
        ref = a[:32].double() @ b.double()
        err = ((C[:32].double() - ref).abs() / (a[:32].abs().double() @ b.abs().double())).max().item()
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                gemm(a, b, C)
        graphs[(lib, spec)] = (g, reps, err, (a, b, C))   # (tensors kept alive by the cases list too)
res = {}
for rnd in range(5):
    for spec, a, b, C in cases:
        for lib in libs[rnd % len(libs):] + libs[:rnd % len(libs)]:   # rotate: no first-in-round bias
            g, reps, _, _ = graphs[(lib, spec)]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            res.setdefault((lib, spec), []).append(e0.elapsed_time(e1) / reps * 1e3)
for spec, a, b, C in cases:
    fl = 2.0 * a.shape[0] * b.shape[1] * a.shape[1]
    for lib in libs:
        v = res[(lib, spec)]
        us = statistics.median(v)
        print(f"{os.path.basename(lib):22s} {spec:28s} {us:10.2f} us {fl / us / 1e6:7.2f} TFLOP/s "
              f"err {graphs[(lib, spec)][2]:.1e}  ({' '.join(f'{x:.1f}' for x in v)})", flush=True)

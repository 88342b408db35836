"""One (shape, layouts, tile_n) FFMA product per process: prints OK / the error (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1405_7470_b200 as lpy
M, N, K = (int(x) for x in sys.argv[1:4]); la, lb, tn = sys.argv[4], sys.argv[5], int(sys.argv[6])
plan = int(sys.argv[7]) if len(sys.argv) > 7 else 0
a = torch.rand(M, K, device="cuda") * 2 - 1 if la == "row" else (torch.rand(K, M, device="cuda") * 2 - 1).t()
b = torch.rand(K, N, device="cuda") * 2 - 1 if lb == "row" else (torch.rand(N, K, device="cuda") * 2 - 1).t()
o = lpy.GemmOpts(); o.tile_n = tn; o.plan_sms = plan
try:
    C = lpy.gemm(a, b, path="ffma", opts=o)
    torch.cuda.synchronize()
    ref = a.double() @ b.double()
    err = ((C.double() - ref).abs() / (a.abs().double() @ b.abs().double())).max().item()
    print(f"OK {M}x{N}x{K} {la}{lb} tile_n={tn} plan={plan} err={err:.2e}")
except Exception as e:
    print(f"FAIL {M}x{N}x{K} {la}{lb} tile_n={tn} plan={plan}: {str(e).splitlines()[0]}")

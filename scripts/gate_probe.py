"""Diagnostics: a gated product whose flags are raised late by a side stream.
Prints host-call times and the stream flags of torch's side stream."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1405_7470_b200 as lpy
from cuda.bindings import runtime as rt

path = sys.argv[1] if len(sys.argv) > 1 else "ffma"
mode = sys.argv[2] if len(sys.argv) > 2 else "sleep"
torch.cuda._sleep(1)      # load the spin kernel (lazy loading would block behind the product)
M, N, K, ck = 512, 1024, 2048, 256
A = torch.rand(M, K, device="cuda"); B = torch.rand(K, N, device="cuda")
flags = torch.zeros(K // ck, dtype=torch.int32, device="cuda")
side = torch.cuda.Stream()
print("side stream flags", rt.cudaStreamGetFlags(side.cuda_stream), "current", torch.cuda.current_stream().cuda_stream, flush=True)
o = lpy.GemmOpts(); o.plan_sms = 140
torch.cuda.synchronize()
t0 = time.time()
C = lpy.gemm(A, B, path=path, opts=o, gate=lpy.KGate(flags.data_ptr(), ck, 1, 3000))
print(f"gemm launched after {time.time()-t0:.4f}s", flush=True)
try:
    with torch.cuda.stream(side):
        if mode == "sleep":
            torch.cuda._sleep(20_000_000)
        print(f"sleep launched {time.time()-t0:.4f}s", flush=True)
        for c in range(K // ck):
            lpy.kgate_signal(flags, c, 1, stream=side)
    print(f"signals launched {time.time()-t0:.4f}s", flush=True)
    torch.cuda.synchronize()
    print(f"done {time.time()-t0:.4f}s err", ((C - A @ B).abs().max() / (A @ B).abs().max()).item(), flush=True)
except Exception as e:
    print(f"EXC at {time.time()-t0:.4f}s: {e}".splitlines()[0], flush=True)

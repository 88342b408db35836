import sys, torch
sys.path.insert(0, "/root/repo")
import paper_1405_7470_b200 as lpy
A = torch.randn(1000, 780, device="cuda")[:, :777]
Bs = torch.randn(3000, 780, device="cuda")[:, :777]
B = Bs.t()
C = torch.empty(1000, 3000, device="cuda")
for p in ("ffma", "3xtf32"):
    for _ in range(3):
        lpy.gemm(A, B, out=C, path=p)
torch.cuda.synchronize()

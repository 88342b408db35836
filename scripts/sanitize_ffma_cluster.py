import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import synth
from gpu_util import check, run_gemm
for (M, N, K) in ((1024, 1024, 1024), (128, 128, 128), (1000, 1024, 600)):
    A = synth.matrix(M, K, seed=5, matrix_id=0); B = synth.matrix(K, N, seed=5, matrix_id=1)
    C, ok = run_gemm(A, B, 0, 0, 0, path="ffma"); assert ok; print(M, N, K, check(C, A, B))

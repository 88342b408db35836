#!/usr/bin/env python
"""Randomised parity sweep through the C ABI: random shapes (1..3000 per dim, some chosen to hit the 176-wide
3xTF32 tiles and the FFMA split / stream-K schedules), random layouts and leading-dimension pads, both paths;
every element within the 1e-5 bound of a float64 reference (cuBLAS DGEMM on the same inputs) and C's padding
untouched (sentinel).  usage: python scripts/fuzz_parity.py [cases] [seed]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1405_7470_b200 as lpy

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
SENT = -31337.0
bad = 0
for i in range(cases):
    if i % 4 == 0:
        M, N, K = (int(x) for x in rng.integers(1, 3001, 3))
    elif i % 4 == 1:      # wide / ragged K-major shapes (176-wide tiles, split-K)
        M, N, K = int(rng.integers(200, 2100)), int(rng.integers(1500, 5200)), int(rng.integers(100, 2100))
    elif i % 4 == 2:      # small
        M, N, K = (int(x) for x in rng.integers(1, 300, 3))
    else:                 # long K
        M, N, K = int(rng.integers(1, 1200)), int(rng.integers(1, 1200)), int(rng.integers(2000, 9000))
    la, lb, lc = (int(x) for x in rng.integers(0, 2, 3))
    pa, pb, pc = (int(x) for x in rng.choice([0, 1, 3, 4], 3))
    path = ["ffma", "3xtf32"][i % 2] if i % 8 < 6 else "auto"
    A = torch.rand(M, K, dtype=torch.float64, device="cuda") * 2 - 1
    B = torch.rand(K, N, dtype=torch.float64, device="cuda") * 2 - 1
    A32, B32 = A.float(), B.float()

    def lay(X, layout, pad):
        r, c = X.shape
        if layout == 0:
            buf = torch.full((r, c + pad), SENT, device="cuda")
            buf[:, :c] = X
            return buf, c + pad, buf
        buf = torch.full((c, r + pad), SENT, device="cuda")
        buf[:, :r] = X.t()
        return buf, r + pad, buf
    ab, lda, _ = lay(A32, la, pa)
    bb, ldb, _ = lay(B32, lb, pb)
    cbuf, ldc, _ = lay(torch.zeros(M, N, device="cuda"), lc, pc)
    cbuf.fill_(SENT)
    st = lpy.lpy_gemm_f32_ex(M, N, K, ab.data_ptr(), lda, la, bb.data_ptr(), ldb, lb, cbuf.data_ptr(), ldc, lc,
                             torch.cuda.current_stream().cuda_stream, lpy.PATHS[path], None)
    torch.cuda.synchronize()
    if st != 0:
        print(f"case {i}: status {st} for {M}x{N}x{K} {la}{lb}{lc} pads {pa}{pb}{pc} {path}", flush=True)
        bad += 1
        continue
    C = cbuf[:, :N] if lc == 0 else cbuf[:, :M].t()
    ref = A32.double() @ B32.double()
    D = A32.abs().double() @ B32.abs().double()
    err = ((C.double() - ref).abs() / D.clamp_min(1e-300)).max().item() if M * N else 0.0
    pad_ok = True
    if lc == 0 and pc:
        pad_ok = bool((cbuf[:, N:] == SENT).all())
    elif lc == 1 and pc:
        pad_ok = bool((cbuf[:, M:] == SENT).all())
    if not (err <= 1e-5) or not pad_ok:
        bad += 1
        print(f"case {i}: FAIL {M}x{N}x{K} la{la} lb{lb} lc{lc} pads {pa},{pb},{pc} {path}: err {err:.3e} pad_ok {pad_ok}",
              flush=True)
print(f"fuzz: {cases} cases, {bad} failures")

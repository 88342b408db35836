#!/usr/bin/env python
"""Small products on both paths for compute-sanitizer (memcheck / racecheck /
synccheck): ragged shapes, every layout, the repack path, and a check against
the oracle so a silent corruption under the tool is caught too.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_small.py
"""
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import synth  # noqa: E402
from gpu_util import check, run_gemm  # noqa: E402

worst = 0.0
for path in ("ffma", "3xtf32"):
    for (M, N, K), (la, lb, lc) in itertools.product([(129, 257, 33), (300, 200, 130)],
                                                       itertools.product((0, 1), (0, 1), (0, 1))):
        A = synth.matrix(M, K, seed=M + K, matrix_id=0)
        B = synth.matrix(K, N, seed=M + K, matrix_id=1)
        C, pad_ok = run_gemm(A, B, la, lb, lc, lda=synth.min_ld(M, K, la) + 3,
                             ldb=synth.min_ld(K, N, lb), ldc=synth.min_ld(M, N, lc) + 1, path=path)
        assert pad_ok
        worst = max(worst, check(C, A, B))
    # C rows 16-byte but not 32-byte aligned (ldc % 8 == 4): the float4 store path
    A = synth.matrix(300, 130, seed=3, matrix_id=0)
    B = synth.matrix(130, 200, seed=3, matrix_id=1)
    C, pad_ok = run_gemm(A, B, 0, 0, 0, ldc=204, path=path)
    assert pad_ok
    worst = max(worst, check(C, A, B))
print(f"sanitize_small: all products within tolerance (worst {worst:.2e})")

# split-K FFMA (under-filled grid: 72 tiles -> 2 slices), the 3xTF32 tail
# split (90 pair tiles = 2 waves, the last 16 cut into k-slices) and the 3xTF32
# cluster split (single under-filled waves: k-slices summed through DSMEM)
import paper_1405_7470_b200 as lpy  # noqa: E402
import oracle  # noqa: E402
import torch  # noqa: E402
for path, (M, N, K) in (("ffma", (1000, 1100, 600)), ("ffma", (1024, 1024, 1024)), ("ffma", (128, 128, 128)),
                        ("3xtf32", (2560, 2304, 1024)),
                        ("3xtf32", (512, 512, 512)), ("3xtf32", (1024, 1024, 1024)), ("3xtf32", (700, 600, 520))):
    A = synth.matrix(M, K, seed=5, matrix_id=0)
    B = synth.matrix(K, N, seed=5, matrix_id=1)
    C, pad_ok = run_gemm(A, B, 0, 0, 0, path=path)
    assert pad_ok
    worst = max(worst, check(C, A, B))
print(f"sanitize_small: split products within tolerance (worst {worst:.2e})")

# round 2: FFMA stream-K (a single wave of 64 tiles over every SM, in-kernel
# fix-up), the 3xTF32 stream-K tail (K >= 4096), the TMEM-A narrow tiles, and
# the K-gated product with its flags raised by the signal kernel on a second stream
for path, (M, N, K), plan in (("ffma", (1024, 3000, 2048), 0), ("3xtf32", (768, 1536, 4096), 16),
                              ("3xtf32", (512, 768, 256), 0)):
    A = synth.matrix(M, K, seed=6, matrix_id=0)
    B = synth.matrix(K, N, seed=6, matrix_id=1)
    o = lpy.GemmOpts()
    o.plan_sms = plan
    C, pad_ok = run_gemm(A, B, 0, 0, 0, path=path, opts=o)
    assert pad_ok
    worst = max(worst, check(C, A, B))
for path in ("ffma", "3xtf32"):
    M, N, K = 512, 1024, 1024
    A = synth.matrix(M, K, seed=7, matrix_id=0)
    B = synth.matrix(K, N, seed=7, matrix_id=1)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    side = torch.cuda.Stream()
    o = lpy.GemmOpts()
    o.plan_sms = torch.cuda.get_device_properties(0).multi_processor_count - 16
    C = lpy.gemm(dA, dB, path=path, opts=o, gate=lpy.KGate(flags.data_ptr(), 256, 1, 60000))
    with torch.cuda.stream(side):
        for c in range(4):
            lpy.kgate_signal(flags, c, 1, stream=side)
    torch.cuda.synchronize()
    worst = max(worst, check(C.cpu().numpy(), A, B))
print(f"sanitize_small: round-2 schedules within tolerance (worst {worst:.2e})")

# saxpy edges (head / tail, misaligned x, x == y, strided)
for n, offx, offy in ((1, 0, 0), (13, 1, 3), (1001, 2, 0), (4099, 0, 5)):
    x = synth.vector(n, 1, synth.VECTOR_X)
    y = synth.vector(n, 1, synth.VECTOR_Y)
    tx = torch.zeros(n + 8, device="cuda")
    ty = torch.zeros(n + 8, device="cuda")
    tx[offx:offx + n] = torch.from_numpy(x)
    ty[offy:offy + n] = torch.from_numpy(y)
    lpy.saxpy(1.5, tx[offx:offx + n], ty[offy:offy + n])
    torch.cuda.synchronize()
    assert oracle.saxpy_error_ulps(ty[offy:offy + n].cpu().numpy(), oracle.saxpy(n, 1.5, x, 1, y, 1)) <= 1
tz = torch.from_numpy(synth.vector(777, 2)).cuda()
lpy.saxpy(0.5, tz[::3], tz[::3])
torch.cuda.synchronize()
print("sanitize_small: saxpy edges ok")

# Coulomb: self-potential with source slices, separate sets, the coincident fallback
for nt, ns in ((300, 300), (7, 2000), (1500, 1500)):
    pos, q = synth.particles(max(nt, ns), 3)
    P = torch.from_numpy(pos.reshape(-1, 3)).cuda()
    Q = torch.from_numpy(q).cuda()
    if nt == ns:
        phi = lpy.coulomb(P[:nt], P[:ns], Q[:ns])
        ref, D = oracle.coulomb(nt, pos[:3 * nt].copy(), 3, ns, pos[:3 * ns].copy(), 3, q[:ns].copy())
    else:
        T = P[ns - nt:ns].clone()          # targets on top of sources: the fallback path
        phi = lpy.coulomb(T, P[:ns], Q[:ns])
        ref, D = oracle.coulomb(nt, pos[3 * (ns - nt):3 * ns].copy(), 3, ns, pos[:3 * ns].copy(), 3,
                                q[:ns].copy())
    torch.cuda.synchronize()
    assert np.max(np.abs(phi.cpu().numpy() - ref) / D) <= 5e-6
print("sanitize_small: coulomb ok")

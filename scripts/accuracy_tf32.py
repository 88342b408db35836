#!/usr/bin/env python
"""Measured accuracy of the 3xTF32 path vs the promotion interval (and of the
FFMA path for reference): max normalised error over sampled elements at n
(default 8192) on the stress distribution uniform[0,1) and the default
uniform[-1,1).  Feeds DESIGN.md reading A10 and the promote default.

usage: python scripts/accuracy_tf32.py [n] [samples]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the checker)
import paper_1405_7470_b200 as lpy  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
samples = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
rng = np.random.default_rng(1)
for dist in ("uniform01", "uniform"):
    A = synth.matrix(n, n, seed=0, matrix_id=0, dist=dist)
    B = synth.matrix(n, n, seed=0, matrix_id=1, dist=dist)
    ii = rng.integers(0, n, samples)
    jj = rng.integers(0, n, samples)
    Cref, D = oracle.gemm_elems(n, n, n, A.reshape(-1), n, 0, B.reshape(-1), n, 0, ii, jj)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    for path, promote in (("ffma", 0), ("3xtf32", 4), ("3xtf32", 8), ("3xtf32", 16), ("3xtf32", 32)):
        o = lpy.GemmOpts()
        o.promote_kblocks = promote
        C = lpy.gemm(dA, dB, path=path, opts=o).cpu().numpy()
        err = oracle.normalized_error(C[ii, jj], Cref, D)
        signed = float(np.mean((C[ii, jj] - Cref) / D))
        print(f"{dist:9s} n={n} {path:6s} promote={promote:2d}: max norm err {err:.3e}  mean signed {signed:+.3e}")

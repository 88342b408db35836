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
print(f"sanitize_small: all products within tolerance (worst {worst:.2e})")

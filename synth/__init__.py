"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no product, no sum over k): it
only draws fp32 matrices from a counter-based generator and lays them out in
memory.  Both the oracle tests and the GPU tests/bench take their inputs from
here, so the two sides agree on the input bits without sharing any compute
code.

Generator: SplitMix64 (Steele, Lea, Flood 2014 finaliser) keyed on
(seed, matrix_id, logical row, logical column).  Because the key is the
LOGICAL index, the same matrix comes out whatever layout / leading dimension
it is later stored with -- the paper's data-layout tags change where an
element lives, not its value (section 2.4.3).

Distributions (readings A2/A3):
  "uniform"   : k * 2^-23, k uniform in [-2^23, 2^23)   -> [-1, 1)  (default)
  "uniform01" : k * 2^-23, k uniform in [0, 2^23)       -> [0, 1)   (stress)
  "int"       : integers uniform in [-8, 8]             (bit-exact tests)
  "wide"      : +-(1 + f) * 2^e, f on a 2^-23 grid, e uniform in [-20, 20]
All values are exactly representable in fp32.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "DISTS", "ROW_MAJOR", "COL_MAJOR", "MATRIX_A", "MATRIX_B",
    "splitmix64", "matrix", "store", "load_logical", "identity", "permutation",
    "min_ld", "VECTOR_X", "VECTOR_Y", "vector", "strided", "PARTICLES", "CHARGES", "particles",
]

ROW_MAJOR = 0
COL_MAJOR = 1
MATRIX_A = 0
MATRIX_B = 1
VECTOR_X = 2
VECTOR_Y = 3
PARTICLES = 4
CHARGES = 5
DISTS = ("uniform", "uniform01", "int", "wide")

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x):
    """SplitMix64 step on a uint64 scalar or array (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def _hash_block(seed: int, matrix_id: int, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    base = splitmix64(np.uint64((int(seed) & 0xFFFFFFFF) | ((int(matrix_id) & 0xFFFF) << 32)))
    rk = splitmix64(base ^ rows.astype(np.uint64))
    return splitmix64(rk[:, None] ^ cols.astype(np.uint64)[None, :])


def _to_dist(h: np.ndarray, dist: str) -> np.ndarray:
    if dist == "uniform":
        k = (h >> np.uint64(40)).astype(np.int64) - (1 << 23)
        return (k.astype(np.float64) * 2.0 ** -23).astype(np.float32)
    if dist == "uniform01":
        k = (h >> np.uint64(41)).astype(np.int64)
        return (k.astype(np.float64) * 2.0 ** -23).astype(np.float32)
    if dist == "int":
        return ((h % np.uint64(17)).astype(np.int64) - 8).astype(np.float32)
    if dist == "wide":
        frac = ((h >> np.uint64(40)) & np.uint64(0x7FFFFF)).astype(np.float64) * 2.0 ** -23
        e = ((h >> np.uint64(8)) % np.uint64(41)).astype(np.int64) - 20
        sign = np.where((h >> np.uint64(63)) == 1, -1.0, 1.0)
        return (sign * (1.0 + frac) * np.ldexp(1.0, e)).astype(np.float32)
    raise ValueError(f"unknown dist {dist!r}; expected one of {DISTS}")


def matrix(rows: int, cols: int, seed: int = 0, matrix_id: int = 0, dist: str = "uniform",
           row0: int = 0, col0: int = 0, block_rows: int = 1024) -> np.ndarray:
    """Logical rows x cols fp32 matrix; element (r, c) depends only on
    (seed, matrix_id, row0 + r, col0 + c).  `row0` lets a rank draw just its
    row panel of a larger matrix (reading A12)."""
    out = np.empty((rows, cols), dtype=np.float32)
    cidx = np.arange(col0, col0 + cols, dtype=np.uint64)
    for r in range(0, rows, block_rows):
        rr = min(block_rows, rows - r)
        ridx = np.arange(row0 + r, row0 + r + rr, dtype=np.uint64)
        out[r:r + rr] = _to_dist(_hash_block(seed, matrix_id, ridx, cidx), dist)
    return out


def vector(n: int, seed: int = 0, vector_id: int = VECTOR_X, dist: str = "uniform",
           start: int = 0) -> np.ndarray:
    """Logical fp32 vector of n elements; element i depends only on
    (seed, vector_id, start + i) -- row 0 of a 1 x n matrix of the same
    generator, so a rank or chunk can draw its slice alone."""
    return matrix(1, n, seed=seed, matrix_id=vector_id, dist=dist, col0=start)[0]


def strided(v: np.ndarray, inc: int, pad_value: float = float("nan")) -> np.ndarray:
    """Lay vector v out with increment inc (element i at buf[i*inc]); the gaps
    hold pad_value (NaN: a kernel that reads them poisons its result)."""
    n = v.shape[0]
    if n == 0:
        return np.zeros(0, dtype=np.float32)
    buf = np.full((n - 1) * inc + 1, pad_value, dtype=np.float32)
    buf[::inc] = v
    return buf


def particles(n: int, seed: int = 0, charges: str = "uniform", start: int = 0,
              ld: int = 3) -> tuple[np.ndarray, np.ndarray]:
    """n point charges for the 3D Coulomb row:
    positions uniform in the unit cube [0, 1)^3 on a 2^-23 grid (so every
    coordinate difference is exact in fp32 and float64), charges from
    `charges` ("uniform": [-1, 1), "uniform01": [0, 1), "int": [-8, 8]).
    Returns (flat positions buffer, point i at [i*ld : i*ld+3]; charges)."""
    pos = matrix(n, 3, seed=seed, matrix_id=PARTICLES, dist="uniform01", row0=start)
    q = vector(n, seed=seed, vector_id=CHARGES, dist=charges, start=start)
    if ld == 3:
        return np.ascontiguousarray(pos).reshape(-1), q
    buf = np.full((n, ld), np.nan, dtype=np.float32)
    buf[:, :3] = pos
    return buf.reshape(-1)[: max(0, (n - 1) * ld + 3)].copy(), q


def min_ld(rows: int, cols: int, layout: int) -> int:
    """Smallest legal leading dimension (include/lpy.h: ld >= max(1, minor extent))."""
    return max(1, cols if layout == ROW_MAJOR else rows)


def store(logical: np.ndarray, layout: int = ROW_MAJOR, ld: int | None = None,
          pad_value: float = float("nan")) -> tuple[np.ndarray, int]:
    """Lay a logical (rows, cols) matrix out in memory.

    Row-major: X(r, c) = buf[r * ld + c];  column-major: X(r, c) = buf[r + c * ld]
    (include/lpy.h; PAPER.md P:278-280 'dim_tags: (stride:1)').
    Padding between lines is filled with `pad_value` (NaN by default) so a
    kernel that reads outside the logical matrix poisons its result.
    Returns (flat fp32 buffer, ld)."""
    rows, cols = logical.shape
    if ld is None:
        ld = min_ld(rows, cols, layout)
    lines, inner = (rows, cols) if layout == ROW_MAJOR else (cols, rows)
    if ld < max(1, inner):
        raise ValueError("ld smaller than the minor extent")
    if lines == 0:
        return np.zeros(0, dtype=np.float32), ld
    buf = np.full((lines, ld), pad_value, dtype=np.float32)
    buf[:, :inner] = logical if layout == ROW_MAJOR else logical.T
    flat = buf.reshape(-1)
    # the last line needs only `inner` elements
    return np.ascontiguousarray(flat[: (lines - 1) * ld + inner]), ld


def load_logical(buf: np.ndarray, rows: int, cols: int, layout: int, ld: int) -> np.ndarray:
    """Inverse of `store`: read the logical (rows, cols) matrix out of `buf`."""
    if rows == 0 or cols == 0:
        return np.zeros((rows, cols), dtype=buf.dtype)
    if layout == ROW_MAJOR:
        idx = np.arange(rows)[:, None] * ld + np.arange(cols)[None, :]
    else:
        idx = np.arange(rows)[:, None] + np.arange(cols)[None, :] * ld
    return buf[idx]


def identity(n: int) -> np.ndarray:
    return np.eye(n, dtype=np.float32)


def permutation(n: int, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """A permutation matrix P (P[i, perm[i]] = 1) drawn from the counter-based
    generator, and the permutation itself."""
    keys = splitmix64(np.arange(n, dtype=np.uint64) ^ splitmix64(np.uint64(seed + 0x5EED)))
    perm = np.argsort(keys, kind="stable")
    P = np.zeros((n, n), dtype=np.float32)
    P[np.arange(n), perm] = 1.0
    return P, perm

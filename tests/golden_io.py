"""Reader for the worked-example fixtures under tests/golden/ (each file cites
the passage its values come from in its header comments)."""
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_files():
    return sorted(f for f in os.listdir(GOLDEN_DIR) if f.endswith(".txt"))


def read_golden(name):
    lines = [ln.split("#", 1)[0].strip() for ln in open(os.path.join(GOLDEN_DIR, name))]
    lines = [ln for ln in lines if ln]
    assert lines[0] == "M N K"
    M, N, K = (int(x) for x in lines[1].split())
    pos = 2

    def block(tag, rows):
        nonlocal pos
        assert lines[pos] == tag, (name, lines[pos], tag)
        pos += 1
        out = np.array([[float(x) for x in lines[pos + r].split()] for r in range(rows)])
        pos += rows
        return out

    A = block("A", M)
    B = block("B", K)
    C = block("C", M)
    assert A.shape == (M, K) and B.shape == (K, N) and C.shape == (M, N)
    return M, N, K, A.astype(np.float32), B.astype(np.float32), C


SAXPY_DIR = os.path.join(GOLDEN_DIR, "saxpy")


def saxpy_golden_files():
    return sorted(f for f in os.listdir(SAXPY_DIR) if f.endswith(".txt"))


def read_saxpy_golden(name):
    """(n, alpha, incx, incy, x buffer, y buffer, expected out[0:n])."""
    lines = [ln.split("#", 1)[0].strip() for ln in open(os.path.join(SAXPY_DIR, name))]
    lines = [ln for ln in lines if ln]
    assert lines[0] == "n alpha incx incy"
    n, alpha, incx, incy = lines[1].split()
    assert lines[2] == "x" and lines[4] == "y" and lines[6] == "out"
    x = np.array([float(v) for v in lines[3].split()], dtype=np.float32)
    y = np.array([float(v) for v in lines[5].split()], dtype=np.float32)
    out = np.array([float(v) for v in lines[7].split()])
    return int(n), float(alpha), int(incx), int(incy), x, y, out


COULOMB_DIR = os.path.join(GOLDEN_DIR, "coulomb")


def coulomb_golden_files():
    return sorted(f for f in os.listdir(COULOMB_DIR) if f.endswith(".txt"))


def read_coulomb_golden(name):
    """(sources (ns,3) f32, charges (ns,) f32, targets (nt,3) f32, expected phi (nt,),
    expected normaliser D (nt,) = sum_j |q_j| / r_ij, worked by hand in each file)."""
    lines = [ln.split("#", 1)[0].strip() for ln in open(os.path.join(COULOMB_DIR, name))]
    lines = [ln for ln in lines if ln]
    i_t, i_p = lines.index("targets x y z"), lines.index("phi")
    i_d = lines.index("D")
    assert lines[0] == "sources x y z q"
    src = np.array([[float(v) for v in ln.split()] for ln in lines[1:i_t]])
    tgt = np.array([[float(v) for v in ln.split()] for ln in lines[i_t + 1:i_p]])
    phi = np.array([float(ln) for ln in lines[i_p + 1:i_d]])
    D = np.array([float(ln) for ln in lines[i_d + 1:]])
    assert src.shape[1] == 4 and tgt.shape[1] == 3 and phi.shape[0] == tgt.shape[0] == D.shape[0]
    return (src[:, :3].astype(np.float32), src[:, 3].astype(np.float32), tgt.astype(np.float32), phi, D)

"""Pins for the 3D Coulomb oracle (oracle/oracle.c lpy_oracle_coulomb_f64,
Table 1's "3D Coulomb pot." row): hand-worked fixtures
(tests/golden/coulomb/, each citing its arithmetic), 40-digit decimal brute
force, exact symmetries (power-of-two scaling, integer translation, pair
reciprocity, target order), superposition, coincident-point exclusion and a
scipy cross-check.  A wrong sign, a dropped coordinate, r^2 instead of r, a
missing exclusion or a target/source mix-up fails at least one.  No GPU."""
from decimal import Decimal, getcontext

import numpy as np
import pytest

import oracle
import synth
from golden_io import coulomb_golden_files, read_coulomb_golden


def run(tgt, src, q, ldt=3, lds=3, nthreads=0):
    """tgt (nt,3), src (ns,3) float32 arrays -> oracle (phi, D)."""
    def lay(p, ld):
        if p.shape[0] == 0:
            return np.zeros(0, np.float32)
        buf = np.full((p.shape[0], ld), np.nan, np.float32)
        buf[:, :3] = p
        return buf.reshape(-1)[: (p.shape[0] - 1) * ld + 3].copy()
    return oracle.coulomb(tgt.shape[0], lay(tgt, ldt), ldt, src.shape[0], lay(src, lds), lds,
                          np.ascontiguousarray(q, dtype=np.float32), nthreads=nthreads)


def cloud(n, seed, charges="uniform"):
    pos, q = synth.particles(n, seed, charges)
    return pos.reshape(n, 3), q


@pytest.mark.parametrize("name", coulomb_golden_files())
@pytest.mark.parametrize("ldt,lds", [(3, 3), (4, 7), (7, 3)])
def test_coulomb_golden(name, ldt, lds):
    src, q, tgt, phi_exp, D_exp = read_coulomb_golden(name)
    phi, D = run(tgt, src, q, ldt, lds)
    # phi within a few float64 roundings of the hand value (relative to D: a
    # cancelling sum such as the dipole's phi = 0 has no relative precision)
    assert np.all(np.abs(phi - phi_exp) <= 4e-16 * D_exp)
    # the normaliser is pinned independently of the oracle's formula: hand
    # values with mixed-sign charges (dipole.txt, mixed_two.txt) catch a
    # missing |q|, a scaled D or D computed from phi
    np.testing.assert_allclose(D, D_exp, rtol=4e-16, atol=0)


def test_coulomb_golden_D_is_phi_for_positive_charges():
    """For non-negative charges every term of D equals the term of phi, so D == phi
    bitwise (the same float64 operations in the same order)."""
    for name in coulomb_golden_files():
        src, q, tgt, _, _ = read_coulomb_golden(name)
        if np.all(q >= 0):
            phi, D = run(tgt, src, q)
            np.testing.assert_array_equal(D, phi)
    src, q = cloud(300, 11, "uniform01")
    phi, D = run(src[:40], src, q)
    np.testing.assert_array_equal(D, phi)
    # flipping every sign flips phi and leaves D unchanged
    phi_n, D_n = run(src[:40], src, -q)
    np.testing.assert_array_equal(phi_n, -phi)
    np.testing.assert_array_equal(D_n, D)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_coulomb_decimal_brute_force(seed):
    getcontext().prec = 40
    src, q = cloud(23, seed)
    tgt, _ = cloud(7, seed + 100)
    tgt = np.concatenate([tgt, src[:3]])           # three targets coincide with sources
    phi, D = run(tgt, src, q)
    for i in range(tgt.shape[0]):
        exact = Decimal(0)
        for j in range(src.shape[0]):
            d2 = sum((Decimal(float(tgt[i, c])) - Decimal(float(src[j, c]))) ** 2 for c in range(3))
            if d2 != 0:
                exact += Decimal(float(q[j])) / d2.sqrt()
        assert abs(Decimal(float(phi[i])) - exact) <= Decimal(1e-14) * Decimal(float(D[i]))


def test_coulomb_exact_symmetries():
    src, q = cloud(300, 3)
    tgt, _ = cloud(50, 4)
    phi, D = run(tgt, src, q)
    # power-of-two scaling of all positions: every float64 step scales exactly
    phi_s, _ = run(tgt * np.float32(4), src * np.float32(4), q)
    np.testing.assert_array_equal(phi_s, phi / 4)
    # target order does not matter (each target is computed alone)
    perm = np.random.default_rng(0).permutation(tgt.shape[0])
    np.testing.assert_array_equal(run(tgt[perm], src, q)[0], phi[perm])
    # source order changes only the summation rounding
    sp = np.random.default_rng(1).permutation(src.shape[0])
    assert np.max(np.abs(run(tgt, src[sp], q[sp])[0] - phi) / D) < 1e-14
    # thread count does not matter
    np.testing.assert_array_equal(run(tgt, src, q, nthreads=3)[0], phi)


def test_coulomb_integer_translation_and_reciprocity():
    rng = np.random.default_rng(5)
    src = rng.integers(-50, 50, size=(40, 3)).astype(np.float32)
    q = rng.integers(-8, 9, size=40).astype(np.float32)
    phi, _ = run(src, src, q)
    shift = np.array([1024, -512, 7], np.float32)
    np.testing.assert_array_equal(run(src + shift, src + shift, q)[0], phi)   # exact differences
    a = np.array([[0.25, -1.5, 3.0], [2.0, 0.5, -0.75]], np.float32)
    qa = np.array([0.5, -3.0], np.float32)
    pa, _ = run(a, a, qa)
    assert pa[0] * qa[0] == pa[1] * qa[1]                                       # q0 q1 / r both ways


def test_coulomb_superposition_and_exclusion():
    src, q1 = cloud(200, 6)
    q2 = synth.vector(200, 7, synth.CHARGES, "int") * np.float32(2.0 ** -10)
    q12 = q1 + q2
    assert np.array_equal(q12.astype(np.float64), q1.astype(np.float64) + q2.astype(np.float64))
    tgt, _ = cloud(30, 8)
    p1, D1 = run(tgt, src, q1)
    p2, D2 = run(tgt, src, q2)
    p12, _ = run(tgt, src, q12)
    assert np.max(np.abs(p12 - (p1 + p2)) / (D1 + D2)) < 1e-14
    # a target on top of source k sees exactly the set without source k
    k = 17
    on = src[k:k + 1]
    keep = np.arange(200) != k
    np.testing.assert_array_equal(run(on, src, q1)[0], run(on, src[keep], q1[keep])[0])
    # zero charges and an empty source set give zero
    np.testing.assert_array_equal(run(tgt, src, np.zeros(200, np.float32))[0], np.zeros(30))
    np.testing.assert_array_equal(run(tgt, src[:0], q1[:0])[0], np.zeros(30))
    assert run(tgt[:0], src, q1)[0].shape == (0,)


def test_coulomb_scipy_crosscheck():
    from scipy.spatial.distance import cdist
    src, q = cloud(2000, 9)
    tgt = src[:500]
    phi, D = run(tgt, src, q)
    d = cdist(tgt.astype(np.float64), src.astype(np.float64))
    with np.errstate(divide="ignore"):
        w = np.where(d > 0, 1.0 / d, 0.0)
    ref = w @ q.astype(np.float64)
    assert np.max(np.abs(phi - ref) / D) < 1e-13
    np.testing.assert_allclose(D, w @ np.abs(q.astype(np.float64)), rtol=1e-13)


def test_coulomb_rejects_bad_arguments():
    p = np.zeros(6, np.float32)
    with pytest.raises(ValueError):
        oracle.coulomb(2, p, 2, 2, p, 3, np.zeros(2, np.float32))      # ld < 3
    with pytest.raises(ValueError):
        oracle.coulomb(3, p, 3, 2, p, 3, np.zeros(2, np.float32))      # buffer too short

"""Pins for the saxpy oracle (oracle/oracle.c lpy_oracle_saxpy_f64, Table 1's
saxpy row) and for the half-ulp checker the GPU parity tests
use -- against exact rational arithmetic, hand-worked fixtures
(tests/golden/saxpy/, each citing its source), closed forms and numpy.  A
dropped term, a wrong sign, alpha applied to y instead of x, or a wrong
increment fails at least one of them.  No GPU involved."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from golden_io import read_saxpy_golden, saxpy_golden_files


@pytest.mark.parametrize("name", saxpy_golden_files())
def test_saxpy_golden(name):
    n, alpha, incx, incy, x, y, out = read_saxpy_golden(name)
    ref = oracle.saxpy(n, alpha, x, incx, y, incy)
    assert np.array_equal(ref, out)
    y0 = y.copy()
    oracle.saxpy(n, alpha, x, incx, y, incy)
    assert np.array_equal(y, y0), "the oracle only reads y"


@pytest.mark.parametrize("dist", synth.DISTS)
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_saxpy_exact_rational(dist, seed):
    n = 64
    x = synth.vector(n, seed, synth.VECTOR_X, dist)
    y = synth.vector(n, seed, synth.VECTOR_Y, dist)
    for alpha in (1.0, -0.75, 3.0517578125e-05, float(np.float32(1 / 3)), 12345.678):
        alpha = float(np.float32(alpha))
        ref = oracle.saxpy(n, alpha, x, 1, y, 1)
        for i in range(n):
            exact = Fraction(alpha) * Fraction(float(x[i])) + Fraction(float(y[i]))
            err = abs(Fraction(float(ref[i])) - exact)
            assert err <= abs(exact) * Fraction(1, 2 ** 53), (dist, alpha, i)
            if dist == "int" and alpha == 1.0:
                assert Fraction(float(ref[i])) == exact


def test_saxpy_closed_forms():
    n = 1000
    x = synth.vector(n, 4, synth.VECTOR_X)
    y = synth.vector(n, 4, synth.VECTOR_Y)
    assert np.array_equal(oracle.saxpy(n, 0.0, x, 1, y, 1), y.astype(np.float64))     # alpha = 0
    assert np.array_equal(oracle.saxpy(n, 1.0, x, 1, np.zeros(n, np.float32), 1),
                          x.astype(np.float64))                                       # y = 0
    assert np.array_equal(oracle.saxpy(n, -1.0, x, 1, x, 1), np.zeros(n))             # x - x
    assert np.array_equal(oracle.saxpy(n, 1.0, x, 1, x, 1), 2.0 * x.astype(np.float64))
    assert np.array_equal(oracle.saxpy(n, 2.0, x, 1, y, 1) - y.astype(np.float64),
                          2.0 * x.astype(np.float64))                                 # exact here
    assert oracle.saxpy(0, 2.0, x, 1, y, 1).shape == (0,)


@pytest.mark.parametrize("incx,incy", [(1, 1), (2, 1), (1, 3), (5, 7)])
def test_saxpy_increments(incx, incy):
    n = 333
    x = synth.vector(n, 5, synth.VECTOR_X)
    y = synth.vector(n, 5, synth.VECTOR_Y)
    dense = oracle.saxpy(n, 1.5, x, 1, y, 1)
    got = oracle.saxpy(n, 1.5, synth.strided(x, incx), incx, synth.strided(y, incy), incy)
    assert np.array_equal(got, dense)


def test_saxpy_library_crosscheck():
    n = 1 << 16
    x = synth.vector(n, 6, synth.VECTOR_X, "wide")
    y = synth.vector(n, 6, synth.VECTOR_Y, "wide")
    ref = oracle.saxpy(n, -2.5, x, 1, y, 1, nthreads=3)
    np.testing.assert_array_equal(ref, -2.5 * x.astype(np.float64) + y.astype(np.float64))


def test_saxpy_rejects_bad_arguments():
    x = np.zeros(4, np.float32)
    with pytest.raises(ValueError):
        oracle.saxpy(4, 1.0, x, 0, x, 1)
    with pytest.raises(ValueError):
        oracle.saxpy(4, 1.0, x, 2, x, 1)   # buffer too short for the stride


def test_half_ulp_checker():
    """saxpy_error_ulps: the fp32 round-to-nearest of a value scores <= 1, the
    neighbouring fp32 values score > 1 -- including at binade edges, for
    negatives and in the subnormal range."""
    ref = np.array([1.0 + 2.0 ** -30, 1.0 - 2.0 ** -30, -3.0 + 2.0 ** -26, 0.7, 2.0 ** -140 * 1.3,
                    2.0 ** 20 + 0.3, 0.0])
    rn = ref.astype(np.float32)
    assert oracle.saxpy_error_ulps(rn, ref) <= 1.0
    for i in range(ref.size):
        for direction in (np.inf, -np.inf):
            bad = rn.copy()
            bad[i] = np.nextafter(rn[i], np.float32(direction))
            if np.float64(bad[i]) == np.float64(rn[i]):
                continue
            assert oracle.saxpy_error_ulps(bad, ref) > 1.0, (i, direction)

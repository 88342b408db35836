"""Pins for the float64 CPU oracle (oracle/oracle.c) -- checked against things
other than itself: exact rational brute force, hand-worked examples with
citations (tests/golden/), closed forms, invariants and a library routine.
Each pin is chosen so a plausible slip in the oracle (dropped term, wrong sign,
swapped index, transposed operand, wrong layout accessor, missing zero-init)
fails at least one of them.  No GPU involved."""
from fractions import Fraction
import itertools

import numpy as np
import pytest

import oracle
import synth
from golden_io import golden_files, read_golden

LAYOUTS = (synth.ROW_MAJOR, synth.COL_MAJOR)
U = 2.0 ** -53


def run_oracle(A, B, la=0, lb=0, pad_a=0, pad_b=0, nthreads=0):
    M, K = A.shape
    _, N = B.shape
    abuf, lda = synth.store(A, la, synth.min_ld(M, K, la) + pad_a)
    bbuf, ldb = synth.store(B, lb, synth.min_ld(K, N, lb) + pad_b)
    return oracle.gemm(M, N, K, abuf, lda, la, bbuf, ldb, lb, nthreads=nthreads)


def exact_product(A, B):
    """Brute force in exact rational arithmetic (fp32 values are dyadic)."""
    M, K = A.shape
    N = B.shape[1]
    Af = [[Fraction(float(A[i, k])) for k in range(K)] for i in range(M)]
    Bf = [[Fraction(float(B[k, j])) for j in range(N)] for k in range(K)]
    return [[sum((Af[i][k] * Bf[k][j] for k in range(K)), Fraction(0)) for j in range(N)]
            for i in range(M)]


@pytest.mark.parametrize("name", golden_files())
@pytest.mark.parametrize("la,lb", list(itertools.product(LAYOUTS, LAYOUTS)))
@pytest.mark.parametrize("pad", [0, 3])
def test_golden_worked_examples(name, la, lb, pad):
    M, N, K, A, B, Cexp = read_golden(name)
    C, D = run_oracle(A, B, la, lb, pad, pad)
    assert np.array_equal(C, Cexp)
    assert np.all(D >= np.abs(C))


@pytest.mark.parametrize("dist", synth.DISTS)
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_brute_force_exact_rational_tiny(dist, seed):
    rng = np.random.default_rng(seed)
    for trial in range(4):
        M, N, K = (int(x) for x in rng.integers(1, 7, size=3))
        A = synth.matrix(M, K, seed=seed * 10 + trial, matrix_id=0, dist=dist)
        B = synth.matrix(K, N, seed=seed * 10 + trial, matrix_id=1, dist=dist)
        exact = exact_product(A, B)
        for la, lb in itertools.product(LAYOUTS, LAYOUTS):
            C, D = run_oracle(A, B, la, lb, pad_a=trial, pad_b=1)
            for i in range(M):
                for j in range(N):
                    err = abs(Fraction(C[i, j]) - exact[i][j])
                    # float64 recursive summation bound: (K-1) u sum|terms| (+ tiny slack)
                    bound = Fraction((K - 1) * U * (1 + 1e-12)) * Fraction(D[i, j])
                    assert err <= bound, (dist, M, N, K, la, lb, i, j)
                    if dist == "int":
                        assert err == 0


def test_identity_gives_b_exactly():
    n = 37
    B = synth.matrix(n, 23, seed=5, matrix_id=1)
    for la, lb in itertools.product(LAYOUTS, LAYOUTS):
        C, _ = run_oracle(synth.identity(n), B, la, lb)
        assert np.array_equal(C, B.astype(np.float64))
        C2, _ = run_oracle(B.T.copy(), synth.identity(n), la, lb)   # right identity
        assert np.array_equal(C2, B.T.astype(np.float64))


def test_permutation_permutes_rows_exactly():
    n = 41
    P, perm = synth.permutation(n, seed=3)
    B = synth.matrix(n, 19, seed=6, matrix_id=1, dist="wide")
    for la, lb in itertools.product(LAYOUTS, LAYOUTS):
        C, _ = run_oracle(P, B, la, lb)
        assert np.array_equal(C, B[perm].astype(np.float64))


def test_rank_one_k1_is_outer_product():
    u = synth.matrix(29, 1, seed=7, matrix_id=0)
    v = synth.matrix(1, 31, seed=7, matrix_id=1)
    C, D = run_oracle(u, v)
    exp = u.astype(np.float64) * v.astype(np.float64)    # fp32*fp32 exact in float64
    assert np.array_equal(C, exp)
    assert np.array_equal(D, np.abs(exp))


def test_rank_one_constant_along_k():
    # A[i,k] = u_i, B[k,j] = v_j  =>  C = K u v^T   (rank-1 idea)
    K = 32                      # 48-bit products, K*p needs <= 53 bits: exact
    u = synth.matrix(17, 1, seed=8, matrix_id=0)
    v = synth.matrix(1, 13, seed=8, matrix_id=1)
    A = np.repeat(u, K, axis=1)
    B = np.repeat(v, K, axis=0)
    C, _ = run_oracle(A, B, 0, 1)
    assert np.array_equal(C, K * (u.astype(np.float64) * v.astype(np.float64)))


def test_zero_inputs_and_k_zero():
    A = np.zeros((5, 4), np.float32)
    B = synth.matrix(4, 6, seed=1, matrix_id=1)
    C, D = run_oracle(A, B)
    assert np.array_equal(C, np.zeros((5, 6))) and np.array_equal(D, np.zeros((5, 6)))
    # K == 0: sum over an empty k range is the identity 0
    C0, D0 = oracle.gemm(3, 4, 0, np.zeros(0, np.float32), 1, 0, np.zeros(0, np.float32), 4, 0)
    assert C0.shape == (3, 4) and not C0.any() and not D0.any()
    # M == 0 / N == 0: empty domain
    Ce, _ = oracle.gemm(0, 4, 3, np.zeros(0, np.float32), 3, 0, np.ones(12, np.float32), 4, 0)
    assert Ce.shape == (0, 4)


def test_sign_flip_and_transpose_identities():
    A = synth.matrix(11, 9, seed=2, matrix_id=0)
    B = synth.matrix(9, 7, seed=2, matrix_id=1)
    C, D = run_oracle(A, B)
    Cn, Dn = run_oracle(-A, B)
    assert np.array_equal(Cn, -C) and np.array_equal(Dn, D)
    # (A B)^T = B^T A^T, exactly: same products, same k order
    Ct, Dt = run_oracle(B.T.copy(), A.T.copy())
    assert np.array_equal(Ct, C.T) and np.array_equal(Dt, D.T)


def test_nonnegative_inputs_D_equals_C():
    A = synth.matrix(13, 21, seed=4, matrix_id=0, dist="uniform01")
    B = synth.matrix(21, 8, seed=4, matrix_id=1, dist="uniform01")
    C, D = run_oracle(A, B)
    assert np.array_equal(C, D)
    C2, D2 = run_oracle(A, -B)
    assert np.array_equal(C2, -D) and np.array_equal(D2, D)


@pytest.mark.parametrize("shape", [(64, 48, 80), (130, 70, 257), (257, 129, 300)])
def test_numpy_float64_cross_check(shape):
    M, N, K = shape
    A = synth.matrix(M, K, seed=9, matrix_id=0)
    B = synth.matrix(K, N, seed=9, matrix_id=1)
    for la, lb in itertools.product(LAYOUTS, LAYOUTS):
        C, D = run_oracle(A, B, la, lb, pad_a=5, pad_b=2)
        ref = A.astype(np.float64) @ B.astype(np.float64)
        Dref = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64))
        assert oracle.normalized_error(C, ref, D) <= 1e-12
        np.testing.assert_allclose(D, Dref, rtol=1e-12)


def test_layout_invariance_and_thread_invariance_bitwise():
    A = synth.matrix(45, 33, seed=11, matrix_id=0, dist="uniform01")
    B = synth.matrix(33, 27, seed=11, matrix_id=1, dist="uniform01")
    C0, D0 = run_oracle(A, B, 0, 0, nthreads=1)
    for la, lb in itertools.product(LAYOUTS, LAYOUTS):
        for nt in (1, 3, 0):
            C, D = run_oracle(A, B, la, lb, pad_a=2, pad_b=7, nthreads=nt)
            assert np.array_equal(C, C0) and np.array_equal(D, D0)


def test_rows_and_elements_match_full_bitwise():
    M, N, K = 50, 40, 70
    A = synth.matrix(M, K, seed=12, matrix_id=0)
    B = synth.matrix(K, N, seed=12, matrix_id=1)
    abuf, lda = synth.store(A, 1, M + 3)
    bbuf, ldb = synth.store(B, 0, N)
    C, D = oracle.gemm(M, N, K, abuf, lda, 1, bbuf, ldb, 0)
    Cr, Dr = oracle.gemm_rows(M, N, K, abuf, lda, 1, bbuf, ldb, 0, 17, 33)
    assert np.array_equal(Cr, C[17:33]) and np.array_equal(Dr, D[17:33])
    ii = np.array([0, 49, 17, 3, 49])
    jj = np.array([0, 39, 5, 38, 0])
    Ce, De = oracle.gemm_elems(M, N, K, abuf, lda, 1, bbuf, ldb, 0, ii, jj)
    assert np.array_equal(Ce, C[ii, jj]) and np.array_equal(De, D[ii, jj])


def test_oracle_rejects_bad_arguments():
    with pytest.raises(ValueError):
        oracle.gemm_rows(4, 4, 4, np.ones(16, np.float32), 4, 0, np.ones(16, np.float32), 4, 0, 3, 2)
    with pytest.raises(ValueError):
        oracle.gemm_elems(4, 4, 4, np.ones(16, np.float32), 4, 0, np.ones(16, np.float32), 4, 0,
                          [4], [0])


def test_normalized_error_metric():
    Cref = np.array([[1.0, 0.0], [2.0, -3.0]])
    D = np.array([[2.0, 0.0], [4.0, 6.0]])
    assert oracle.normalized_error(Cref, Cref, D) == 0.0
    C = Cref + np.array([[1e-6, 0.0], [0.0, 0.0]])
    assert abs(oracle.normalized_error(C, Cref, D) - 5e-7) < 1e-15
    C[0, 1] = 1e-30                              # D == 0 needs an exact zero (reading A1)
    assert oracle.normalized_error(C, Cref, D) == float("inf")
    C[0, 1] = np.nan
    assert oracle.normalized_error(C, Cref, D) == float("inf")
